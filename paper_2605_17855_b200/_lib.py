"""ctypes binding of libtgs.so (include/tgs.h).  No CPU fallback: if the library cannot be
loaded (or built in-tree with nvcc) importing the render API fails loudly."""
from __future__ import annotations

import ctypes as C
import os
import threading

from . import build as _build

_LOCK = threading.Lock()
_LIB = None

c_status = C.c_int


class tgs_camera(C.Structure):
    _fields_ = [("view", C.c_float * 16), ("focal_x", C.c_float), ("focal_y", C.c_float),
                ("width", C.c_int32), ("height", C.c_int32), ("near", C.c_float),
                ("far", C.c_float)]


class tgs_options(C.Structure):
    _fields_ = [("backend", C.c_int32), ("mode", C.c_int32), ("group_size", C.c_int32),
                ("workers", C.c_int32), ("chunk_len", C.c_int32), ("alpha_skip", C.c_float),
                ("alpha_clamp", C.c_float), ("t_terminate", C.c_float)]


class tgs_stats(C.Structure):
    _fields_ = [("input", C.c_uint64), ("culled", C.c_uint64), ("dropped_degenerate", C.c_uint64),
                ("entries", C.c_uint64), ("tile_appearances", C.c_uint64), ("visible", C.c_uint64),
                ("ms_preprocess", C.c_float), ("ms_binning", C.c_float), ("ms_sort", C.c_float),
                ("ms_raster", C.c_float), ("ms_total", C.c_float),
                ("fragment_ops", C.c_uint64), ("chunk_loads", C.c_uint64), ("skipped_pairs", C.c_uint64),
                ("used_lanes", C.c_uint64), ("total_lanes", C.c_uint64)]


P = C.c_void_p
F32P = C.POINTER(C.c_float)

# name -> (restype, argtypes); the ABI test checks this table against include/tgs.h.
SIGNATURES = {
    "tgs_last_error": (C.c_char_p, []),
    "tgs_abi_version": (C.c_int, []),
    "tgs_ctx_create": (c_status, [C.c_int, C.POINTER(P)]),
    "tgs_ctx_destroy": (None, [P]),
    "tgs_ctx_stream": (P, [P]),
    "tgs_set_tile_cull": (c_status, [P, C.c_int]),
    "tgs_set_graphs": (c_status, [P, C.c_int]),
    "tgs_set_exact_emulation": (c_status, [P, C.c_int]),
    "tgs_scene_upload": (c_status, [P, F32P, C.c_int64, C.c_int, C.POINTER(P)]),
    "tgs_scene_free": (None, [P]),
    "tgs_render": (c_status, [P, P, C.POINTER(tgs_camera), C.POINTER(tgs_options), F32P,
                              C.POINTER(tgs_stats)]),
    "tgs_render_records": (c_status, [P, F32P, C.c_int64, C.c_int, C.POINTER(tgs_camera),
                                      C.POINTER(tgs_options), F32P, C.POINTER(tgs_stats)]),
    "tgs_render_enqueue": (c_status, [P, P, C.POINTER(tgs_camera), C.POINTER(tgs_options)]),
    "tgs_sync": (c_status, [P, C.POINTER(tgs_stats)]),
    "tgs_image_device": (P, [P]),
    "tgs_render_band": (c_status, [P, P, C.POINTER(tgs_camera), C.POINTER(tgs_options), C.c_int,
                                   C.c_int, F32P, C.POINTER(tgs_stats)]),
    "tgs_render_batch": (c_status, [P, P, C.POINTER(tgs_camera), C.c_int, C.POINTER(tgs_options),
                                    F32P, C.POINTER(tgs_stats)]),
    "tgs_read_projected": (c_status, [P, P, C.c_int64, C.POINTER(C.c_int64)]),
    "tgs_read_lists": (c_status, [P, P, C.c_int64, P, C.c_int64, C.POINTER(C.c_int64)]),
    "tgs_count_pairs": (c_status, [P, C.POINTER(C.c_uint64), C.POINTER(C.c_uint64)]),
    "tgs_reuse_report": (c_status, [P, C.POINTER(C.c_uint64), C.POINTER(C.c_uint64), C.POINTER(C.c_double),
                                    C.POINTER(C.c_uint64)]),
    "tgs_tile_trips": (c_status, [P, P, C.c_int64, C.POINTER(C.c_int64)]),
    "tgs_gen_synthetic_scene": (c_status, [C.c_uint64, C.c_int, C.c_float, C.c_float, C.c_float,
                                           C.c_uint64, F32P]),
    "tgs_encode_u8": (c_status, [P, P, C.c_int64, P]),
    "tgs_group_row_entries": (c_status, [P, P, C.POINTER(tgs_camera), C.POINTER(tgs_options), P, C.c_int64,
                                         C.POINTER(C.c_int64)]),
    "tgs_project_scene": (c_status, [P, F32P, C.c_int64, C.c_int, C.POINTER(tgs_camera), P, C.c_int64,
                                     C.POINTER(C.c_int64), C.POINTER(tgs_stats)]),
    "tgs_build_group_entries": (c_status, [P, P, C.c_int64, C.c_int, C.c_int, C.c_int, P, C.c_int64,
                                           C.POINTER(C.c_int64)]),
    "tgs_sort_entries": (c_status, [P, P, C.c_int64, C.c_int, C.c_int, C.c_int, P, P, C.c_int64]),
    "tgs_rasterize_lists": (c_status, [P, P, C.c_int64, P, C.c_int64, P, C.c_int64, C.c_int, C.c_int,
                                       C.POINTER(tgs_options), F32P]),
}


def lib_path() -> str:
    return _build.LIB


def load():
    """Load (building in-tree if needed) and type the library; raises on any failure."""
    global _LIB
    with _LOCK:
        if _LIB is not None:
            return _LIB
        path = os.environ.get("TGS_LIB") or _build.LIB  # TGS_LIB: a variant build (tools/build_variant.py)
        if not os.path.exists(path):
            _build.build()
        lib = C.CDLL(path)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        if lib.tgs_abi_version() != 2:
            raise ImportError("libtgs ABI version mismatch")
        _LIB = lib
        return lib


def last_error() -> str:
    return load().tgs_last_error().decode(errors="replace")
