"""oracle.oracle — TEST INFRASTRUCTURE ONLY.

ctypes bindings for the two CPU oracles of the forward render path:

* ``Port``  -> oracle/libtgs_oracle.so: our C restatement (tgs_oracle.c), built by ``make port``.
* ``Ref``   -> oracle/_ref/libgsr_ref.so: the reference's own sources compiled against the
  vendored Eigen subset (``make ref``, needs /root/reference; the built .so travels to the GPU
  box with the snapshot).

Only tests/, ``__graft_entry__.smoke()`` and bench.py's CPU legs may import this module, and only
as the checker / the timed CPU baseline.  The product path (paper_2605_17855_b200) never imports
it.  Both classes expose the same methods so tests can parametrise over them.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
PORT_SO = os.path.join(HERE, "libtgs_oracle.so")
REF_SO = os.path.join(HERE, "_ref", "libgsr_ref.so")
REF_SRC = "/root/reference/proj"

PROJ_DTYPE = np.dtype([("mean2d", "<f4", 2), ("conic", "<f4", 3), ("color", "<f4", 3),
                       ("opacity", "<f4"), ("depth", "<f4"), ("radius", "<i4")])
ENTRY_DTYPE = np.dtype([("gaussian_index", "<u4"), ("depth", "<f4"), ("mask", "<u4")])
assert PROJ_DTYPE.itemsize == 44 and ENTRY_DTYPE.itemsize == 12


class CCamera(C.Structure):
    _fields_ = [("view", C.c_float * 16), ("focal_x", C.c_float), ("focal_y", C.c_float),
                ("width", C.c_int32), ("height", C.c_int32), ("near", C.c_float),
                ("far", C.c_float)]


class COptions(C.Structure):
    _fields_ = [("backend", C.c_int32), ("mode", C.c_int32), ("group_size", C.c_int32),
                ("workers", C.c_int32), ("chunk_len", C.c_int32), ("alpha_skip", C.c_float),
                ("alpha_clamp", C.c_float), ("t_terminate", C.c_float)]


class CCounters(C.Structure):
    _fields_ = [(n, C.c_uint64) for n in ("fragment_ops", "chunk_loads", "skipped_pairs",
                                          "used_lanes", "total_lanes", "walked_pairs",
                                          "blended_pairs")]


def build(ref: bool | None = None) -> None:
    """Build the port (always) and the reference oracle (when /root/reference is present)."""
    subprocess.run(["make", "-s", "-C", HERE, "port"], check=True)
    if ref is None:
        ref = os.path.isdir(REF_SRC)
    if ref:
        subprocess.run(["make", "-s", "-C", HERE, "ref"], check=True)


def make_camera(cam) -> CCamera:
    """Accepts anything with view (4x4, row-major), focal_x/y, width, height, near, far."""
    c = CCamera()
    v = np.asarray(cam.view, dtype=np.float32).reshape(4, 4)
    for i in range(16):
        c.view[i] = float(v.flat[i])
    c.focal_x, c.focal_y = float(cam.focal_x), float(cam.focal_y)
    c.width, c.height = int(cam.width), int(cam.height)
    c.near, c.far = float(cam.near), float(cam.far)
    return c


def make_options(backend=1, mode=0, group_size=2, workers=1, chunk_len=16,
                 alpha_skip=1.0 / 255.0, alpha_clamp=0.99, t_terminate=1e-4) -> COptions:
    o = COptions()
    o.backend, o.mode, o.group_size = int(backend), int(mode), int(group_size)
    o.workers, o.chunk_len = int(workers), int(chunk_len)
    o.alpha_skip = np.float32(alpha_skip)
    o.alpha_clamp = np.float32(alpha_clamp)
    o.t_terminate = np.float32(t_terminate)
    return o


def _f32p(a):
    return a.ctypes.data_as(C.POINTER(C.c_float))


class _Base:
    prefix = ""
    so_path = ""

    def __init__(self):
        if not os.path.exists(self.so_path):
            raise FileNotFoundError(f"oracle library missing: {self.so_path} (run oracle.build())")
        self.lib = C.CDLL(self.so_path)

    def _fn(self, name):
        return getattr(self.lib, self.prefix + name)

    # -- scenes ------------------------------------------------------------------------------
    def gen_scene(self, seed, count, extent=1.0, smin=0.01, smax=0.05, sh_seed=0):
        rf = 59 if sh_seed else 14
        out = np.zeros((count, rf), dtype=np.float32)
        f = self._fn("gen_scene")
        f.restype = C.c_int
        f.argtypes = [C.c_uint64, C.c_int, C.c_float, C.c_float, C.c_float, C.c_uint64,
                      C.POINTER(C.c_float)]
        rc = f(seed, count, extent, smin, smax, sh_seed, _f32p(out))
        if rc != 0:
            raise ValueError("gen_scene failed")
        return out

    # -- projection --------------------------------------------------------------------------
    def project(self, rec, cam):
        rec = np.ascontiguousarray(rec, dtype=np.float32)
        deg = 3 if rec.shape[1] == 59 else 0
        out = np.zeros(max(len(rec), 1), dtype=PROJ_DTYPE)
        st = np.zeros(3, dtype=np.uint64)
        f = self._fn("project")
        f.restype = C.c_int64
        args = [_f32p(rec), C.c_int64(len(rec)), C.c_int(deg), C.byref(make_camera(cam))]
        if self.prefix == "gref_":
            args.append(C.c_int(1))
        args += [out.ctypes.data_as(C.c_void_p), st.ctypes.data_as(C.POINTER(C.c_uint64))]
        n = f(*args)
        if n < 0:
            raise ValueError("project failed")
        return out[:n].copy(), st

    # -- binning + sort ------------------------------------------------------------------------
    def bin_sort(self, proj, width, height, g):
        proj = np.ascontiguousarray(proj, dtype=PROJ_DTYPE)
        f = self._fn("bin_sort")
        f.restype = C.c_int64
        f.argtypes = [C.c_void_p, C.c_int64, C.c_int, C.c_int, C.c_int, C.c_void_p, C.c_int64,
                      C.c_void_p, C.c_void_p]
        app = np.zeros(1, dtype=np.uint64)
        total = f(proj.ctypes.data, len(proj), width, height, g, None, 0, None,
                  app.ctypes.data)
        if total < 0:
            raise ValueError("bin_sort failed")
        tiles_x, tiles_y = (width + 15) // 16, (height + 15) // 16
        ng = ((tiles_x + g - 1) // g) * ((tiles_y + g - 1) // g)
        ent = np.zeros(max(total, 1), dtype=ENTRY_DTYPE)
        off = np.zeros(ng + 1, dtype=np.uint32)
        t2 = f(proj.ctypes.data, len(proj), width, height, g, ent.ctypes.data, total,
               off.ctypes.data, None)
        if t2 != total:
            raise ValueError("bin_sort failed (second pass)")
        return ent[:total].copy(), off, int(app[0])

    # -- full render -----------------------------------------------------------------------
    def render(self, rec, cam, **opt):
        rec = np.ascontiguousarray(rec, dtype=np.float32)
        deg = 3 if rec.shape[1] == 59 else 0
        img = np.zeros((int(cam.height), int(cam.width), 3), dtype=np.float32)
        st = np.zeros(10, dtype=np.uint64)
        f = self._fn("render")
        f.restype = C.c_int
        args = [_f32p(rec), C.c_int64(len(rec)), C.c_int(deg), C.byref(make_camera(cam)),
                C.byref(make_options(**opt)), _f32p(img), st.ctypes.data_as(C.c_void_p)]
        if self.prefix == "tor_":
            args.append(None)
        rc = f(*args)
        if rc != 0:
            raise ValueError(f"render failed ({rc})")
        keys = ("input", "culled", "dropped_degenerate", "entries", "tile_appearances",
                "fragment_ops", "chunk_loads", "skipped_pairs", "used_lanes", "total_lanes")
        return img, {k: int(v) for k, v in zip(keys, st)}

    def reference_render(self, proj, width, height):
        proj = np.ascontiguousarray(proj, dtype=PROJ_DTYPE)
        img = np.zeros((height, width, 3), dtype=np.float32)
        f = self._fn("reference_render")
        f.restype = C.c_int
        f(proj.ctypes.data_as(C.c_void_p), C.c_int64(len(proj)), C.c_int(width),
          C.c_int(height), _f32p(img))
        return img


class Port(_Base):
    prefix = "tor_"
    so_path = PORT_SO

    def bin_sort_fast(self, proj, width, height, g):
        """tor_bin_sort_fast: the same lists in O(entries) (full-size frames)."""
        proj = np.ascontiguousarray(proj, dtype=PROJ_DTYPE)
        f = self.lib.tor_bin_sort_fast
        f.restype = C.c_int64
        f.argtypes = [C.c_void_p, C.c_int64, C.c_int, C.c_int, C.c_int, C.c_void_p, C.c_int64,
                      C.c_void_p, C.c_void_p]
        app = np.zeros(1, dtype=np.uint64)
        total = f(proj.ctypes.data, len(proj), width, height, g, None, 0, None, app.ctypes.data)
        if total < 0:
            raise ValueError("bin_sort_fast failed")
        tiles_x, tiles_y = (width + 15) // 16, (height + 15) // 16
        ng = ((tiles_x + g - 1) // g) * ((tiles_y + g - 1) // g)
        ent = np.zeros(max(total, 1), dtype=ENTRY_DTYPE)
        off = np.zeros(ng + 1, dtype=np.uint32)
        t2 = f(proj.ctypes.data, len(proj), width, height, g, ent.ctypes.data, total, off.ctypes.data, None)
        if t2 != total:
            raise ValueError("bin_sort_fast failed (second pass)")
        return ent[:total], off, int(app[0])

    def rasterize(self, entries, offsets, proj, width, height, **opt):
        """Rasterise sorted lists; returns (image, counters dict incl. walked/blended pairs)."""
        entries = np.ascontiguousarray(entries, dtype=ENTRY_DTYPE)
        offsets = np.ascontiguousarray(offsets, dtype=np.uint32)
        proj = np.ascontiguousarray(proj, dtype=PROJ_DTYPE)
        img = np.zeros((height, width, 3), dtype=np.float32)
        cnt = CCounters()
        f = self.lib.tor_rasterize
        f.restype = C.c_int
        rc = f(entries.ctypes.data_as(C.c_void_p), offsets.ctypes.data_as(C.c_void_p),
               proj.ctypes.data_as(C.c_void_p), C.c_int(width), C.c_int(height),
               C.byref(make_options(**opt)), _f32p(img), C.byref(cnt))
        if rc != 0:
            raise ValueError("rasterize failed")
        return img, {n: int(getattr(cnt, n)) for n, _ in CCounters._fields_}

    def f32_to_f16(self, x: float) -> int:
        f = self.lib.tor_f32_to_f16
        f.restype = C.c_uint16
        f.argtypes = [C.c_float]
        return int(f(x))

    def encode_ppm(self, img):
        img = np.ascontiguousarray(img, dtype=np.float32)
        out = np.zeros(img.size, dtype=np.uint8)
        self.lib.tor_encode_ppm(_f32p(img), C.c_int64(img.size), out.ctypes.data_as(C.c_void_p))
        return out.reshape(img.shape)


class Ref(_Base):
    prefix = "gref_"
    so_path = REF_SO

    @staticmethod
    def available() -> bool:
        return os.path.exists(REF_SO)

    def hardware_concurrency(self) -> int:
        return int(self.lib.gref_hardware_concurrency())

    def save_scene(self, rec, path: str) -> None:
        rec = np.ascontiguousarray(rec, dtype=np.float32)
        deg = 3 if rec.shape[1] == 59 else 0
        rc = self.lib.gref_save_scene(_f32p(rec), C.c_int64(len(rec)), C.c_int(deg), path.encode())
        if rc:
            raise RuntimeError(f"reference save_scene failed ({rc}): {self.last_error()}")

    def load_scene(self, path: str):
        """(records, None) or (None, (code, message)) when the reference throws."""
        cnt, deg = C.c_int64(), C.c_int()
        rc = self.lib.gref_load_scene(path.encode(), None, C.c_int64(0), C.byref(cnt), C.byref(deg))
        if rc:
            return None, (rc, self.last_error())
        rf = 59 if deg.value == 3 else 14
        out = np.zeros((cnt.value, rf), np.float32)
        rc = self.lib.gref_load_scene(path.encode(), _f32p(out), C.c_int64(out.size), C.byref(cnt),
                                      C.byref(deg))
        if rc:
            return None, (rc, self.last_error())
        return out, None

    def raster_projected(self, proj, width, height, **opt):
        proj = np.ascontiguousarray(proj, dtype=PROJ_DTYPE)
        img = np.zeros((height, width, 3), dtype=np.float32)
        f = self.lib.gref_raster_projected
        f.restype = C.c_int
        rc = f(proj.ctypes.data_as(C.c_void_p), C.c_int64(len(proj)), C.c_int(width),
               C.c_int(height), C.byref(make_options(**opt)), _f32p(img))
        if rc != 0:
            raise ValueError(self.last_error())
        return img

    def time_stages(self, rec, cam, band_y0=0, band_h=0, **opt):
        """Reference stage API timed with steady_clock: (entries, {project,bin,sort,raster} ms)."""
        rec = np.ascontiguousarray(rec, dtype=np.float32)
        deg = 3 if rec.shape[1] == 59 else 0
        ms = np.zeros(4, dtype=np.float64)
        f = self.lib.gref_time_stages
        f.restype = C.c_int64
        n = f(_f32p(rec), C.c_int64(len(rec)), C.c_int(deg), C.byref(make_camera(cam)),
              C.byref(make_options(**opt)), C.c_int(band_y0), C.c_int(band_h),
              ms.ctypes.data_as(C.c_void_p))
        if n < 0:
            raise ValueError(self.last_error())
        return int(n), dict(zip(("project", "bin", "sort", "raster"), ms.tolist()))

    def time_bands(self, rec, cam, n_bands, band_first, band_count, image=None, **opt):
        """project_scene once, then bin/sort/raster per band (gref_time_bands):
        (image rows covered, project ms, [(bin, sort, raster) ms per band]).  `image` (optional,
        float32 H x W x 3, C-contiguous) receives the rendered bands' rows (copied after timing)."""
        rec = np.ascontiguousarray(rec, dtype=np.float32)
        deg = 3 if rec.shape[1] == 59 else 0
        ms = np.zeros(1 + 3 * band_count, dtype=np.float64)
        f = self.lib.gref_time_bands
        f.restype = C.c_int64
        rows = f(_f32p(rec), C.c_int64(len(rec)), C.c_int(deg), C.byref(make_camera(cam)),
                 C.byref(make_options(**opt)), C.c_int(n_bands), C.c_int(band_first), C.c_int(band_count),
                 ms.ctypes.data_as(C.c_void_p), None if image is None else _f32p(image))
        if rows < 0:
            raise ValueError(self.last_error())
        return int(rows), float(ms[0]), [tuple(ms[1 + 3 * b: 4 + 3 * b]) for b in range(band_count)]

    def last_error(self) -> str:
        f = self.lib.gref_last_error
        f.restype = C.c_char_p
        return f().decode()
