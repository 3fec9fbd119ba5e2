"""Python mirror of the reference's render API (namespace ``gsr``) on top of libtgs.

Names, argument meaning and error behaviour follow the reference headers so parity tests read like
the reference's own tests:

* types      — Gaussian3D, Camera, ImageBuffer, FormatError, ValidationError (types.hpp:14-69)
* options    — Backend, PrecisionMode, RasterConstants, RenderOptions, RenderResult
               (render.hpp:8-25, raster_scalar.hpp:14-18, operands.hpp:13)
* entry      — render(scene, cam, opt)  (render.hpp:30-31)
* stages     — project_scene, sort_entries-equivalent ``sorted_group_lists``, ``load_reduction``
               (projection.hpp:48-50, binning.hpp:68-73, metrics.hpp:29-34)
* scene I/O  — gen_synthetic_scene, SplitMix64 (scene_io.hpp:14-60), encode_ppm

Scenes are carried as ``Scene`` (an (n, 14|59) float32 record array in .gsb record order) so
million-splat scenes never become Python objects; ``render`` also accepts a list of Gaussian3D.
Everything here runs on the GPU through the C ABI; there is no CPU fallback.
"""
from __future__ import annotations

import ctypes as C
import enum
import math
from dataclasses import dataclass, field
from typing import Iterable, Optional, Sequence

import numpy as np

from . import _lib

kShRestCoeffs = 45
kTileSize = 16
kPsnrCap = 99.0


# --------------------------------------------------------------------------------------------
# errors (types.hpp:14-21)
# --------------------------------------------------------------------------------------------
class FormatError(RuntimeError):
    pass


class ValidationError(RuntimeError):
    pass


class DeviceError(RuntimeError):
    """CUDA failure or out-of-memory (no reference counterpart)."""


def _check(status: int):
    if status == 0:
        return
    msg = _lib.last_error()
    if status == 1:
        raise ValidationError(msg)
    if status == 2:
        raise FormatError(msg)
    raise DeviceError(msg)


# --------------------------------------------------------------------------------------------
# domain types
# --------------------------------------------------------------------------------------------
@dataclass
class Gaussian3D:
    """World-space anisotropic Gaussian (types.hpp:26-33); rotation is (w, x, y, z)."""
    mean: Sequence[float] = (0.0, 0.0, 0.0)
    scale: Sequence[float] = (1.0, 1.0, 1.0)
    rotation: Sequence[float] = (1.0, 0.0, 0.0, 0.0)
    opacity: float = 1.0
    sh_dc: Sequence[float] = (0.0, 0.0, 0.0)
    sh_rest: Optional[Sequence[float]] = None

    def record(self) -> np.ndarray:
        r = [*self.mean, *self.scale, *self.rotation, self.opacity, *self.sh_dc]
        if self.sh_rest is not None:
            if len(self.sh_rest) != kShRestCoeffs:
                raise ValidationError("Gaussian3D.sh_rest must hold 45 coefficients")
            r += list(self.sh_rest)
        return np.asarray(r, dtype=np.float32)


class Scene:
    """(n, 14) or (n, 59) float32 records in .gsb order: mean3 scale3 quat4(w,x,y,z) opacity
    sh_dc3 [sh_rest45]."""

    def __init__(self, records: np.ndarray):
        records = np.ascontiguousarray(records, dtype=np.float32)
        if records.ndim != 2 or records.shape[1] not in (14, 59):
            raise FormatError("scene records must have shape (n, 14) or (n, 59)")
        self.records = records

    @property
    def sh_degree(self) -> int:
        return 3 if self.records.shape[1] == 59 else 0

    def __len__(self) -> int:
        return len(self.records)

    @staticmethod
    def from_gaussians(gs: Iterable[Gaussian3D]) -> "Scene":
        gs = list(gs)
        if not gs:
            return Scene(np.zeros((0, 14), np.float32))
        # eval_sh_color (projection.cpp:55-77) takes sh_rest per Gaussian; a scene where only some
        # Gaussians carry it becomes degree 3 with zero coefficients for the others (+-0 terms:
        # their colours are bit-identical).  save_scene keeps the reference's mixed-presence error.
        recs = [g.record() for g in gs]
        if any(len(r) == 59 for r in recs):
            recs = [r if len(r) == 59 else list(r) + [0.0] * kShRestCoeffs for r in recs]
        return Scene(np.stack([np.asarray(r, np.float32) for r in recs]))

    def gaussian(self, i: int) -> Gaussian3D:
        r = self.records[i]
        return Gaussian3D(tuple(r[0:3]), tuple(r[3:6]), tuple(r[6:10]), float(r[10]),
                          tuple(r[11:14]), tuple(r[14:59]) if self.sh_degree == 3 else None)


def as_scene(scene) -> Scene:
    if isinstance(scene, Scene):
        return scene
    if isinstance(scene, np.ndarray):
        return Scene(scene)
    return Scene.from_gaussians(scene)


@dataclass
class Camera:
    """Pinhole camera, row-major 4x4 world->camera view (types.hpp:36-49)."""
    view: np.ndarray = field(default_factory=lambda: np.eye(4, dtype=np.float32))
    focal_x: float = 0.0
    focal_y: float = 0.0
    width: int = 0
    height: int = 0
    near: float = 0.0
    far: float = 0.0

    def rotation(self) -> np.ndarray:
        return np.asarray(self.view, np.float32)[:3, :3]

    def translation(self) -> np.ndarray:
        return np.asarray(self.view, np.float32)[:3, 3]

    def position(self) -> np.ndarray:
        return -(self.rotation().T @ self.translation())

    def to_c(self) -> _lib.tgs_camera:
        c = _lib.tgs_camera()
        v = np.asarray(self.view, dtype=np.float32).reshape(4, 4)
        for i in range(16):
            c.view[i] = float(v.flat[i])
        c.focal_x, c.focal_y = float(self.focal_x), float(self.focal_y)
        c.width, c.height = int(self.width), int(self.height)
        c.near, c.far = float(self.near), float(self.far)
        return c


def make_camera(width: int, height: int, focal_scale: float = 0.75) -> Camera:
    """Canonical camera of the reference tests (testutil.hpp:14-24)."""
    return Camera(np.eye(4, dtype=np.float32), focal_scale * width, focal_scale * width, width, height,
                  0.2, 100.0)


def orbit_cameras(n: int, width: int, height: int, center=(0.0, 0.0, 3.0), distance: float = 3.0,
                  focal_scale: float = 0.75):
    """Config-5 camera batch: k = 0..n-1 orbiting `center` at `distance`,
    yaw = -20 + 40 k/(n-1) deg, pitch = 10 sin(2 pi k / n) deg, view = [R | -R c]."""
    cams = []
    c0 = np.asarray(center, dtype=np.float64)
    for k in range(n):
        yaw = math.radians(-20.0 + 40.0 * k / max(n - 1, 1))
        pitch = math.radians(10.0 * math.sin(2.0 * math.pi * k / n))
        # camera looks at the centre from centre - distance * forward
        fwd = np.array([math.sin(yaw) * math.cos(pitch), math.sin(pitch), math.cos(yaw) * math.cos(pitch)])
        eye = c0 - distance * fwd
        z = fwd / np.linalg.norm(fwd)
        up = np.array([0.0, 1.0, 0.0])
        x = np.cross(up, z)
        x /= np.linalg.norm(x)
        y = np.cross(z, x)
        R = np.stack([x, y, z]).astype(np.float32)
        view = np.eye(4, dtype=np.float32)
        view[:3, :3] = R
        view[:3, 3] = (-(R.astype(np.float64) @ eye)).astype(np.float32)
        cams.append(Camera(view, focal_scale * width, focal_scale * width, width, height, 0.2, 100.0))
    return cams


class ImageBuffer:
    """Row-major RGB float image, values in [0,1] after render (types.hpp:52-69)."""

    def __init__(self, width: int = 0, height: int = 0, rgb: Optional[np.ndarray] = None):
        self.width, self.height = int(width), int(height)
        self.rgb = rgb if rgb is not None else np.zeros((height, width, 3), np.float32)

    def pixel(self, x: int, y: int) -> np.ndarray:
        return self.rgb[y, x]

    def finalize(self):
        np.clip(self.rgb, 0.0, 1.0, out=self.rgb)


class Backend(enum.IntEnum):
    scalar = 0
    tensor = 1


class PrecisionMode(enum.IntEnum):
    fp32 = 0
    fp16 = 1


@dataclass
class RasterConstants:
    alpha_skip: float = 1.0 / 255.0
    alpha_clamp: float = 0.99
    t_terminate: float = 1e-4


@dataclass
class RenderOptions:
    backend: Backend = Backend.tensor
    mode: PrecisionMode = PrecisionMode.fp32
    group_size: int = 2
    workers: int = 1
    chunk_len: int = 16
    constants: RasterConstants = field(default_factory=RasterConstants)

    def to_c(self) -> _lib.tgs_options:
        o = _lib.tgs_options()
        o.backend, o.mode, o.group_size = int(self.backend), int(self.mode), int(self.group_size)
        o.workers, o.chunk_len = int(self.workers), int(self.chunk_len)
        o.alpha_skip = np.float32(self.constants.alpha_skip)
        o.alpha_clamp = np.float32(self.constants.alpha_clamp)
        o.t_terminate = np.float32(self.constants.t_terminate)
        return o


@dataclass
class ProjectionStats:
    input: int = 0
    culled: int = 0
    dropped_degenerate: int = 0


@dataclass
class RenderResult:
    image: ImageBuffer
    projection: ProjectionStats
    entries: int = 0           # group-level entries (N_group)
    tile_appearances: int = 0  # tile-level appearances (N_total)
    stage_ms: dict = field(default_factory=dict)
    ops: "OpReport" = None     # OpReport (metrics.hpp:49-69) of the tensor rasteriser


@dataclass
class OpReport:
    """OpReport (metrics.hpp:49-69) in the reference's units (include/tgs.h tgs_stats)."""
    fragment_ops: int = 0
    chunk_loads: int = 0
    skipped_pairs: int = 0
    used_lanes: int = 0
    total_lanes: int = 0

    def padding_waste(self) -> float:
        return 1.0 - self.used_lanes / self.total_lanes if self.total_lanes else 0.0


PROJ_DTYPE = np.dtype([("mean2d", "<f4", 2), ("conic", "<f4", 3), ("color", "<f4", 3),
                       ("opacity", "<f4"), ("depth", "<f4"), ("radius", "<i4")])
ENTRY_DTYPE = np.dtype([("gaussian_index", "<u4"), ("depth", "<f4"), ("mask", "<u4")])


# --------------------------------------------------------------------------------------------
# device context / scenes
# --------------------------------------------------------------------------------------------
class Context:
    """One CUDA device + stream (tgs_ctx)."""

    def __init__(self, device: int = 0):
        self.lib = _lib.load()
        h = C.c_void_p()
        _check(self.lib.tgs_ctx_create(int(device), C.byref(h)))
        self.h = h
        self.device = device

    def close(self):
        if self.h:
            self.lib.tgs_ctx_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def set_exact_emulation(self, on: bool) -> None:
        """Route fp32 frames through the exact-emulation rasteriser (bit-exact with the reference
        CPU build; PrecisionMode.fp16 always uses it)."""
        _check(self.lib.tgs_set_exact_emulation(self.h, int(bool(on))))

    def set_graphs(self, on: bool) -> None:
        """CUDA-graph capture/replay of the per-frame launches (tgs_set_graphs, default on)."""
        _check(self.lib.tgs_set_graphs(self.h, int(bool(on))))

    def set_tile_cull(self, on: bool) -> None:
        """Rasteriser tile cull by the alpha_skip ellipse box (default on; images identical)."""
        _check(self.lib.tgs_set_tile_cull(self.h, 1 if on else 0))

    @property
    def stream(self) -> int:
        return int(self.lib.tgs_ctx_stream(self.h) or 0)

    def upload(self, scene) -> "DeviceScene":
        return DeviceScene(self, as_scene(scene))

    # -- single frame --------------------------------------------------------------------------
    def render(self, dscene: "DeviceScene", cam: Camera, opt: RenderOptions = None,
               out: Optional[np.ndarray] = None) -> RenderResult:
        opt = opt or RenderOptions()
        img = out if out is not None else np.empty((cam.height, cam.width, 3), np.float32)
        st = _lib.tgs_stats()
        _check(self.lib.tgs_render(self.h, dscene.h, C.byref(cam.to_c()), C.byref(opt.to_c()),
                                   img.ctypes.data_as(_lib.F32P), C.byref(st)))
        return _result(img, cam, st)

    def render_band(self, dscene, cam: Camera, opt: RenderOptions, row0: int, row1: int, copy: bool = True):
        """Group rows [row0, row1) of the frame; copy=False leaves the band image on the device
        (image_device_ptr) and returns (None, stats)."""
        g = opt.group_size
        y0 = row0 * g * kTileSize
        y1 = min(cam.height, row1 * g * kTileSize)
        img = np.empty((y1 - y0, cam.width, 3), np.float32) if copy else None
        st = _lib.tgs_stats()
        _check(self.lib.tgs_render_band(self.h, dscene.h, C.byref(cam.to_c()), C.byref(opt.to_c()),
                                        int(row0), int(row1), img.ctypes.data_as(_lib.F32P) if copy else None,
                                        C.byref(st)))
        return img, st

    def group_row_entries(self, dscene, cam: Camera, opt: RenderOptions) -> np.ndarray:
        """Entries per group row of the frame (screen-band work estimate, tgs_group_row_entries)."""
        n = C.c_int64()
        _check(self.lib.tgs_group_row_entries(self.h, dscene.h, C.byref(cam.to_c()), C.byref(opt.to_c()), None, 0,
                                              C.byref(n)))
        out = np.zeros(max(n.value, 1), np.uint64)
        _check(self.lib.tgs_group_row_entries(self.h, dscene.h, C.byref(cam.to_c()), C.byref(opt.to_c()),
                                              out.ctypes.data, n.value, C.byref(n)))
        return out[:n.value]

    def render_batch(self, dscene, cams: Sequence[Camera], opt: RenderOptions,
                     out: Optional[np.ndarray] = None):
        n = len(cams)
        arr = (_lib.tgs_camera * n)(*[c.to_c() for c in cams])
        if out is None and n:
            out = np.empty((n, cams[0].height, cams[0].width, 3), np.float32)
        st = _lib.tgs_stats()
        _check(self.lib.tgs_render_batch(self.h, dscene.h, arr, n, C.byref(opt.to_c()),
                                         out.ctypes.data_as(_lib.F32P) if n else None, C.byref(st)))
        return out, st

    # -- async (benchmark) ------------------------------------------------------------------------
    def enqueue(self, dscene, cam: Camera, opt: RenderOptions):
        _check(self.lib.tgs_render_enqueue(self.h, dscene.h, C.byref(cam.to_c()), C.byref(opt.to_c())))

    def sync(self) -> _lib.tgs_stats:
        st = _lib.tgs_stats()
        _check(self.lib.tgs_sync(self.h, C.byref(st)))
        return st

    def image_device_ptr(self) -> int:
        return int(self.lib.tgs_image_device(self.h) or 0)

    # -- readback of the last frame -----------------------------------------------------------
    def read_projected(self) -> np.ndarray:
        n = C.c_int64()
        _check(self.lib.tgs_read_projected(self.h, None, 0, C.byref(n)))
        out = np.zeros(max(n.value, 1), PROJ_DTYPE)
        _check(self.lib.tgs_read_projected(self.h, out.ctypes.data, n.value, C.byref(n)))
        return out[:n.value]

    def read_lists(self, n_groups: int):
        n = C.c_int64()
        _check(self.lib.tgs_read_lists(self.h, None, 0, None, 0, C.byref(n)))
        ent = np.zeros(max(n.value, 1), ENTRY_DTYPE)
        off = np.zeros(n_groups + 1, np.uint32)
        _check(self.lib.tgs_read_lists(self.h, ent.ctypes.data, n.value, off.ctypes.data, len(off),
                                       C.byref(n)))
        return ent[:n.value], off

    def count_pairs(self):
        w, b = C.c_uint64(), C.c_uint64()
        _check(self.lib.tgs_count_pairs(self.h, C.byref(w), C.byref(b)))
        return int(w.value), int(b.value)

    def reuse_report(self) -> dict:
        """ReuseReport of the last frame (reference load_reduction, metrics.cpp:45-57)."""
        ng, nt, lr = C.c_uint64(), C.c_uint64(), C.c_double()
        hist = (C.c_uint64 * 17)()
        _check(self.lib.tgs_reuse_report(self.h, C.byref(ng), C.byref(nt), C.byref(lr), hist))
        return {"n_group": int(ng.value), "n_total": int(nt.value), "load_reduction": float(lr.value),
                "mask_popcount_hist": [int(v) for v in hist]}

    def encode_u8(self, img_device_ptr: int, n: int) -> np.ndarray:
        out = np.empty(n, np.uint8)
        _check(self.lib.tgs_encode_u8(self.h, C.c_void_p(img_device_ptr), n, out.ctypes.data))
        return out


class DeviceScene:
    def __init__(self, ctx: Context, scene: Scene):
        self.ctx = ctx
        self.n = len(scene)
        h = C.c_void_p()
        _check(ctx.lib.tgs_scene_upload(ctx.h, scene.records.ctypes.data_as(_lib.F32P), len(scene),
                                        scene.sh_degree, C.byref(h)))
        self.h = h

    def free(self):
        if self.h:
            self.ctx.lib.tgs_scene_free(self.h)
            self.h = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


_DEFAULT = {}


def default_context(device: int = 0) -> Context:
    if device not in _DEFAULT:
        _DEFAULT[device] = Context(device)
    return _DEFAULT[device]


def _result(img: np.ndarray, cam: Camera, st: _lib.tgs_stats) -> RenderResult:
    return RenderResult(
        ImageBuffer(cam.width, img.shape[0], img),
        ProjectionStats(int(st.input), int(st.culled), int(st.dropped_degenerate)),
        int(st.entries), int(st.tile_appearances),
        {"preprocess": st.ms_preprocess, "binning": st.ms_binning, "sort": st.ms_sort,
         "raster": st.ms_raster, "total": st.ms_total},
        OpReport(int(st.fragment_ops), int(st.chunk_loads), int(st.skipped_pairs), int(st.used_lanes),
                 int(st.total_lanes)))


# --------------------------------------------------------------------------------------------
# reference-shaped entry points
# --------------------------------------------------------------------------------------------
def render(scene, cam: Camera, opt: RenderOptions = None, device: int = 0) -> RenderResult:
    """gsr::render (render.hpp:30-31): project -> bin -> sort -> rasterise, all on the GPU.
    Host scene in, host image out (the scene is uploaded per call, like the reference's
    by-value API; use Context.upload for persistent scenes)."""
    opt = opt or RenderOptions()
    sc = as_scene(scene)
    ctx = default_context(device)
    img = np.empty((cam.height, cam.width, 3), np.float32) if cam.width > 0 and cam.height > 0 \
        else np.empty((0,), np.float32)
    st = _lib.tgs_stats()
    rec = sc.records if len(sc) else np.zeros((1, 14), np.float32)
    _check(ctx.lib.tgs_render_records(ctx.h, rec.ctypes.data_as(_lib.F32P), len(sc), sc.sh_degree,
                                      C.byref(cam.to_c()), C.byref(opt.to_c()),
                                      img.ctypes.data_as(_lib.F32P), C.byref(st)))
    return _result(img, cam, st)


def project_scene(scene, cam: Camera, workers: int = 1, stats: Optional[ProjectionStats] = None,
                  device: int = 0) -> np.ndarray:
    """project_scene (projection.hpp:48-50) on the GPU (tgs_project_scene): ProjectedGaussian
    records (PROJ_DTYPE) in input order.  ValidationError for non-positive scales
    (projection.cpp:37); workers is validated and ignored, like every launch-config knob here."""
    if workers < 1:
        raise ValidationError("project_scene: workers must be >= 1")
    sc = as_scene(scene)
    ctx = default_context(device)
    rec = sc.records if len(sc) else np.zeros((1, 14), np.float32)
    n = C.c_int64()
    st = _lib.tgs_stats()
    _check(ctx.lib.tgs_project_scene(ctx.h, rec.ctypes.data_as(_lib.F32P), len(sc), sc.sh_degree,
                                     C.byref(cam.to_c()), None, 0, C.byref(n), C.byref(st)))
    out = np.zeros(max(n.value, 1), PROJ_DTYPE)
    _check(ctx.lib.tgs_read_projected(ctx.h, out.ctypes.data, n.value, C.byref(n)))
    if stats is not None:
        stats.input, stats.culled, stats.dropped_degenerate = int(st.input), int(st.culled), \
            int(st.dropped_degenerate)
    return out[:n.value]


@dataclass
class GroupConfig:
    """GroupConfig (binning.hpp:15-31): group_h x group_w blocks of 16x16 tiles."""
    group_h: int = 2
    group_w: int = 2
    image_width: int = 0
    image_height: int = 0

    @staticmethod
    def square(g: int, image_width: int, image_height: int) -> "GroupConfig":
        cfg = GroupConfig(g, g, image_width, image_height)
        cfg.validate()
        return cfg

    def tiles_x(self) -> int:
        return (self.image_width + kTileSize - 1) // kTileSize

    def tiles_y(self) -> int:
        return (self.image_height + kTileSize - 1) // kTileSize

    def groups_x(self) -> int:
        return (self.tiles_x() + self.group_w - 1) // self.group_w

    def groups_y(self) -> int:
        return (self.tiles_y() + self.group_h - 1) // self.group_h

    def group_count(self) -> int:
        return self.groups_x() * self.groups_y()

    def validate(self) -> None:  # binning.cpp:22-30
        if self.image_width <= 0 or self.image_height <= 0:
            raise ValidationError("GroupConfig: image dimensions must be positive")
        if not (self.group_h == self.group_w and self.group_h in (1, 2, 4)):
            raise ValidationError("GroupConfig: supported group sizes are 1x1, 2x2, 4x4")


KEYED_DTYPE = np.dtype([("group_id", "<u4"), ("entry", ENTRY_DTYPE)])


@dataclass
class SortedGroupLists:
    """SortedGroupLists (binning.hpp:53-59): (group, depth)-sorted entries + group offsets."""
    entries: np.ndarray  # ENTRY_DTYPE
    offsets: np.ndarray  # uint32, group_count + 1

    def group_begin(self, g: int) -> int:
        return int(self.offsets[g])

    def group_end(self, g: int) -> int:
        return int(self.offsets[g + 1])


@dataclass
class TensorRasterOptions:
    """TensorRasterOptions (raster_tensor.hpp:45-50)."""
    constants: RasterConstants = field(default_factory=RasterConstants)
    mode: PrecisionMode = PrecisionMode.fp32
    chunk_len: int = 16
    workers: int = 1


def _proj_array(projected) -> np.ndarray:
    p = np.ascontiguousarray(projected, dtype=PROJ_DTYPE)
    return p if len(p) else np.zeros(1, PROJ_DTYPE)


def build_group_entries(projected, cfg: GroupConfig, device: int = 0) -> np.ndarray:
    """build_group_entries (binning.hpp:68-69) on the GPU: KEYED_DTYPE entries in splat order,
    then group id (gy outer, gx inner)."""
    cfg.validate()
    n = len(projected)
    p = _proj_array(projected)
    ctx = default_context(device)
    m = C.c_int64()
    _check(ctx.lib.tgs_build_group_entries(ctx.h, p.ctypes.data, n, cfg.image_width, cfg.image_height,
                                           cfg.group_h, None, 0, C.byref(m)))
    out = np.zeros(max(m.value, 1), KEYED_DTYPE)
    if m.value:
        _check(ctx.lib.tgs_build_group_entries(ctx.h, p.ctypes.data, n, cfg.image_width, cfg.image_height,
                                               cfg.group_h, out.ctypes.data, m.value, C.byref(m)))
    return out[:m.value]


def sort_entries(entries, cfg: GroupConfig, device: int = 0) -> SortedGroupLists:
    """sort_entries (binning.hpp:72-73) on the GPU: stable (group_id << 32 | depth bits) order;
    ValidationError for a non-finite or negative depth (binning.cpp:78-83)."""
    cfg.validate()
    e = np.ascontiguousarray(entries, dtype=KEYED_DTYPE)
    n = len(e)
    ctx = default_context(device)
    out = np.zeros(max(n, 1), ENTRY_DTYPE)
    off = np.zeros(cfg.group_count() + 1, np.uint32)
    ebuf = e if n else np.zeros(1, KEYED_DTYPE)
    _check(ctx.lib.tgs_sort_entries(ctx.h, ebuf.ctypes.data, n, cfg.image_width, cfg.image_height, cfg.group_h,
                                    out.ctypes.data, off.ctypes.data, len(off)))
    return SortedGroupLists(out[:n], off)


def _rasterize(lists: SortedGroupLists, projected, cfg: GroupConfig, backend: Backend, constants: RasterConstants,
               mode: PrecisionMode, workers: int, chunk_len: int, device: int) -> ImageBuffer:
    cfg.validate()
    opt = RenderOptions(backend, mode, cfg.group_h, workers, chunk_len, constants)
    ent = np.ascontiguousarray(lists.entries, dtype=ENTRY_DTYPE)
    off = np.ascontiguousarray(lists.offsets, dtype=np.uint32)
    p = _proj_array(projected)
    img = np.empty((cfg.image_height, cfg.image_width, 3), np.float32)
    ebuf = ent if len(ent) else np.zeros(1, ENTRY_DTYPE)
    ctx = default_context(device)
    _check(ctx.lib.tgs_rasterize_lists(ctx.h, ebuf.ctypes.data, len(ent), off.ctypes.data, len(off), p.ctypes.data,
                                       len(projected), cfg.image_width, cfg.image_height, C.byref(opt.to_c()),
                                       img.ctypes.data_as(_lib.F32P)))
    return ImageBuffer(cfg.image_width, cfg.image_height, img)


def rasterize_tiles_scalar(lists: SortedGroupLists, projected, cfg: GroupConfig, k: RasterConstants = None,
                           mode: PrecisionMode = PrecisionMode.fp32, workers: int = 1, device: int = 0) -> ImageBuffer:
    """rasterize_tiles_scalar (raster_scalar.hpp:59-62): the CUDA-core baseline kernel on caller
    lists (1x1 groups required, raster_scalar.cpp:56-57)."""
    return _rasterize(lists, projected, cfg, Backend.scalar, k or RasterConstants(), mode, workers, 16, device)


def rasterize_groups_tensor(lists: SortedGroupLists, projected, cfg: GroupConfig,
                            opt: TensorRasterOptions = None, device: int = 0) -> ImageBuffer:
    """rasterize_groups_tensor (raster_tensor.hpp:62-65): the tcgen05 grouped kernel on caller lists."""
    opt = opt or TensorRasterOptions()
    return _rasterize(lists, projected, cfg, Backend.tensor, opt.constants, opt.mode, opt.workers, opt.chunk_len,
                      device)


def sorted_group_lists(scene, cam: Camera, group_size: int, device: int = 0):
    """The render path's own (fused) bin + sort of a frame, read back: (entries[GroupEntry],
    offsets[group_count + 1], projected) — equal to sort_entries(build_group_entries(...))."""
    ctx = default_context(device)
    ds = ctx.upload(scene)
    opt = RenderOptions(Backend.scalar if group_size == 1 else Backend.tensor, group_size=group_size)
    ctx.render(ds, cam, opt)
    tx, ty = -(-cam.width // kTileSize), -(-cam.height // kTileSize)
    ng = (-(-tx // group_size)) * (-(-ty // group_size))
    ent, off = ctx.read_lists(ng)
    return ent, off, ctx.read_projected()


def gen_synthetic_scene(seed: int, count: int, extent: float = 1.0, scale_range=(0.01, 0.05),
                        sh_seed: int = 0) -> Scene:
    """gen_synthetic_scene (scene_io.cpp:218-251), host code in libtgs; sh_seed != 0 adds
    SplitMix64(sh_seed) U[-1,1] sh_rest coefficients (degree 3)."""
    lib = _lib.load()
    rf = 59 if sh_seed else 14
    out = np.zeros((max(count, 0), rf), np.float32)
    buf = out if count > 0 else np.zeros((1, rf), np.float32)
    _check(lib.tgs_gen_synthetic_scene(int(seed), int(count), float(extent), float(scale_range[0]),
                                       float(scale_range[1]), int(sh_seed), buf.ctypes.data_as(_lib.F32P)))
    return Scene(out)


# --------------------------------------------------------------------------------------------
# metrics (metrics.hpp) — host-side, used by tests and the CLI-style tooling
# --------------------------------------------------------------------------------------------
def psnr(a, b) -> float:
    a = a.rgb if isinstance(a, ImageBuffer) else a
    b = b.rgb if isinstance(b, ImageBuffer) else b
    if a.shape != b.shape:
        raise ValidationError("psnr: image dimensions differ")
    se = float(np.sum((a.astype(np.float64) - b.astype(np.float64)) ** 2))
    if se == 0.0:
        return kPsnrCap
    return 10.0 * math.log10(1.0 / (se / a.size))


def max_abs_diff(a, b) -> float:
    a = a.rgb if isinstance(a, ImageBuffer) else a
    b = b.rgb if isinstance(b, ImageBuffer) else b
    if a.shape != b.shape:
        raise ValidationError("max_abs_diff: image dimensions differ")
    return float(np.max(np.abs(a - b))) if a.size else 0.0


_GSB_MAGIC = b"GSB1"
_GSB_HEADER = 16


def save_scene(scene, path: str) -> None:
    """save_scene (scene_io.cpp:103-136): 16-byte header (magic "GSB1", u32 count, u32 sh_degree,
    u32 reserved 0) then little-endian float32 records (14, or 59 with sh_rest)."""
    if not isinstance(scene, (Scene, np.ndarray)):
        scene = list(scene)
        have = [g.sh_rest is not None for g in scene]
        if any(have) and not all(have):  # save_scene, scene_io.cpp:103-109
            raise ValidationError("save_scene: mixed sh_rest presence across records")
    sc = as_scene(scene)
    deg = sc.sh_degree if len(sc) else 0
    head = _GSB_MAGIC + np.array([len(sc), deg, 0], dtype="<u4").tobytes()
    try:
        with open(path, "wb") as f:
            f.write(head)
            f.write(np.ascontiguousarray(sc.records, dtype="<f4").tobytes())
    except OSError:
        raise FormatError("cannot open for writing: " + path)


def load_scene(path: str) -> Scene:
    """load_scene (scene_io.cpp:43-101): the reference's header and payload checks (FormatError),
    per-record validation in record order (ValidationError: opacity in [0,1], finite mean/scale,
    positive scale, finite non-zero quaternion norm) and its renormalisation of quaternions whose
    float32 norm (Eigen coefficient order x, y, z, w, packet sum (x2+z2)+(y2+w2)) drifts from 1 by
    more than 1e-6."""
    try:
        with open(path, "rb") as f:
            data = f.read()
    except OSError:
        raise FormatError("cannot open scene file: " + path)
    if len(data) < _GSB_HEADER:
        raise FormatError(f"{path}: truncated header at byte offset {len(data)} (need 16)")
    if data[:4] != _GSB_MAGIC:
        raise FormatError(f"{path}: bad magic at byte offset 0")
    count, degree = (int(v) for v in np.frombuffer(data, dtype="<u4", count=2, offset=4))
    if degree not in (0, 3):
        raise FormatError(f"{path}: unsupported sh_degree at byte offset 8")
    rf = 59 if degree == 3 else 14
    need = _GSB_HEADER + count * rf * 4
    if len(data) < need:
        raise FormatError(f"{path}: truncated payload at byte offset {len(data)} (need {need})")
    rec = np.frombuffer(data, dtype="<f4", count=count * rf, offset=_GSB_HEADER).reshape(count, rf)
    rec = rec.astype(np.float32, copy=True)
    if count:
        with np.errstate(invalid="ignore", over="ignore"):
            op = rec[:, 10]
            bad_op = ~((op >= 0.0) & (op <= 1.0))
            bad_fin = ~np.isfinite(rec[:, 0:6]).all(axis=1)
            bad_scale = ~(rec[:, 3:6].min(axis=1) > 0.0)
            x, y, z, w = rec[:, 7], rec[:, 8], rec[:, 9], rec[:, 6]
            n = np.sqrt((x * x + z * z) + (y * y + w * w), dtype=np.float32)
            bad_q = ~((n > 0.0) & np.isfinite(n))
        bad = bad_op | bad_fin | bad_scale | bad_q
        if bad.any():
            i = int(np.argmax(bad))
            if bad_op[i]:
                raise ValidationError(f"{path}: scene record {i}: opacity outside [0,1]")
            if bad_fin[i]:
                raise ValidationError(f"{path}: scene record {i}: non-finite mean or scale")
            if bad_scale[i]:
                raise ValidationError(f"{path}: scene record {i}: non-positive scale")
            raise ValidationError(f"scene record {i}: quaternion has non-finite or zero norm")
        drift = np.abs(n - np.float32(1.0)) > np.float32(1e-6)
        if drift.any():
            rec[drift, 6:10] = rec[drift, 6:10] / n[drift, None]
    return Scene(rec)


def encode_ppm(img) -> bytes:
    """encode_ppm (scene_io.cpp:253-263): P6 header + lrintf(clamp(v)*255) bytes."""
    rgb = img.rgb if isinstance(img, ImageBuffer) else img
    h, w = rgb.shape[:2]
    c = np.clip(rgb.astype(np.float32), 0.0, 1.0) * np.float32(255.0)
    payload = np.rint(c.astype(np.float32)).astype(np.uint8)  # rint = round half to even
    return f"P6\n{w} {h}\n255\n".encode() + payload.tobytes()
