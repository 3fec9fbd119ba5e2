"""The C++ drop-in (cpp/gsr_b200.hpp): a program written against the reference's gsr::render API,
compiled against this header and linked with libtgs.so.

CPU: the drop-in and a reference-API driver compile (g++ -std=c++20, the caller's Eigen — here the
oracle's Eigen-subset headers stand in for the user's Eigen install) and link against libtgs.
GPU: the driver renders through gsr::render and gsr::b200::DeviceScene; the image matches the
oracle within the parity tolerance and the RenderResult counters equal the reference's
(render.hpp:19-25); invalid options raise ValidationError (render.cpp:9-11) -> exit code 2 like the
reference CLI (tools/gsrender.cpp:237-240).
"""
import os
import subprocess

import numpy as np
import pytest

from tests.cases import make_camera, rotated_camera

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
BIN = os.path.join(ROOT, "tests", "cpp", "_build", "dropin")


def build_driver() -> str:
    from paper_2605_17855_b200 import build as b
    b.build()
    os.makedirs(os.path.dirname(BIN), exist_ok=True)
    cmd = ["g++", "-std=c++20", "-O2", "-ffp-contract=off", "-I", os.path.join(ROOT, "oracle", "eigen_min"),
           "-I", os.path.join(ROOT, "cpp"), os.path.join(ROOT, "cpp", "gsr_b200.cpp"),
           os.path.join(ROOT, "tests", "cpp", "dropin_main.cpp"), "-L", os.path.dirname(b.LIB), "-ltgs",
           f"-Wl,-rpath,{os.path.dirname(b.LIB)}", "-o", BIN]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    return BIN


def test_dropin_compiles_against_reference_api():
    assert os.path.exists(build_driver())


def _run(tmp_path, rec, cam, backend, group):
    deg = 3 if rec.shape[1] == 59 else 0
    rp, cp, op = tmp_path / "rec.f32", tmp_path / "cam.f32", tmp_path / "out.f32"
    np.ascontiguousarray(rec, np.float32).tofile(rp)
    cv = np.concatenate([np.asarray(cam.view, np.float32).reshape(16),
                         np.asarray([cam.focal_x, cam.focal_y, cam.width, cam.height, cam.near, cam.far],
                                    np.float32)])
    cv.tofile(cp)
    r = subprocess.run([BIN, str(rp), str(len(rec)), str(deg), str(cp), str(backend), str(group), str(op)],
                       capture_output=True, text=True, timeout=300)
    if r.returncode != 0:
        return r.returncode, r.stderr, None, None
    raw = np.fromfile(op, np.uint8)
    npx = cam.width * cam.height * 3
    img = np.frombuffer(raw[:npx * 4].tobytes(), np.float32).reshape(cam.height, cam.width, 3)
    counters = np.frombuffer(raw[npx * 4:].tobytes(), np.float64).astype(np.int64)
    return 0, "", img, counters


@pytest.mark.gpu
def test_dropin_render_matches_oracle(port, tmp_path):
    from tests.test_gpu_parity import check_image
    build_driver()
    for seed, n, sh, cam in [(41, 3000, 5, make_camera(200, 144)), (42, 2000, 0, rotated_camera(160, 120))]:
        rec = port.gen_scene(seed, n, 1.0, 0.01, 0.08, sh)
        for backend, group in ((1, 2), (0, 1)):
            rc, err, img, counters = _run(tmp_path, rec, cam, backend, group)
            assert rc == 0, err
            ref_img, st = port.render(rec, cam, backend=backend, group_size=group)
            check_image(img, ref_img, f"drop-in seed {seed} b{backend} g{group}")
            assert counters.tolist() == [st["input"], st["culled"], st["dropped_degenerate"], st["entries"],
                                         st["tile_appearances"]]


@pytest.mark.gpu
def test_dropin_validation_error_exit_code(port, tmp_path):
    build_driver()
    rec = port.gen_scene(43, 100, 1.0, 0.01, 0.08, 0)
    rc, err, _, _ = _run(tmp_path, rec, make_camera(64, 64), 0, 2)  # scalar backend with G=2
    assert rc == 2 and "validation" in err


STAGE_BIN = os.path.join(ROOT, "tests", "cpp", "_build", "stage")


def build_stage_driver() -> str:
    from paper_2605_17855_b200 import build as b
    b.build()
    os.makedirs(os.path.dirname(STAGE_BIN), exist_ok=True)
    cmd = ["g++", "-std=c++20", "-O2", "-ffp-contract=off", "-I", os.path.join(ROOT, "oracle", "eigen_min"),
           "-I", os.path.join(ROOT, "cpp"), os.path.join(ROOT, "cpp", "gsr_b200.cpp"),
           os.path.join(ROOT, "tests", "cpp", "stage_main.cpp"), "-L", os.path.dirname(b.LIB), "-ltgs",
           f"-Wl,-rpath,{os.path.dirname(b.LIB)}", "-o", STAGE_BIN]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    return STAGE_BIN


def test_stage_api_driver_compiles_against_reference_api():
    """project_scene / build_group_entries / sort_entries / rasterize_* with the reference's
    declarations (projection.hpp:48-50, binning.hpp:68-73, raster_scalar.hpp:59-62,
    raster_tensor.hpp:62-65) compile against cpp/gsr_b200.hpp."""
    assert os.path.exists(build_stage_driver())


@pytest.mark.gpu
def test_stage_api_driver_matches_oracle(port, tmp_path):
    from oracle.oracle import PROJ_DTYPE, ENTRY_DTYPE
    from tests.test_gpu_parity import check_image
    build_stage_driver()
    for seed, n, sh, cam in [(51, 3000, 5, make_camera(200, 144)), (52, 2000, 0, rotated_camera(160, 120))]:
        rec = port.gen_scene(seed, n, 1.0, 0.01, 0.08, sh)
        proj_ref, _ = port.project(rec, cam)
        for backend, group in ((1, 2), (0, 1), (1, 4)):
            rp, cp, op = tmp_path / "rec.f32", tmp_path / "cam.f32", tmp_path / "out.bin"
            np.ascontiguousarray(rec, np.float32).tofile(rp)
            cv = np.concatenate([np.asarray(cam.view, np.float32).reshape(16),
                                 np.asarray([cam.focal_x, cam.focal_y, cam.width, cam.height, cam.near, cam.far],
                                            np.float32)])
            cv.tofile(cp)
            r = subprocess.run([STAGE_BIN, str(rp), str(len(rec)), str(3 if sh else 0), str(cp), str(backend),
                                str(group), str(op)], capture_output=True, text=True, timeout=300)
            assert r.returncode == 0, r.stderr
            raw = np.fromfile(op, np.uint8)
            o = 0
            npj = int(raw[o:o + 8].view(np.int64)[0]); o += 8
            proj = raw[o:o + 44 * npj].view(PROJ_DTYPE); o += 44 * npj
            ne = int(raw[o:o + 8].view(np.int64)[0]); o += 8
            ent = raw[o:o + 12 * ne].view(ENTRY_DTYPE); o += 12 * ne
            ent_ref, off_ref, _ = port.bin_sort(proj_ref, cam.width, cam.height, group)
            off = raw[o:o + 4 * len(off_ref)].view(np.uint32); o += 4 * len(off_ref)
            img = raw[o:].view(np.float32).reshape(cam.height, cam.width, 3)
            assert np.array_equal(proj.view(np.uint8), proj_ref.view(np.uint8))
            assert np.array_equal(off, off_ref) and np.array_equal(ent.view(np.uint8), ent_ref.view(np.uint8))
            img_ref, _ = port.rasterize(ent_ref, off_ref, proj_ref, cam.width, cam.height, backend=backend,
                                        group_size=group)
            check_image(img, img_ref, f"C++ stage API seed {seed} b{backend} g{group}")
