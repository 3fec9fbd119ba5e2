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
