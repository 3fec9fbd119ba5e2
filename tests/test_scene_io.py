"""`.gsb` scene files: gsr.load_scene / gsr.save_scene against the reference's
own load_scene / save_scene (scene_io.cpp:43-136, built in oracle/_ref): byte layout, the
quaternion renormalisation, and the FormatError / ValidationError cases with their messages."""
import os
import subprocess

import numpy as np
import pytest

from oracle.oracle import Port, Ref
from paper_2605_17855_b200 import gsr

pytestmark = pytest.mark.skipif(not Ref.available(), reason="reference build oracle/_ref not present")


@pytest.fixture(scope="module")
def ref():
    return Ref()


def _records(sh: bool, n: int = 257):
    rec = Port().gen_scene(11, n, 1.0, 0.01, 0.05, 5 if sh else 0)
    return np.ascontiguousarray(rec, np.float32)


@pytest.mark.parametrize("sh", [False, True])
def test_round_trip_and_cross_with_reference(ref, tmp_path, sh):
    rec = _records(sh)
    p_ours, p_ref = str(tmp_path / "ours.gsb"), str(tmp_path / "ref.gsb")
    gsr.save_scene(rec, p_ours)
    ref.save_scene(rec, p_ref)
    assert open(p_ours, "rb").read() == open(p_ref, "rb").read()  # identical bytes
    ours = gsr.load_scene(p_ref).records
    theirs, err = ref.load_scene(p_ours)
    assert err is None
    assert np.array_equal(ours.view(np.uint32), theirs.view(np.uint32))
    assert np.array_equal(ours.view(np.uint32), rec.view(np.uint32))


def test_quaternion_renormalisation_bitexact(ref, tmp_path):
    rec = _records(False, 64)
    rng = np.random.default_rng(3)
    rec[:, 6:10] = rng.normal(size=(64, 4)).astype(np.float32)  # far from unit norm
    rec[0, 6:10] = (1.0 + 2e-6, 0.0, 0.0, 0.0)                   # just above the 1e-6 drift bar
    rec[1, 6:10] = (1.0 + 5e-7, 0.0, 0.0, 0.0)                   # below it: kept as stored
    path = str(tmp_path / "q.gsb")
    gsr.save_scene(rec, path)
    ours = gsr.load_scene(path).records
    theirs, err = ref.load_scene(path)
    assert err is None
    assert np.array_equal(ours.view(np.uint32), theirs.view(np.uint32))
    assert ours[1, 6] == np.float32(1.0 + 5e-7)


def _expect_same_error(ref, path):
    with pytest.raises((gsr.FormatError, gsr.ValidationError)) as ei:
        gsr.load_scene(path)
    _, err = ref.load_scene(path)
    assert err is not None, "reference accepted a file we rejected"
    code, msg = err
    assert (abs(code) == 2) == isinstance(ei.value, gsr.FormatError)  # shim: -1 validation, -2 format
    assert str(ei.value) == msg


@pytest.mark.parametrize("case", ["short_header", "bad_magic", "bad_degree", "short_payload", "opacity",
                                  "nan_mean", "zero_scale", "zero_quat"])
def test_errors_match_reference(ref, tmp_path, case):
    rec = _records(False, 8)
    path = str(tmp_path / f"{case}.gsb")
    gsr.save_scene(rec, path)
    data = bytearray(open(path, "rb").read())
    if case == "short_header":
        data = data[:10]
    elif case == "bad_magic":
        data[0:4] = b"GSB2"
    elif case == "bad_degree":
        data[8:12] = np.array([2], "<u4").tobytes()
    elif case == "short_payload":
        data = data[:-5]
    else:
        r = rec.copy()
        if case == "opacity":
            r[5, 10] = 1.5
        elif case == "nan_mean":
            r[6, 1] = np.nan
        elif case == "zero_scale":
            r[3, 4] = 0.0
        elif case == "zero_quat":
            r[2, 6:10] = 0.0
        gsr.save_scene(r, path)
        data = bytearray(open(path, "rb").read())
    open(path, "wb").write(bytes(data))
    _expect_same_error(ref, path)


def test_missing_file(ref, tmp_path):
    _expect_same_error(ref, str(tmp_path / "nope.gsb"))
    assert not os.path.exists(str(tmp_path / "nope.gsb"))


# ---- the C++ drop-in's load_scene / save_scene (cpp/gsr_b200.cpp) ----------------------------------
ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
CPP_BIN = os.path.join(ROOT, "tests", "cpp", "_build", "scene_io")


@pytest.fixture(scope="module")
def cpp_driver():
    from paper_2605_17855_b200 import build as b
    b.build()
    os.makedirs(os.path.dirname(CPP_BIN), exist_ok=True)
    cmd = ["g++", "-std=c++20", "-O2", "-ffp-contract=off", "-I", os.path.join(ROOT, "oracle", "eigen_min"),
           "-I", os.path.join(ROOT, "cpp"), os.path.join(ROOT, "cpp", "gsr_b200.cpp"),
           os.path.join(ROOT, "tests", "cpp", "scene_io_main.cpp"), "-L", os.path.dirname(b.LIB), "-ltgs",
           f"-Wl,-rpath,{os.path.dirname(b.LIB)}", "-o", CPP_BIN]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    return CPP_BIN


@pytest.mark.parametrize("sh", [False, True])
def test_cpp_dropin_load_and_copy_match_reference(ref, cpp_driver, tmp_path, sh):
    rec = _records(sh, 65)
    rec[3, 6:10] = (0.5, 0.5, 0.5, 0.6)  # drifted quaternion: renormalised on load
    src, out, cpy = str(tmp_path / "s.gsb"), str(tmp_path / "o.f32"), str(tmp_path / "c.gsb")
    ref.save_scene(rec, src)
    assert subprocess.run([cpp_driver, "load", src, out]).returncode == 0
    theirs, err = ref.load_scene(src)
    assert err is None
    ours = np.fromfile(out, np.float32).reshape(theirs.shape)
    assert np.array_equal(ours.view(np.uint32), theirs.view(np.uint32))
    assert subprocess.run([cpp_driver, "copy", src, cpy]).returncode == 0
    ref_copy = str(tmp_path / "rc.gsb")
    ref.save_scene(theirs, ref_copy)
    assert open(cpy, "rb").read() == open(ref_copy, "rb").read()


def test_cpp_dropin_errors_match_reference(ref, cpp_driver, tmp_path):
    rec = _records(False, 4)
    rec[2, 10] = -0.25  # opacity outside [0,1]
    path = str(tmp_path / "bad.gsb")
    gsr.save_scene(rec, path)
    r = subprocess.run([cpp_driver, "load", path, str(tmp_path / "x.f32")], capture_output=True, text=True)
    _, err = ref.load_scene(path)
    assert r.returncode == 2 and err is not None and r.stderr.strip() == err[1]
