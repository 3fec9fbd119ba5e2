"""CPU tests of the drop-in boundary: libtgs.so builds for sm_100a, loads, exports every symbol
include/tgs.h declares with the signature table the Python mirror binds, and its host-side code
(scene generator, validation, failure without a GPU) behaves like the reference."""
import os
import re
import subprocess

import numpy as np
import pytest

from paper_2605_17855_b200 import _lib, build

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))


def _declared():
    src = open(os.path.join(ROOT, "include", "tgs.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return set(re.findall(r"\b(tgs_[a-z0-9_]+)\s*\(", src))


def test_library_builds_and_exports_header_symbols():
    path = build.build()
    assert path.endswith("libtgs.so") and os.path.exists(path)
    out = subprocess.run(["nm", "-D", "--defined-only", path], capture_output=True, text=True).stdout
    exported = set(re.findall(r"\bT (tgs_[a-z0-9_]+)$", out, flags=re.M))
    declared = _declared()
    assert declared, "no declarations parsed"
    assert declared <= exported, f"missing exports: {sorted(declared - exported)}"
    assert declared == set(_lib.SIGNATURES), "Python signature table out of sync with tgs.h"


def test_cubin_is_sm100a_with_tcgen05():
    path = build.build()
    r = subprocess.run(["cuobjdump", "-sass", path], capture_output=True, text=True)
    assert r.returncode == 0
    assert "sm_100a" in subprocess.run(["cuobjdump", "-lelf", path], capture_output=True, text=True).stdout
    sass = r.stdout
    assert "UTCHMMA" in sass or "UTCMMA" in sass, "tensor rasterizer must issue tcgen05.mma"
    assert "LDTM" in sass, "epilogue must read TMEM with tcgen05.ld"


def test_loads_and_abi_version():
    lib = _lib.load()
    assert lib.tgs_abi_version() == 2


def test_generator_matches_port(port):
    from paper_2605_17855_b200 import gsr
    for seed, n, sh in [(1, 3000, 0), (4, 500, 5), (99, 2000, 5)]:
        a = gsr.gen_synthetic_scene(seed, n, 1.0, (0.01, 0.05), sh_seed=sh).records
        b = port.gen_scene(seed, n, 1.0, 0.01, 0.05, sh)
        assert np.array_equal(a.view(np.uint32), b.view(np.uint32))


def test_generator_validation():
    from paper_2605_17855_b200 import gsr
    with pytest.raises(gsr.ValidationError):
        gsr.gen_synthetic_scene(1, -1)
    with pytest.raises(gsr.ValidationError):
        gsr.gen_synthetic_scene(1, 10, extent=0.0)
    with pytest.raises(gsr.ValidationError):
        gsr.gen_synthetic_scene(1, 10, scale_range=(0.2, 0.1))
    assert len(gsr.gen_synthetic_scene(1, 0)) == 0


def test_no_cpu_fallback_without_gpu():
    """On a machine without a B200 the product path fails loudly (no CPU fallback)."""
    from paper_2605_17855_b200 import gsr
    if os.path.exists("/dev/nvidia0"):
        pytest.skip("GPU present")
    with pytest.raises(gsr.DeviceError):
        gsr.Context(0)


def test_ppm_encoding_matches_reference(port):
    from paper_2605_17855_b200 import gsr
    rng = np.random.default_rng(0)
    img = rng.uniform(-0.2, 1.2, size=(7, 5, 3)).astype(np.float32)
    img[0, 0] = [0.5 / 255, 1.5 / 255, 254.5 / 255]  # half-way cases
    data = gsr.encode_ppm(img)
    assert data.startswith(b"P6\n5 7\n255\n")
    assert np.array_equal(np.frombuffer(data[len(b"P6\n5 7\n255\n"):], np.uint8).reshape(img.shape),
                          port.encode_ppm(img))
