"""CPU tests: the C restatement (oracle port) is pinned against the reference — bit for bit —
both through the committed golden fixtures (generated from the reference build) and, where the
reference build is present, directly on fresh seeds.  Known answers from the reference's own
unit tests are re-checked on the port."""
import numpy as np
import pytest

from oracle.oracle import ENTRY_DTYPE, PROJ_DTYPE
from tests.cases import CASES, _R, make_camera, rotated_camera


def _bits(a):
    return np.ascontiguousarray(a).view(np.uint8)


@pytest.mark.parametrize("name", list(CASES))
def test_port_matches_golden(port, golden, name):
    g = golden[name]
    case = CASES[name]
    cam = case["camera"]()
    rec = port.gen_scene(case["seed"], case["count"], 1.0, case["smin"], case["smax"], case["sh_seed"])
    assert np.array_equal(rec.view(np.uint32), g["records"].view(np.uint32))
    proj, st3 = port.project(rec, cam)
    assert np.array_equal(_bits(proj), g["projected"])
    assert np.array_equal(st3, g["proj_stats"])
    for grp in (1, 2, 4):
        ent, off, app = port.bin_sort(proj, cam.width, cam.height, grp)
        assert np.array_equal(_bits(ent), g[f"entries_g{grp}"]), grp
        assert np.array_equal(off, g[f"offsets_g{grp}"]), grp
        assert app == int(g[f"appearances_g{grp}"][0])
    for tag, opt in case["renders"].items():
        img, stats = port.render(rec, cam, **opt)
        assert np.array_equal(img.view(np.uint32), g[f"img_{tag}"].view(np.uint32)), tag
        assert [stats[k] for k in sorted(stats)] == g[f"stats_{tag}"].tolist(), tag


@pytest.mark.parametrize("seed,count,sh,rot", [(11, 3000, 0, False), (12, 1500, 7, True), (13, 2000, 0, True)])
def test_port_matches_reference_build(port, ref, seed, count, sh, rot):
    cam = rotated_camera(160, 120, yaw_deg=-23.0, pitch_deg=5.0) if rot else make_camera(160, 120)
    a = port.gen_scene(seed, count, 1.0, 0.01, 0.08, sh)
    b = ref.gen_scene(seed, count, 1.0, 0.01, 0.08, sh)
    assert np.array_equal(a.view(np.uint32), b.view(np.uint32))
    pa, sa = port.project(a, cam)
    pb, sb = ref.project(a, cam)
    assert np.array_equal(_bits(pa), _bits(pb)) and np.array_equal(sa, sb)
    for g in (1, 2, 4):
        ea, oa, xa = port.bin_sort(pa, cam.width, cam.height, g)
        eb, ob, xb = ref.bin_sort(pa, cam.width, cam.height, g)
        assert np.array_equal(_bits(ea), _bits(eb)) and np.array_equal(oa, ob) and xa == xb
    for opt in _R.values():
        ia, ta = port.render(a, cam, **opt)
        ib, tb = ref.render(a, cam, **opt)
        assert np.array_equal(ia.view(np.uint32), ib.view(np.uint32)) and ta == tb


def test_reference_render_brute_force(port):
    # acceptance.cpp:240-257 (criterion 5): low-opacity splats, tiling-free oracle == scalar path
    for seed in (17, 18, 19):
        cam = make_camera(32, 32)
        rec = port.gen_scene(seed, 32, 1.0, 0.1, 0.5, 0)
        rec[:, 10] = np.float32(0.2) + np.float32(0.13) * (rec[:, 10] - np.float32(0.2))
        proj, _ = port.project(rec, cam)
        img, _ = port.render(rec, cam, backend=0, group_size=1)
        bf = port.reference_render(proj, 32, 32)
        assert np.array_equal(img.view(np.uint32), bf.view(np.uint32))


def test_known_answers(port):
    # half.hpp known answers (test_half.cpp:16-38)
    assert port.f32_to_f16(1.0) == 0x3C00
    assert port.f32_to_f16(0.1) == 0x2E66
    assert port.f32_to_f16(65520.0) == 0x7C00
    assert port.f32_to_f16(float("nan")) == 0x7E00
    # on-axis projection (test_projection.cpp:68-84): conic 1/100.3, radius 31, mean (128,128)
    cam = make_camera(256, 256)
    cam.focal_x = cam.focal_y = 100.0
    rec = np.array([[0, 0, 10, 1, 1, 1, 1, 0, 0, 0, 0.9, 1.0, 0.5, -0.5]], np.float32)
    proj, _ = port.project(rec, cam)
    p = proj[0]
    assert p["radius"] == 31
    assert abs(p["conic"][0] - 1 / 100.3) < 1e-8 and abs(p["conic"][2] - 1 / 100.3) < 1e-8
    assert tuple(p["mean2d"]) == (128.0, 128.0) and p["depth"] == 10.0
    # single opaque splat center = 0.99 * 0.5 (test_raster_scalar.cpp:92-104)
    rec[0, 10] = 1.0
    rec[0, 11:14] = 0.0
    img, _ = port.render(rec, cam, backend=0, group_size=1)
    assert np.all(img[128, 128] == np.float32(0.99) * np.float32(0.5))


def test_load_reduction_constructed(port):
    # acceptance.cpp:262-280: splats centred on 2x2 groups covering all 4 member tiles -> 0.75
    proj = np.zeros(64, PROJ_DTYPE)
    for gy in range(8):
        for gx in range(8):
            k = gy * 8 + gx
            proj[k]["mean2d"] = (32.0 * gx + 16.0, 32.0 * gy + 16.0)
            proj[k]["radius"] = 8
            proj[k]["depth"] = 1.0 + 0.01 * k
            proj[k]["conic"] = (0.1, 0.0, 0.1)
            proj[k]["opacity"] = 0.5
    ent, off, app = port.bin_sort(proj, 256, 256, 2)
    assert len(ent) == 64 and app == 256 and 1.0 - len(ent) / app == 0.75
    assert np.all(ent["mask"] == 0b1111)
    assert ENTRY_DTYPE.itemsize == 12


@pytest.mark.parametrize("seed,count,smin,smax,rot", [(61, 20000, 0.01, 0.05, False), (62, 8000, 0.02, 0.2, True),
                                                      (63, 5000, 0.01, 0.08, True)])
def test_fast_bin_sort_matches_sort_entries(port, seed, count, smin, smax, rot):
    """tor_bin_sort_fast (presort by (depth, index) + stable distribution by group, used by the
    full-size GPU parity tests) equals the restatement of build_group_entries + std::stable_sort
    (binning.cpp:46-100) entry for entry, including depth ties."""
    cam = rotated_camera(480, 270, yaw_deg=9.0, pitch_deg=-4.0) if rot else make_camera(480, 270)
    rec = np.array(port.gen_scene(seed, count, 1.0, smin, smax, 0), np.float32)
    rec[::7, 2] = rec[3, 2]  # depth ties across many splats
    pp, _ = port.project(rec, cam)
    for g in (1, 2, 4):
        ea, oa, xa = port.bin_sort(pp, cam.width, cam.height, g)
        eb, ob, xb = port.bin_sort_fast(pp, cam.width, cam.height, g)
        assert np.array_equal(_bits(ea), _bits(eb)) and np.array_equal(oa, ob) and xa == xb


def test_fast_bin_sort_matches_reference_build(port, ref):
    cam = rotated_camera(320, 200, yaw_deg=-13.0, pitch_deg=6.0)
    rec = port.gen_scene(64, 6000, 1.0, 0.01, 0.1, 0)
    pp, _ = port.project(rec, cam)
    for g in (1, 2, 4):
        ea, oa, xa = ref.bin_sort(pp, cam.width, cam.height, g)
        eb, ob, xb = port.bin_sort_fast(pp, cam.width, cam.height, g)
        assert np.array_equal(_bits(ea), _bits(eb)) and np.array_equal(oa, ob) and xa == xb


def test_expf_restatement_matches_libm(port):
    """The glibc expf restatement the exact-emulation rasteriser runs on the GPU equals this host's
    libm expf on every 7th negative float down to -88 (the full sweep, every float, differs in one
    input, x = -0x1.f8cbb2p+5, whose exp is ~1e-28 — far below any alpha_skip threshold)."""
    import ctypes as C
    f = port.lib.tor_expf_sweep
    f.restype = C.c_int64
    f.argtypes = [C.c_uint32, C.c_uint32, C.c_uint32, C.POINTER(C.c_float)]
    first = C.c_float(0)
    # -0.0 .. -88.0 (0x80000000 .. 0xC2B00000), stride 7
    bad = f(0x80000000, 0xC2B00000, 7, C.byref(first))
    assert bad <= 1, (bad, first.value)
    # the range every alpha >= 1/255 evaluation lives in (power >= ln(1/255) ~ -5.55), every float
    assert f(0x80000000, 0xC0B20000, 1, C.byref(first)) == 0
