"""GPU parity tests (B200): the CUDA path through the C ABI against the oracle.

Bar (north_star): projected splats, tile/group lists and sort order are BIT-EXACT against the
reference (golden fixtures generated from the reference build, and the C restatement on fresh
seeds); images are within a stated tolerance of the reference's FP32 image:

    IMG_MAX_ABS = 2/255 per channel (a splat whose alpha sits within rounding of the
                  alpha_skip = 1/255 threshold, or whose blend crosses t_terminate, may flip),
    IMG_PSNR    = 50 dB,
    IMG_MEAN    = 2e-5 mean absolute error.
"""
import math
import os

import numpy as np
import pytest

from tests.cases import CASES, make_camera, rotated_camera

pytestmark = pytest.mark.gpu

IMG_MAX_ABS = 2.0 / 255.0
IMG_PSNR = 50.0
IMG_MEAN = 2e-5


@pytest.fixture(scope="module")
def gsr():
    from paper_2605_17855_b200 import gsr as g
    return g


@pytest.fixture(scope="module")
def ctx(gsr):
    return gsr.default_context(0)


def _cam(gsr, c):
    return gsr.Camera(np.asarray(c.view, np.float32), c.focal_x, c.focal_y, c.width, c.height, c.near, c.far)


def _opt(gsr, backend, group, mode=0):
    return gsr.RenderOptions(gsr.Backend(backend), gsr.PrecisionMode(mode), group)


def check_image(got, ref, what=""):
    got = np.asarray(got, np.float64)
    ref = np.asarray(ref, np.float64)
    assert got.shape == ref.shape
    d = np.abs(got - ref)
    se = float(np.sum(d * d))
    psnr = 99.0 if se == 0 else 10 * math.log10(1.0 / (se / d.size))
    assert d.max() <= IMG_MAX_ABS, f"{what}: max abs {d.max():.3g}"
    assert d.mean() <= IMG_MEAN, f"{what}: mean abs {d.mean():.3g}"
    assert psnr >= IMG_PSNR, f"{what}: psnr {psnr:.1f}"
    return psnr, d.max()


# ---------------------------------------------------------------------------------------------
@pytest.mark.parametrize("name", list(CASES))
def test_projection_bitexact_vs_golden(gsr, ctx, golden, name):
    g = golden[name]
    cam = _cam(gsr, CASES[name]["camera"]())
    ds = ctx.upload(g["records"])
    res = ctx.render(ds, cam, _opt(gsr, 1, 2))
    proj = ctx.read_projected()
    assert np.array_equal(proj.view(np.uint8), g["projected"])
    st = g["proj_stats"]
    assert (res.projection.input, res.projection.culled, res.projection.dropped_degenerate) == tuple(st)


@pytest.mark.parametrize("name", list(CASES))
@pytest.mark.parametrize("group", [1, 2, 4])
def test_lists_bitexact_vs_golden(gsr, ctx, golden, name, group):
    g = golden[name]
    cam = _cam(gsr, CASES[name]["camera"]())
    ds = ctx.upload(g["records"])
    res = ctx.render(ds, cam, _opt(gsr, 0 if group == 1 else 1, group))
    ng = len(g[f"offsets_g{group}"]) - 1
    ent, off = ctx.read_lists(ng)
    assert np.array_equal(off, g[f"offsets_g{group}"])
    assert np.array_equal(ent.view(np.uint8), g[f"entries_g{group}"])
    assert res.entries == len(ent)
    assert res.tile_appearances == int(g[f"appearances_g{group}"][0])


@pytest.mark.parametrize("name", list(CASES))
@pytest.mark.parametrize("group", [1, 2, 4])
def test_reuse_report_vs_golden_masks(gsr, ctx, golden, name, group):
    """ReuseReport (metrics.cpp:45-57 load_reduction) is a pure function of the reference's entry
    masks: recompute it from the golden lists and compare with the device-side report."""
    g = golden[name]
    cam = _cam(gsr, CASES[name]["camera"]())
    ds = ctx.upload(g["records"])
    ctx.render(ds, cam, _opt(gsr, 0 if group == 1 else 1, group))
    ng = len(g[f"offsets_g{group}"]) - 1
    ent, _ = ctx.read_lists(ng)
    assert np.array_equal(ent.view(np.uint8), g[f"entries_g{group}"])
    pc = np.unpackbits(np.ascontiguousarray(ent["mask"]).view(np.uint8).reshape(len(ent), -1), axis=1).sum(1)
    hist = np.bincount(pc, minlength=17)[:17]
    rep = ctx.reuse_report()
    assert rep["mask_popcount_hist"] == [int(v) for v in hist]
    assert rep["n_group"] == len(ent) and rep["n_total"] == int(pc.sum())
    assert rep["load_reduction"] == pytest.approx(1.0 - len(ent) / int(pc.sum()), rel=0, abs=1e-15)


@pytest.mark.parametrize("name", list(CASES))
@pytest.mark.parametrize("backend,group,mode,tag", [
    (0, 1, 0, "scalar_g1"), (1, 1, 0, "tensor_g2"), (1, 2, 0, "tensor_g2"), (1, 4, 0, "tensor_g2"),
    (1, 2, 1, "tensor_g4_fp16"), (1, 4, 1, "tensor_g4_fp16"), (0, 1, 1, "tensor_g4_fp16")])
def test_image_within_tolerance_vs_golden(gsr, ctx, golden, name, backend, group, mode, tag):
    g = golden[name]
    cam = _cam(gsr, CASES[name]["camera"]())
    ds = ctx.upload(g["records"])
    res = ctx.render(ds, cam, _opt(gsr, backend, group, mode))
    ref = g[f"img_{tag}"]
    if mode == 1:
        # fp16 mode runs the exact emulation of the reference's fp16 lanes: bit for bit, for every
        # backend and G (the reference's fp16 image is G- and backend-invariant itself,
        # test_raster_tensor.cpp:159-165 and acceptance.cpp:199-238)
        assert np.array_equal(res.image.rgb.view(np.uint32), ref.astype(np.float32).view(np.uint32))
        assert gsr.psnr(res.image.rgb, g["img_tensor_g2"]) >= 40.0  # the reference's fp16 bar
    else:
        check_image(res.image.rgb, ref, f"{name} b{backend} g{group} m{mode}")


def test_fresh_seeds_vs_port(gsr, ctx, port):
    for seed, n, sh, rot, (w, h) in [(31, 4000, 0, False, (200, 120)), (32, 2500, 5, True, (160, 160)),
                                     (33, 6000, 0, True, (333, 187))]:
        c = rotated_camera(w, h, yaw_deg=11.0 * seed % 40 - 20, pitch_deg=-6.0) if rot else make_camera(w, h)
        cam = _cam(gsr, c)
        rec = port.gen_scene(seed, n, 1.0, 0.01, 0.08, sh)
        pp, _ = port.project(rec, c)
        ds = ctx.upload(rec)
        for group in (1, 2, 4):
            res = ctx.render(ds, cam, _opt(gsr, 0 if group == 1 else 1, group))
            assert np.array_equal(ctx.read_projected().view(np.uint8), pp.view(np.uint8))
            ent_p, off_p, app_p = port.bin_sort(pp, w, h, group)
            ent, off = ctx.read_lists(len(off_p) - 1)
            assert np.array_equal(off, off_p) and np.array_equal(ent.view(np.uint8), ent_p.view(np.uint8))
            assert res.tile_appearances == app_p
            img_p, cnt = port.rasterize(ent_p, off_p, pp, w, h, backend=0 if group == 1 else 1, group_size=group)
            check_image(res.image.rgb, img_p, f"seed {seed} g{group}")
            walked, blended = ctx.count_pairs()
            assert abs(walked - cnt["walked_pairs"]) <= max(16, 1e-4 * cnt["walked_pairs"])
            assert abs(blended - cnt["blended_pairs"]) <= max(16, 1e-4 * cnt["blended_pairs"])


def test_config1_scale_vs_port(gsr, ctx, port):
    """BASELINE config 1: 100K splats, SH degree 3, 800x800 — lists bit-exact, image in tolerance."""
    c = make_camera(800, 800)
    rec = port.gen_scene(1, 100_000, 1.0, 0.01, 0.05, 5)
    pp, _ = port.project(rec, c)
    ds = ctx.upload(rec)
    cam = _cam(gsr, c)
    res = ctx.render(ds, cam, _opt(gsr, 1, 2))
    assert np.array_equal(ctx.read_projected().view(np.uint8), pp.view(np.uint8))
    ent_p, off_p, app_p = port.bin_sort(pp, 800, 800, 2)
    ent, off = ctx.read_lists(len(off_p) - 1)
    assert np.array_equal(off, off_p) and np.array_equal(ent.view(np.uint8), ent_p.view(np.uint8))
    img_p, _ = port.rasterize(ent_p, off_p, pp, 800, 800, backend=1, group_size=2)
    check_image(res.image.rgb, img_p, "config1 tensor g2")
    res1 = ctx.render(ds, cam, _opt(gsr, 0, 1))
    check_image(res1.image.rgb, img_p, "config1 scalar g1")


@pytest.mark.parametrize("depths", ["ties", "narrow", "wide"])
def test_presort_key_ranges_vs_port(gsr, ctx, port, depths):
    """The presort ranks (key - min key): a key range of a few bits leaves passes 1-3 as copies,
    equal depths leave every pass after the culling one trivial, a wide range needs all four."""
    w, h = 240, 160
    c = make_camera(w, h)
    rec = np.array(port.gen_scene(41, 5000, 1.0, 0.01, 0.06, 0), np.float32)
    rng = np.random.default_rng(7)
    z = {"ties": np.full(5000, 3.0), "narrow": 2.0 + rng.random(5000) * 1e-3,
         "wide": np.exp(rng.uniform(np.log(0.25), np.log(90.0), 5000))}[depths]
    rec[:, 0] = rng.uniform(-0.6, 0.6, 5000) * z
    rec[:, 1] = rng.uniform(-0.4, 0.4, 5000) * z
    rec[:, 2] = z
    rec[::97, 2] = -1.0  # some culled behind the camera
    pp, _ = port.project(rec, c)
    ds = ctx.upload(rec)
    for group in (1, 2):
        ctx.render(ds, _cam(gsr, c), _opt(gsr, 0 if group == 1 else 1, group))
        ent_p, off_p, _ = port.bin_sort(pp, w, h, group)
        ent, off = ctx.read_lists(len(off_p) - 1)
        assert np.array_equal(off, off_p) and np.array_equal(ent.view(np.uint8), ent_p.view(np.uint8))


def test_placement_stage_overflow_vs_port(gsr, ctx, port):
    """Large splats (mean radius ~130 px at 640x360): a level-2 segment of 2048 row entries emits
    more group entries than the block's shared stage (12K entries: ~35K at G=1, ~18K at G=2), so
    group placement takes its direct-to-global path; lists must still be bit-exact, on the first
    and on a repeated frame.  (The level-1 direct path is covered at full size: the first C3 G=1
    frame, tests/test_gpu_fullsize.py.)"""
    w, h = 640, 360
    c = make_camera(w, h)
    rec = port.gen_scene(51, 40000, 1.0, 0.15, 0.3, 0)
    pp, _ = port.project(rec, c)
    ds = ctx.upload(rec)
    for group in (1, 2, 4):
        ent_p, off_p, app_p = port.bin_sort(pp, w, h, group)
        for _ in range(2):
            res = ctx.render(ds, _cam(gsr, c), _opt(gsr, 0 if group == 1 else 1, group))
            ent, off = ctx.read_lists(len(off_p) - 1)
            assert np.array_equal(off, off_p) and np.array_equal(ent.view(np.uint8), ent_p.view(np.uint8))
            assert res.tile_appearances == app_p


# ---------------------------------------------------------------------------------------------
# edge cases the reference tests
# ---------------------------------------------------------------------------------------------
def test_empty_scene_is_black(gsr):
    for backend, group in [(0, 1), (1, 2), (1, 4)]:
        res = gsr.render([], gsr.make_camera(64, 48), _opt(gsr, backend, group))
        assert res.image.rgb.shape == (48, 64, 3) and not res.image.rgb.any()
        assert res.entries == 0 and res.tile_appearances == 0


def test_all_culled_and_tiny_images(gsr, port):
    rec = port.gen_scene(5, 200, 1.0, 0.01, 0.05, 0)
    rec[:, 2] = -5.0  # behind the camera
    res = gsr.render(rec, gsr.make_camera(37, 19), _opt(gsr, 1, 2))
    assert res.projection.culled == 200 and not res.image.rgb.any()
    rec = port.gen_scene(6, 500, 1.0, 0.05, 0.3, 0)
    for w, h in [(1, 1), (17, 17), (15, 33)]:
        c = make_camera(w, h)
        img_p, _ = port.render(rec, c, backend=0, group_size=1)
        for backend, group in [(0, 1), (1, 1), (1, 2), (1, 4)]:
            res = gsr.render(rec, _cam(gsr, c), _opt(gsr, backend, group))
            check_image(res.image.rgb, img_p, f"{w}x{h} b{backend} g{group}")


def test_single_opaque_splat_center(gsr):
    # test_raster_scalar.cpp:92-104: center pixel = 0.99 * 0.5 (alpha clamp), tolerance for ex2
    cam = gsr.make_camera(256, 256)
    cam.focal_x = cam.focal_y = 100.0
    g = gsr.Gaussian3D(mean=(0, 0, 10), scale=(1, 1, 1), opacity=1.0, sh_dc=(0, 0, 0))
    for backend, group in [(0, 1), (1, 2)]:
        res = gsr.render([g], cam, _opt(gsr, backend, group))
        assert np.allclose(res.image.pixel(128, 128), 0.99 * 0.5, atol=1e-6)


def test_validation_errors(gsr, port):
    cam = gsr.make_camera(64, 64)
    with pytest.raises(gsr.ValidationError):
        gsr.render([], cam, gsr.RenderOptions(gsr.Backend.scalar, group_size=2))
    with pytest.raises(gsr.ValidationError):
        gsr.render([], cam, gsr.RenderOptions(group_size=3))
    with pytest.raises(gsr.ValidationError):
        gsr.render([], cam, gsr.RenderOptions(workers=0))
    with pytest.raises(gsr.ValidationError):
        gsr.render([], gsr.make_camera(0, 10))
    bad = gsr.Gaussian3D(mean=(0, 0, 5), scale=(0.0, 1, 1), opacity=0.5)
    with pytest.raises(gsr.ValidationError):
        gsr.render([bad], cam)
    # culled splats with bad scale are not an error (projection.cpp:121-125 culls first)
    bad_culled = gsr.Gaussian3D(mean=(0, 0, -5), scale=(0.0, 1, 1), opacity=0.5)
    gsr.render([bad_culled], cam)
    # negative depth reaching the binner (near < 0) -> sort_entries ValidationError
    cam2 = gsr.make_camera(64, 64)
    cam2.near = -10.0
    g = gsr.Gaussian3D(mean=(0.0, 0.0, -1.0), scale=(0.05, 0.05, 0.05), opacity=0.5)
    with pytest.raises(gsr.ValidationError):
        gsr.render([g], cam2, gsr.RenderOptions(group_size=2))


def test_determinism_and_option_invariance(gsr, ctx, port):
    """acceptance.cpp:359-382 / :227-238: identical images for repeated runs, any workers and
    chunk_len; tensor G=1/2/4 agree within tolerance of each other."""
    rec = port.gen_scene(8, 2000, 1.0, 0.01, 0.08, 0)
    cam = gsr.make_camera(256, 256)
    ds = ctx.upload(rec)
    for backend, group in [(0, 1), (1, 2), (1, 4)]:
        base = ctx.render(ds, cam, _opt(gsr, backend, group)).image.rgb.copy()
        for rep in range(5):
            o = _opt(gsr, backend, group)
            o.workers = 1 + rep
            o.chunk_len = (1, 5, 16, 3, 9)[rep]
            again = ctx.render(ds, cam, o).image.rgb
            assert np.array_equal(base.view(np.uint32), again.view(np.uint32))


def test_band_and_batch_match_full_frame(gsr, ctx, port):
    rec = port.gen_scene(9, 5000, 1.0, 0.01, 0.08, 0)
    cam = gsr.make_camera(300, 200)
    ds = ctx.upload(rec)
    for backend, group in [(0, 1), (1, 2), (1, 4)]:
        opt = _opt(gsr, backend, group)
        full = ctx.render(ds, cam, opt).image.rgb.copy()
        gy = -(-(-(-200 // 16)) // group)
        cuts = [0, gy // 3, gy // 2 + 1, gy]
        stitched = np.concatenate([ctx.render_band(ds, cam, opt, a, b)[0] for a, b in zip(cuts, cuts[1:])])
        assert np.array_equal(stitched.view(np.uint32), full.view(np.uint32))
    cams = gsr.orbit_cameras(4, 160, 120)
    out, _ = ctx.render_batch(ds, cams, _opt(gsr, 1, 2))
    for k, c in enumerate(cams):
        one = ctx.render(ds, c, _opt(gsr, 1, 2)).image.rgb
        assert np.array_equal(out[k].view(np.uint32), one.view(np.uint32))


def test_capacity_growth_across_scenes(gsr, ctx, port):
    """Entry buffers grow on overflow and the frame is re-rendered transparently."""
    small = ctx.upload(port.gen_scene(10, 100, 1.0, 0.01, 0.05, 0))
    big_rec = port.gen_scene(11, 20000, 1.0, 0.05, 0.2, 0)
    big = ctx.upload(big_rec)
    cam = gsr.make_camera(320, 240)
    ctx.render(small, cam, _opt(gsr, 1, 2))
    res = ctx.render(big, cam, _opt(gsr, 0, 1))
    pp, _ = port.project(big_rec, make_camera(320, 240))
    _, off_p, app_p = port.bin_sort(pp, 320, 240, 1)
    assert res.entries == int(off_p[-1]) and res.tile_appearances == app_p


# ---------------------------------------------------------------------------------------------
# full BASELINE size: size-independent properties (C3: 3M splats, 1080p)
# ---------------------------------------------------------------------------------------------
def test_c3_full_size_properties(gsr, ctx, port):
    c = make_camera(1920, 1080)
    rec = gsr.gen_synthetic_scene(3, 3_000_000, 1.0, (0.01, 0.05)).records
    pp, st = port.project(rec, c)
    ds = ctx.upload(rec)
    cam = _cam(gsr, c)
    for group in (2, 1):
        res = ctx.render(ds, cam, _opt(gsr, 1, group))
        proj = ctx.read_projected()
        assert np.array_equal(proj.view(np.uint8), pp.view(np.uint8))
        # entry count and appearances from the port's projection, vectorised recount
        r = pp["radius"].astype(np.float32)
        mx, my = pp["mean2d"][:, 0], pp["mean2d"][:, 1]
        tx0 = np.maximum(np.floor((mx - r) / np.float32(16)).astype(np.int64), 0)
        tx1 = np.minimum(np.floor((mx + r) / np.float32(16)).astype(np.int64), 119)
        ty0 = np.maximum(np.floor((my - r) / np.float32(16)).astype(np.int64), 0)
        ty1 = np.minimum(np.floor((my + r) / np.float32(16)).astype(np.int64), 67)
        ok = (tx1 >= tx0) & (ty1 >= ty0)
        app = int(np.sum(((tx1 - tx0 + 1) * (ty1 - ty0 + 1))[ok]))
        n_ent = int(np.sum(((tx1 // group - tx0 // group + 1) * (ty1 // group - ty0 // group + 1))[ok]))
        assert res.tile_appearances == app and res.entries == n_ent
        ng = ((120 + group - 1) // group) * ((68 + group - 1) // group)
        ent, off = ctx.read_lists(ng)
        assert off[-1] == n_ent
        # per-group order: (depth bits, index) strictly increasing; masks non-empty; popcounts sum
        gid = np.repeat(np.arange(ng), np.diff(off.astype(np.int64)))
        key = (gid.astype(np.uint64) << np.uint64(32)) | ent["depth"].view(np.uint32).astype(np.uint64)
        dk = np.diff(key.astype(np.int64))
        assert np.all(dk >= 0)
        ties = dk == 0
        assert np.all(np.diff(ent["gaussian_index"].astype(np.int64))[ties] > 0)
        assert np.all(ent["mask"] != 0)
        pc = np.unpackbits(np.ascontiguousarray(ent["mask"]).view(np.uint8)).sum()
        assert int(pc) == app
        img = res.image.rgb
        assert np.isfinite(img).all() and img.min() >= 0 and img.max() <= 1


def test_c4_full_size_properties(gsr, ctx, port):
    """BASELINE config 4 (6M splats, 3840x2160): projection bit-exact vs the port; entry counts and
    tile appearances equal the recount from it (G=2: 386.5M entries, G=4); at G=4 every list in
    (depth, index) order with non-empty masks whose popcounts sum to the appearances (SURVEY §8(d):
    count + popcount conservation at C4).  Each geometry renders twice: the second frame's level-1
    chunks are sized from the first one's row entries, and its lists are the ones checked."""
    c = make_camera(3840, 2160)
    rec = gsr.gen_synthetic_scene(4, 6_000_000, 1.0, (0.01, 0.05)).records
    pp, _ = port.project(rec, c)
    ds = ctx.upload(rec)
    cam = _cam(gsr, c)
    r = pp["radius"].astype(np.float32)
    mx, my = pp["mean2d"][:, 0], pp["mean2d"][:, 1]
    tx0 = np.maximum(np.floor((mx - r) / np.float32(16)).astype(np.int64), 0)
    tx1 = np.minimum(np.floor((mx + r) / np.float32(16)).astype(np.int64), 239)
    ty0 = np.maximum(np.floor((my - r) / np.float32(16)).astype(np.int64), 0)
    ty1 = np.minimum(np.floor((my + r) / np.float32(16)).astype(np.int64), 134)
    ok = (tx1 >= tx0) & (ty1 >= ty0)
    app = int(np.sum(((tx1 - tx0 + 1) * (ty1 - ty0 + 1))[ok]))
    for group in (2, 4):
        ctx.render(ds, cam, _opt(gsr, 1, group))
        res = ctx.render(ds, cam, _opt(gsr, 1, group))
        if group == 2:
            assert np.array_equal(ctx.read_projected().view(np.uint8), pp.view(np.uint8))
        n_ent = int(np.sum(((tx1 // group - tx0 // group + 1) * (ty1 // group - ty0 // group + 1))[ok]))
        assert res.tile_appearances == app and res.entries == n_ent
        if group == 2:
            assert n_ent == 386_505_600
            continue
        ng = ((240 + group - 1) // group) * ((135 + group - 1) // group)
        ent, off = ctx.read_lists(ng)
        assert off[-1] == n_ent
        gid = np.repeat(np.arange(ng), np.diff(off.astype(np.int64)))
        key = (gid.astype(np.uint64) << np.uint64(32)) | ent["depth"].view(np.uint32).astype(np.uint64)
        dk = np.diff(key.astype(np.int64))
        assert np.all(dk >= 0)
        ties = dk == 0
        assert np.all(np.diff(ent["gaussian_index"].astype(np.int64))[ties] > 0)
        assert np.all(ent["mask"] != 0)
        pc = np.unpackbits(np.ascontiguousarray(ent["mask"]).view(np.uint8)).sum()
        assert int(pc) == app
        del ent, gid, key, dk


# ---------------------------------------------------------------------------------------------
# Exact-emulation rasteriser: images BIT-EXACT with the reference build (golden fixtures made by
# oracle/_ref) in fp16 mode (PrecisionMode::fp16 always runs it) and in fp32 mode with
# tgs_set_exact_emulation — the reference's own acceptance invariants (scalar == tensor, any G,
# acceptance.cpp:177-238) make one exact kernel cover every backend/G combination.
@pytest.mark.parametrize("name", list(CASES))
@pytest.mark.parametrize("render", ["scalar_g1", "tensor_g2", "tensor_g4_fp16"])
def test_exact_emulation_bit_exact_vs_reference(gsr, golden, name, render):
    case, gold = CASES[name], golden[name]
    c = case["camera"]()
    r = case["renders"][render]
    ctx = gsr.Context(0)
    try:
        ctx.set_exact_emulation(True)
        res = ctx.render(ctx.upload(gold["records"]), _cam(gsr, c),
                         _opt(gsr, r["backend"], r["group_size"], r["mode"]))
        ref = gold[f"img_{render}"]
        assert np.array_equal(res.image.rgb.view(np.uint32), ref.astype(np.float32).view(np.uint32)), \
            f"{name} {render}: {np.count_nonzero(res.image.rgb != ref)} pixels differ"
    finally:
        ctx.close()


@pytest.mark.parametrize("mode", [0, 1])
def test_exact_emulation_matches_port_every_group(gsr, port, mode):
    """Fresh seeds: the exact kernel equals the C restatement (itself pinned to the reference) for
    G = 1, 2, 4, both precision modes, bit for bit."""
    rec = port.gen_scene(31, 2500, 1.0, 0.01, 0.08, 5 if mode else 0)
    c = rotated_camera(176, 136)
    ctx = gsr.Context(0)
    try:
        ctx.set_exact_emulation(True)
        ds = ctx.upload(rec)
        proj, _ = port.project(rec, c)
        for g in (1, 2, 4):
            backend = 0 if g == 1 else 1
            res = ctx.render(ds, _cam(gsr, c), _opt(gsr, backend, g, mode))
            ent, off, _ = port.bin_sort(proj, c.width, c.height, g)
            img, _ = port.rasterize(ent, off, proj, c.width, c.height, backend=backend, group_size=g, mode=mode)
            assert np.array_equal(res.image.rgb.view(np.uint32), img.astype(np.float32).view(np.uint32)), (mode, g)
    finally:
        ctx.close()
