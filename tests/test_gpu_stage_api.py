"""GPU tests of the reference's public STAGE API on the B200 path:

    project_scene          (proj/include/gsr/projection.hpp:48-50)
    build_group_entries    (proj/include/gsr/binning.hpp:68-69)
    sort_entries           (proj/include/gsr/binning.hpp:72-73)
    rasterize_tiles_scalar (proj/include/gsr/raster_scalar.hpp:59-62)
    rasterize_groups_tensor(proj/include/gsr/raster_tensor.hpp:62-65)

each called on caller-provided data through the C ABI (tgs_project_scene, tgs_build_group_entries,
tgs_sort_entries, tgs_rasterize_lists) and compared with the oracle: projected records, entries
and sorted lists BIT-EXACT, images within the parity tolerance of tests/test_gpu_parity.py.
Error behaviour follows the reference: bad depths and GroupConfig violations raise
ValidationError (binning.cpp:22-30, :78-83), the scalar rasteriser requires 1x1 groups
(raster_scalar.cpp:56-57).
"""
import numpy as np
import pytest

from tests.cases import make_camera, rotated_camera

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def gsr():
    from paper_2605_17855_b200 import gsr as g
    return g


def _cam(gsr, c):
    return gsr.Camera(np.asarray(c.view, np.float32), c.focal_x, c.focal_y, c.width, c.height, c.near, c.far)


SCENES = [(21, 3000, 0, make_camera(200, 144)), (22, 1500, 5, rotated_camera(160, 120)),
          (23, 800, 0, make_camera(100, 72))]


@pytest.mark.parametrize("k", range(len(SCENES)))
def test_project_scene_bit_exact(gsr, port, k):
    seed, n, sh, c = SCENES[k]
    rec = port.gen_scene(seed, n, 1.0, 0.01, 0.08, sh)
    st = gsr.ProjectionStats()
    got = gsr.project_scene(rec, _cam(gsr, c), workers=4, stats=st)
    ref, rst = port.project(rec, c)
    assert np.array_equal(got.view(np.uint8), ref.view(np.uint8))
    assert (st.input, st.culled, st.dropped_degenerate) == tuple(int(v) for v in rst)


@pytest.mark.parametrize("g", [1, 2, 4])
@pytest.mark.parametrize("k", range(len(SCENES)))
def test_build_and_sort_entries_bit_exact(gsr, port, k, g):
    seed, n, sh, c = SCENES[k]
    rec = port.gen_scene(seed, n, 1.0, 0.01, 0.08, sh)
    proj, _ = port.project(rec, c)
    cfg = gsr.GroupConfig.square(g, c.width, c.height)
    keyed = gsr.build_group_entries(proj, cfg)
    ent_ref, off_ref, _ = port.bin_sort(proj, c.width, c.height, g)
    # build_group_entries order is splat index, then group id (binning.cpp:46-74): the sorted
    # reference lists re-ordered by (index, group) must equal it record for record
    gid_ref = np.repeat(np.arange(len(off_ref) - 1, dtype=np.uint32), np.diff(off_ref))
    order = np.lexsort((gid_ref, ent_ref["gaussian_index"]))
    assert len(keyed) == len(ent_ref)
    assert np.array_equal(keyed["group_id"], gid_ref[order])
    assert np.array_equal(np.ascontiguousarray(keyed["entry"]).view(np.uint8), ent_ref[order].view(np.uint8))
    lists = gsr.sort_entries(keyed, cfg)
    assert np.array_equal(lists.offsets, off_ref)
    assert np.array_equal(lists.entries.view(np.uint8), ent_ref.view(np.uint8))


def test_sort_entries_stability_and_ties(gsr):
    """Caller-provided entries with many equal keys: stable (group_id << 32 | depth bits) order,
    ties in input order — numpy's stable sort on the same 64-bit key is the oracle."""
    rng = np.random.default_rng(7)
    cfg = gsr.GroupConfig.square(2, 640, 480)
    n = 200_000
    e = np.zeros(n, gsr.KEYED_DTYPE)
    e["group_id"] = rng.integers(0, cfg.group_count(), n)
    e["entry"]["gaussian_index"] = np.arange(n, dtype=np.uint32)
    e["entry"]["depth"] = rng.choice(np.float32([0.0, -0.0, 0.5, 1.0, 2.5, 3.0e-39, 7.0]), n)
    e["entry"]["mask"] = rng.integers(1, 16, n)
    lists = gsr.sort_entries(e, cfg)
    key = (e["group_id"].astype(np.uint64) << np.uint64(32)) | e["entry"]["depth"].view(np.uint32).astype(np.uint64)
    order = np.argsort(key, kind="stable")
    assert np.array_equal(lists.entries.view(np.uint8), e["entry"][order].view(np.uint8))
    counts = np.bincount(e["group_id"], minlength=cfg.group_count())
    assert np.array_equal(lists.offsets, np.concatenate([[0], np.cumsum(counts)]).astype(np.uint32))


def test_sort_entries_empty_and_errors(gsr):
    cfg = gsr.GroupConfig.square(2, 64, 64)
    empty = gsr.sort_entries(np.zeros(0, gsr.KEYED_DTYPE), cfg)
    assert len(empty.entries) == 0 and np.all(empty.offsets == 0)
    e = np.zeros(3, gsr.KEYED_DTYPE)
    e["entry"]["depth"] = [1.0, -1.0, 2.0]
    with pytest.raises(gsr.ValidationError, match="non-finite or negative depth"):
        gsr.sort_entries(e, cfg)
    e["entry"]["depth"] = [1.0, np.inf, 2.0]
    with pytest.raises(gsr.ValidationError, match="non-finite or negative depth"):
        gsr.sort_entries(e, cfg)
    e["entry"]["depth"] = [1.0, 1.0, 2.0]
    e["group_id"] = [0, 1, cfg.group_count()]
    with pytest.raises(gsr.ValidationError):
        gsr.sort_entries(e, cfg)
    with pytest.raises(gsr.ValidationError, match="group sizes"):
        gsr.GroupConfig.square(3, 64, 64)


@pytest.mark.parametrize("backend,g", [(0, 1), (1, 1), (1, 2), (1, 4)])
def test_rasterize_on_caller_lists(gsr, port, backend, g):
    from tests.test_gpu_parity import check_image
    for seed, n, sh, c in SCENES[:2]:
        rec = port.gen_scene(seed, n, 1.0, 0.01, 0.08, sh)
        proj, _ = port.project(rec, c)
        ent, off, _ = port.bin_sort(proj, c.width, c.height, g)
        lists = gsr.SortedGroupLists(ent, off)
        cfg = gsr.GroupConfig.square(g, c.width, c.height)
        if backend == 0:
            img = gsr.rasterize_tiles_scalar(lists, proj, cfg)
        else:
            img = gsr.rasterize_groups_tensor(lists, proj, cfg)
        ref, _ = port.rasterize(ent, off, proj, c.width, c.height, backend=backend, group_size=g)
        check_image(img.rgb, ref, f"stage raster b{backend} g{g} seed {seed}")


def test_rasterize_rejects_inconsistent_lists(gsr, port):
    seed, n, sh, c = SCENES[0]
    rec = port.gen_scene(seed, n, 1.0, 0.01, 0.08, sh)
    proj, _ = port.project(rec, c)
    ent, off, _ = port.bin_sort(proj, c.width, c.height, 2)
    cfg = gsr.GroupConfig.square(2, c.width, c.height)
    bad = ent.copy()
    bad["mask"][len(bad) // 2] ^= 0x8  # a member-tile bit the splat's rectangle does not give
    with pytest.raises(gsr.ValidationError, match="mask"):
        gsr.rasterize_groups_tensor(gsr.SortedGroupLists(bad, off), proj, cfg)
    bad = ent.copy()
    bad["gaussian_index"][0] = len(proj)
    with pytest.raises(gsr.ValidationError, match="out of range"):
        gsr.rasterize_groups_tensor(gsr.SortedGroupLists(bad, off), proj, cfg)
    with pytest.raises(gsr.ValidationError, match="group size 1"):
        gsr.rasterize_tiles_scalar(gsr.SortedGroupLists(ent, off), proj, cfg)
    with pytest.raises(gsr.ValidationError, match="offsets"):
        gsr.rasterize_groups_tensor(gsr.SortedGroupLists(ent, off[:-1]), proj, cfg)
