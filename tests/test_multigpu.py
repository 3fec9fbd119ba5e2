"""The N>1 path on CPU: world-size-2 gloo process groups exercise the camera-batch schedule, band
splitting, the max-over-ranks timing and the band gather that bench.py / multi-GPU callers use
(DESIGN.md §5).  GPU-side band/batch equivalence is covered by test_gpu_parity.py."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_2605_17855_b200 import multigpu


def test_camera_schedule_partitions_each_step():
    n_cams, world, steps = 256, 8, 40
    per_rank = [multigpu.camera_schedule(n_cams, world, r, steps) for r in range(world)]
    for i in range(steps):
        step = [per_rank[r][i] for r in range(world)]
        assert len(set(step)) == world  # distinct cameras within a step
    flat = [c for r in per_rank for c in r[:n_cams // world]]
    assert sorted(flat) == list(range(n_cams))  # first 32 steps cover the orbit exactly once


@pytest.mark.parametrize("world", [1, 2, 3, 8])
def test_band_split_covers_rows_and_balances(world):
    rng = np.random.default_rng(world)
    work = rng.integers(0, 1000, 68).astype(float)
    work[30:38] *= 20  # a heavy middle, like the centre of a frame
    bands = multigpu.band_split(work, world)
    assert bands[0][0] == 0 and bands[-1][1] == 68
    assert all(b0 < b1 for b0, b1 in bands)
    assert all(bands[k][1] == bands[k + 1][0] for k in range(world - 1))
    loads = [work[b0:b1].sum() for b0, b1 in bands]
    assert max(loads) <= work.sum() / world + work.max()


def test_band_rows_px_clip():
    assert multigpu.band_rows_px((0, 17), 2, 1080) == (0, 544)
    assert multigpu.band_rows_px((17, 34), 2, 1080) == (544, 1080)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        # max over ranks of the timed region
        t = multigpu.max_over_ranks(1.5 + rank)
        # band gather: each rank "renders" its band of a 100x40 frame (rows of value = row index)
        h, w, g = 100, 40, 2
        rows = -(-h // 16)
        groups_y = -(-rows // g)
        bands = multigpu.band_split(np.ones(groups_y), world)
        bands_px = [multigpu.band_rows_px(b, g, h) for b in bands]
        y0, y1 = bands_px[rank]
        img = np.repeat(np.arange(y0, y1, dtype=np.float32)[:, None, None], w, axis=1).repeat(3, axis=2)
        full = multigpu.gather_bands(img, bands_px, w)
        cams = multigpu.camera_schedule(256, world, rank, 4, first_step=3)
        q.put((rank, t, None if full is None else full[:, 0, 0].tolist(), cams))
    finally:
        dist.destroy_process_group()


def test_gloo_world2_timing_and_band_gather():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(world):
        rank, t, col, cams = q.get(timeout=120)
        res[rank] = (t, col, cams)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert res[0][0] == res[1][0] == 2.5  # max over ranks
    assert res[0][1] == list(range(100))  # bands reassembled in order on rank 0
    assert res[1][1] is None
    assert set(res[0][2]).isdisjoint(res[1][2])  # ranks render different cameras each step
