"""Multi-GPU partitioning of the render path: one process per GPU, no collective on
the data path.

* Camera batches (BASELINE config 5): frames are independent.  Rank r of N renders cameras
  ``r, r + N, r + 2N, ...`` of each step ("weak" scaling: per-GPU work is fixed as N grows).
* Screen bands (config 4): every rank runs the full (cheap) preprocess and bins/sorts/rasterises
  only its band of group rows (``tgs_render_band``); band boundaries balance the per-row work.  The
  band images are contiguous row ranges of the frame, so a final gather is a plain concatenation.

The only collectives are for measurement and the optional final gather: the max-over-ranks of the
timed region and a gather of band images to rank 0.  They go through ``torch.distributed`` (NCCL on
the GPU box, gloo in the CPU tests).
"""
from __future__ import annotations

from typing import List, Sequence, Tuple

import numpy as np


def camera_schedule(n_cams: int, world: int, rank: int, n_steps: int, first_step: int = 0) -> List[int]:
    """Orbit-camera indices rank ``rank`` renders at steps ``first_step .. first_step+n_steps-1``:
    step i, rank r -> camera (i * world + r) mod n_cams.  Over world consecutive ranks a step covers
    world distinct cameras (for world <= n_cams)."""
    return [((first_step + i) * world + rank) % n_cams for i in range(n_steps)]


def band_split(row_work: Sequence[float], world: int) -> List[Tuple[int, int]]:
    """Split group rows ``[0, len(row_work))`` into ``world`` contiguous bands of balanced work
    (greedy prefix cut at k/world of the total); every band has at least one row when there are
    at least ``world`` rows.  ``row_work[y]`` is the work estimate of group row y (e.g. its entry
    count, which every rank can compute locally because preprocess is replicated)."""
    w = np.asarray(row_work, dtype=np.float64)
    rows = len(w)
    if world <= 0:
        raise ValueError("world must be >= 1")
    if rows == 0:
        return [(0, 0)] * world
    w = np.maximum(w, 1e-9)  # empty rows still cost a little; keeps cuts well defined
    cum = np.concatenate([[0.0], np.cumsum(w)])
    cuts = [0]
    for k in range(1, world):
        target = cum[-1] * k / world
        c = int(np.searchsorted(cum, target, side="left"))
        lo = cuts[-1] + 1 if rows >= world else cuts[-1]
        hi = rows - (world - k) if rows >= world else rows
        cuts.append(int(min(max(c, lo), hi)))
    cuts.append(rows)
    return [(cuts[k], cuts[k + 1]) for k in range(world)]


def band_rows_px(band: Tuple[int, int], group_size: int, height: int, tile: int = 16) -> Tuple[int, int]:
    """Pixel rows covered by a band of group rows (the last band is clipped to the image)."""
    g0, g1 = band
    return min(height, g0 * group_size * tile), min(height, g1 * group_size * tile)


def max_over_ranks(value: float, device=None) -> float:
    """Max of a per-rank scalar (the timed region of every rank) over the process group."""
    import torch
    import torch.distributed as dist
    if not dist.is_available() or not dist.is_initialized() or dist.get_world_size() == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def gather_bands(band_img: np.ndarray, bands_px: Sequence[Tuple[int, int]], width: int,
                 device=None) -> np.ndarray | None:
    """Gather every rank's band image (rows ``bands_px[rank]``) into the full frame on rank 0
    (other ranks get None).  Bands are contiguous row ranges, so the frame is their concatenation."""
    import torch
    import torch.distributed as dist
    rank, world = dist.get_rank(), dist.get_world_size()
    heights = [b1 - b0 for b0, b1 in bands_px]
    hmax = max(max(heights), 1)
    buf = torch.zeros((hmax, width, 3), dtype=torch.float32, device=device)
    if heights[rank]:
        buf[:heights[rank]] = torch.from_numpy(np.ascontiguousarray(band_img)).to(buf.device)
    out = [torch.zeros_like(buf) for _ in range(world)] if rank == 0 else None
    dist.gather(buf, out, dst=0)
    if rank != 0:
        return None
    return np.concatenate([out[k][:heights[k]].cpu().numpy() for k in range(world)], axis=0)
