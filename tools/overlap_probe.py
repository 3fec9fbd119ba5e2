"""Throughput of camera batches rendered by 1, 2 or 3 contexts (streams) in round robin on one GPU
(C5 workload): frames of different cameras overlap, so one frame's latency-bound raster shares the
SMs with another frame's preprocess/sort/binning.  python tools/overlap_probe.py [frames]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_17855_b200 import gsr  # noqa: E402


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 60
    scene = gsr.gen_synthetic_scene(3, 3_000_000, 1.0, (0.01, 0.05))
    cams = gsr.orbit_cameras(256, 1920, 1080)
    opt = gsr.RenderOptions(gsr.Backend.tensor, gsr.PrecisionMode.fp32, 2)
    ctxs = [gsr.Context(0) for _ in range(3)]
    ds = [c.upload(scene) for c in ctxs]
    for k in (1, 2, 3):
        cs, dd = ctxs[:k], ds[:k]
        streams = [torch.cuda.ExternalStream(c.stream) for c in cs]
        for i in range(2 * k + 6):  # warm-up incl. capacity growth and schedule feedback
            cs[i % k].enqueue(dd[i % k], cams[i % 256], opt)
            cs[i % k].sync()
        torch.cuda.synchronize()
        ev0 = [torch.cuda.Event(enable_timing=True) for _ in cs]
        ev1 = [torch.cuda.Event(enable_timing=True) for _ in cs]
        for e, s in zip(ev0, streams):
            e.record(s)
        for i in range(n):
            cs[i % k].enqueue(dd[i % k], cams[(10 + i) % 256], opt)
        for e, s in zip(ev1, streams):
            e.record(s)
        for c in cs:
            c.sync()
        torch.cuda.synchronize()
        ms = max(ev0[0].elapsed_time(e) for e in ev1)
        print(f"OVERLAP contexts={k}: {n} frames in {ms:.2f} ms -> {n / ms * 1e3:.1f} frames/s", flush=True)


if __name__ == "__main__":
    main()
