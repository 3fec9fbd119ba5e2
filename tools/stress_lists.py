"""Stress check of the binning/sort stage: render the same C3 frame repeatedly and verify that the
per-group offsets are monotone, end at the entry count and are identical across frames."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_17855_b200 import gsr  # noqa: E402

ctx = gsr.Context(0)
ds = ctx.upload(gsr.gen_synthetic_scene(3, 3_000_000, 1.0, (0.01, 0.05)))
cam = gsr.orbit_cameras(256, 1920, 1080)[5]
opt = gsr.RenderOptions(gsr.Backend.scalar, gsr.PrecisionMode.fp32, 1)
ref = None
n_groups = 120 * 68
for i in range(int(sys.argv[1]) if len(sys.argv) > 1 else 20):
    res = ctx.render(ds, cam, opt)
    ent, off = ctx.read_lists(n_groups)
    ok = bool(np.all(np.diff(off.astype(np.int64)) >= 0)) and int(off[-1]) == len(ent)
    same = ref is None or (np.array_equal(off, ref[0]) and np.array_equal(ent.view(np.uint8), ref[1].view(np.uint8)))
    print(i, "entries", len(ent), "monotone+total", ok, "identical", same, flush=True)
    if ref is None:
        ref = (off.copy(), ent.copy())
