import os, sys
import numpy as np
sys.path.insert(0, '/root/repo')
from paper_2605_17855_b200 import gsr
ctx = gsr.Context(0)
ds = ctx.upload(gsr.gen_synthetic_scene(4, 6_000_000, 1.0, (0.01, 0.05)))
cam = gsr.make_camera(3840, 2160)
for g in (2, 4):
    opt = gsr.RenderOptions(gsr.Backend.tensor, gsr.PrecisionMode.fp32, g)
    rows = []
    for i in range(12):
        ctx.enqueue(ds, cam, opt)
        st = ctx.sync()
        rows.append((st.ms_preprocess, st.ms_sort, st.ms_binning, st.ms_raster, st.ms_total, st.entries))
    med = np.median(np.array(rows[4:]), axis=0)
    print("C4 G=%d pre %.3f sort %.3f bin %.3f raster %.3f total %.3f entries %d" % (g, *med[:5], med[5]), flush=True)
