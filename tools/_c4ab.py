"""A/B of binning variants on C4 (6M splats, 3840x2160, identity camera, tensor G=2) and G=1 C3."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_17855_b200 import gsr  # noqa: E402
tag = sys.argv[1]
ctx = gsr.Context(0)
for name, seed, n, w, h, backend, g in (("c4", 4, 6_000_000, 3840, 2160, gsr.Backend.tensor, 2),
                                         ("c3g1", 3, 3_000_000, 1920, 1080, gsr.Backend.scalar, 1)):
    ds = ctx.upload(gsr.gen_synthetic_scene(seed, n, 1.0, (0.01, 0.05)))
    cam = gsr.make_camera(w, h)
    opt = gsr.RenderOptions(backend, gsr.PrecisionMode.fp32, g)
    rows = []
    for i in range(12):
        ctx.enqueue(ds, cam, opt)
        st = ctx.sync()
        rows.append((st.ms_binning, st.ms_total))
    med = np.median(np.array(rows[4:]), axis=0)
    print(f"C4AB {tag} {name}: bin {med[0]:.3f} total {med[1]:.3f} ms", flush=True)
    ds.free()
