"""Render the bench frame (orbit camera CAM) with the default library and save it, or compare two
saved renders: python tools/_imgdiff.py save PATH CAM | python tools/_imgdiff.py cmp A B"""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
if sys.argv[1] == "save":
    from paper_2605_17855_b200 import gsr
    ctx = gsr.Context(0)
    ds = ctx.upload(gsr.gen_synthetic_scene(3, 3_000_000, 1.0, (0.01, 0.05)))
    cam = gsr.orbit_cameras(256, 1920, 1080)[int(sys.argv[3])]
    opt = gsr.RenderOptions(gsr.Backend.tensor, gsr.PrecisionMode.fp32, 2)
    np.save(sys.argv[2], ctx.render(ds, cam, opt).image.rgb)
else:
    a, b = np.load(sys.argv[2]), np.load(sys.argv[3])
    d = np.abs(a.astype(np.float64) - b)
    mse = float((d ** 2).mean())
    psnr = 10 * np.log10(1.0 / mse) if mse > 0 else float("inf")
    print(f"DIFF max_abs {d.max():.3e} psnr {psnr:.1f} dB differing px {(d.max(axis=-1) > 0).sum()}")
