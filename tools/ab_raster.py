"""A/B timing of rasterizer variants on the bench workload (C3: 3M splats, 1080p, G=2, orbit
camera 5): prints the median stage times over N frames and saves the image so variants can be
compared bit for bit.  Variants are selected by env (TGS_LIB, TGS_RASTER_VARIANT).

    python tools/ab_raster.py TAG [frames] [--group G] [--backend tensor|scalar]
"""
import argparse
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_17855_b200 import gsr  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("tag")
    ap.add_argument("frames", type=int, nargs="?", default=20)
    ap.add_argument("--group", type=int, default=2)
    ap.add_argument("--backend", default="tensor")
    ap.add_argument("--cam", type=int, default=5)
    ap.add_argument("--save", action="store_true", help="save the image to gpurun_out/ab_TAG.npy")
    ap.add_argument("--hash", action="store_true", help="print a digest of the image bytes (bit-identity checks)")
    a = ap.parse_args()
    ctx = gsr.Context(0)
    ds = ctx.upload(gsr.gen_synthetic_scene(3, 3_000_000, 1.0, (0.01, 0.05)))
    cam = gsr.orbit_cameras(256, 1920, 1080)[a.cam]
    opt = gsr.RenderOptions(gsr.Backend[a.backend], gsr.PrecisionMode.fp32, a.group)
    rows = []
    for _ in range(3 + a.frames):
        ctx.enqueue(ds, cam, opt)
        st = ctx.sync()
        rows.append((st.ms_preprocess, st.ms_sort, st.ms_binning, st.ms_raster, st.ms_total))
    med = np.median(np.array(rows[3:]), axis=0)
    if a.save:
        img = ctx.render(ds, cam, opt).image.rgb
        os.makedirs("gpurun_out", exist_ok=True)
        np.save(f"gpurun_out/ab_{a.tag}.npy", img)
    if a.hash:
        import hashlib
        img = ctx.render(ds, cam, opt).image.rgb
        print(f"HASH {a.tag}: {hashlib.sha256(np.ascontiguousarray(img).tobytes()).hexdigest()[:16]}", flush=True)
    print(f"AB {a.tag}: pre {med[0]:.3f} sort {med[1]:.3f} bin {med[2]:.3f} raster {med[3]:.3f} "
          f"total {med[4]:.3f} ms", flush=True)


if __name__ == "__main__":
    main()
