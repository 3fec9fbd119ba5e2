"""Render a few C3 frames (3M splats, 1080p) for ncu: tensor G=2 then CUDA-core baseline G=1.

The camera is the bench's first timed orbit camera (orbit index 5 of 256), so launch lists and
ncu captures describe the same frames bench.py times.

    ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file launches.csv \
        python tools/profile_frame.py [frames] [--backend tensor|scalar|both]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2605_17855_b200 import gsr  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("frames", type=int, nargs="?", default=3)
    ap.add_argument("--backend", default="both", choices=["tensor", "scalar", "both"])
    ap.add_argument("--cam", type=int, default=5, help="orbit camera index (-1: identity view)")
    ap.add_argument("--c4", action="store_true", help="BASELINE config 4: 6M splats (seed 4), 3840x2160, identity")
    a = ap.parse_args()
    ctx = gsr.Context(0)
    if a.c4:
        ds = ctx.upload(gsr.gen_synthetic_scene(4, 6_000_000, 1.0, (0.01, 0.05)))
        cam = gsr.make_camera(3840, 2160)
    else:
        ds = ctx.upload(gsr.gen_synthetic_scene(3, 3_000_000, 1.0, (0.01, 0.05)))
        cam = gsr.make_camera(1920, 1080) if a.cam < 0 else gsr.orbit_cameras(256, 1920, 1080)[a.cam]
    runs = []
    if a.backend in ("tensor", "both"):
        runs.append((gsr.Backend.tensor, 2))
    if a.backend in ("scalar", "both"):
        runs.append((gsr.Backend.scalar, 1))
    for backend, group in runs:
        opt = gsr.RenderOptions(backend, gsr.PrecisionMode.fp32, group)
        for _ in range(a.frames):
            ctx.enqueue(ds, cam, opt)
            st = ctx.sync()
        print(backend.name, group, "entries", st.entries, "stage ms", st.ms_preprocess, st.ms_binning,
              st.ms_sort, st.ms_raster, st.ms_total, flush=True)


if __name__ == "__main__":
    main()
