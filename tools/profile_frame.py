"""Render a few C3 frames (3M splats, 1080p) for ncu: tensor G=2 then CUDA-core baseline G=1.

    ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file launches.csv \
        python tools/profile_frame.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2605_17855_b200 import gsr  # noqa: E402


def main(frames=3):
    ctx = gsr.Context(0)
    ds = ctx.upload(gsr.gen_synthetic_scene(3, 3_000_000, 1.0, (0.01, 0.05)))
    cam = gsr.make_camera(1920, 1080)
    for backend, group in ((gsr.Backend.tensor, 2), (gsr.Backend.scalar, 1)):
        opt = gsr.RenderOptions(backend, gsr.PrecisionMode.fp32, group)
        for _ in range(frames):
            ctx.enqueue(ds, cam, opt)
            st = ctx.sync()
        print(backend.name, group, "entries", st.entries, "stage ms", st.ms_preprocess, st.ms_binning,
              st.ms_sort, st.ms_raster, st.ms_total, flush=True)


if __name__ == "__main__":
    main(int(sys.argv[1]) if len(sys.argv) > 1 else 3)
