"""Tile trip statistics of a C3 frame (3M splats, 1080p): entries walked per tile until its last
pixel terminates, vs the tile's list length."""
import ctypes as C, os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_17855_b200 import gsr, _lib
ctx = gsr.Context(0)
ds = ctx.upload(gsr.gen_synthetic_scene(3, 3_000_000, 1.0, (0.01, 0.05)))
for cam_name, cam in [("identity", gsr.make_camera(1920, 1080)), ("orbit5", gsr.orbit_cameras(256, 1920, 1080)[5])]:
    for g in (1, 2):
        ctx.render(ds, cam, gsr.RenderOptions(gsr.Backend.scalar if g == 1 else gsr.Backend.tensor, group_size=g))
        n = C.c_int64()
        lib = ctx.lib
        lib.tgs_tile_trips(ctx.h, None, 0, C.byref(n))
        trips = np.zeros(n.value, np.uint32)
        assert lib.tgs_tile_trips(ctx.h, trips.ctypes.data, n.value, C.byref(n)) == 0
        w, b = ctx.count_pairs()
        q = np.percentile(trips, [50, 90, 99, 99.9, 100])
        print(f"{cam_name} G={g}: tiles {len(trips)} trip mean {trips.mean():.0f} p50/90/99/99.9/max {q.astype(int).tolist()}"
              f" sum {trips.sum()/1e6:.1f}M walked {w/1e6:.0f}M blended {b/1e6:.0f}M", flush=True)
        top = np.argsort(trips)[-6:]
        print("   longest tiles (tx,ty,trip):", [(int(t % 120), int(t // 120), int(trips[t])) for t in top])
        h, e = np.histogram(np.log2(trips + 1), bins=range(0, 18))
        print("   log2 hist:", h.tolist())
