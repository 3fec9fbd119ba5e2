"""Debug helper: render the single-splat scene of test_single_opaque_splat_center per backend."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_17855_b200 import gsr
cam = gsr.make_camera(256, 256); cam.focal_x = cam.focal_y = 100.0
g = gsr.Gaussian3D(mean=(0, 0, 10), scale=(1, 1, 1), opacity=1.0, sh_dc=(0, 0, 0))
for backend, group in [(int(a), int(b)) for a, b in (x.split(':') for x in sys.argv[1:])]:
    t = time.time()
    print("start", backend, group, flush=True)
    res = gsr.render([g], cam, gsr.RenderOptions(gsr.Backend(backend), gsr.PrecisionMode.fp32, group))
    print("done", backend, group, res.image.pixel(128, 128), f"{time.time()-t:.2f}s", flush=True)
