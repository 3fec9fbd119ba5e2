"""Scene/camera cases shared by the golden-fixture generator and the parity tests.

Every scene comes from the reference generator (scene_io.cpp:218-251) with the camera of the
reference tests (testutil.hpp:14-24) or a rotated/translated view like test_projection.cpp:115-146.
"""
from __future__ import annotations

import math
from types import SimpleNamespace

import numpy as np


def make_camera(width, height, focal_scale=0.75):
    return SimpleNamespace(view=np.eye(4, dtype=np.float32), focal_x=focal_scale * width,
                           focal_y=focal_scale * width, width=width, height=height, near=0.2, far=100.0)


def rotated_camera(width, height, yaw_deg=17.0, pitch_deg=-9.0, t=(0.15, -0.1, 0.4)):
    y, p = math.radians(yaw_deg), math.radians(pitch_deg)
    ry = np.array([[math.cos(y), 0, math.sin(y)], [0, 1, 0], [-math.sin(y), 0, math.cos(y)]])
    rx = np.array([[1, 0, 0], [0, math.cos(p), -math.sin(p)], [0, math.sin(p), math.cos(p)]])
    v = np.eye(4, dtype=np.float32)
    v[:3, :3] = (rx @ ry).astype(np.float32)
    v[:3, 3] = np.asarray(t, np.float32)
    return SimpleNamespace(view=v, focal_x=0.7 * width, focal_y=0.72 * width, width=width, height=height,
                           near=0.2, far=100.0)


_R = {
    "scalar_g1": dict(backend=0, group_size=1, mode=0),
    "tensor_g2": dict(backend=1, group_size=2, mode=0),
    "tensor_g4_fp16": dict(backend=1, group_size=4, mode=1),
}

CASES = {
    # SH degree 3, non-multiple-of-16 image, identity view
    "sh3_small": dict(seed=1, count=1000, smin=0.01, smax=0.05, sh_seed=5,
                      camera=lambda: make_camera(100, 72), renders=_R),
    # general rotation + translation, larger splats (many multi-tile entries)
    "rotated": dict(seed=2, count=800, smin=0.02, smax=0.1, sh_seed=0,
                    camera=lambda: rotated_camera(128, 96), renders=_R),
}
