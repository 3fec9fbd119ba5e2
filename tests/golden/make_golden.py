"""Generate tests/golden/*.npz from the REFERENCE ITSELF (oracle/_ref/libgsr_ref.so, built from
/root/reference/proj/src by oracle/Makefile).  Run here, in the container that has
/root/reference:

    make -C oracle ref && python tests/golden/make_golden.py

The fixtures pin both the C restatement (tests/test_oracle.py) and the GPU path
(tests/test_gpu_parity.py) on machines where the reference sources are absent.
"""
from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.abspath(os.path.join(HERE, "..", "..")))

from oracle.oracle import Ref  # noqa: E402
from tests.cases import CASES  # noqa: E402


def main():
    ref = Ref()
    for name, case in CASES.items():
        rec = ref.gen_scene(case["seed"], case["count"], 1.0, case["smin"], case["smax"], case["sh_seed"])
        cam = case["camera"]()
        proj, st3 = ref.project(rec, cam)
        out = {"records": rec, "projected": proj.view(np.uint8), "proj_stats": st3}
        for g in (1, 2, 4):
            ent, off, app = ref.bin_sort(proj, cam.width, cam.height, g)
            out[f"entries_g{g}"] = ent.view(np.uint8)
            out[f"offsets_g{g}"] = off
            out[f"appearances_g{g}"] = np.array([app], np.uint64)
        for tag, opt in case["renders"].items():
            img, stats = ref.render(rec, cam, **opt)
            out[f"img_{tag}"] = img
            out[f"stats_{tag}"] = np.array([stats[k] for k in sorted(stats)], np.uint64)
        path = os.path.join(HERE, f"{name}.npz")
        np.savez_compressed(path, **out)
        print(f"{path}: {len(rec)} splats, {len(proj)} projected, {os.path.getsize(path)} bytes")


if __name__ == "__main__":
    main()
