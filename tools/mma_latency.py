"""tcgen05.mma (M=128, K=16, A/B from shared memory) issue rate and group latency in isolation:
n MMAs, a commit every `per` MMAs, optionally waiting for each commit (latency of a group).
python tools/mma_latency.py"""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from tools.debug.build import load  # noqa: E402


def main():
    lib = load()
    for ncols in (16, 32, 64):
        for per, wait in ((8, 0), (8, 1), (1, 1)):
            n = 4096
            cyc = C.c_longlong()
            variant = 4 << 16  # warp-uniform elected issue, as the rasteriser
            rc = lib.tgs_debug_mma_rate(n, variant | per, wait, ncols, C.byref(cyc))
            assert rc == 0
            print(f"MMA N={ncols:2d} commit every {per} wait={wait}: {cyc.value / n:7.1f} cycles per MMA "
                  f"({cyc.value / n * per:8.1f} per group)", flush=True)


if __name__ == "__main__":
    main()
