"""Per-chunk latency of the producer -> MMA -> epilogue hand-off (no blending work)."""
import ctypes as C, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from tools.debug.build import load
lib = load()
for mode in range(8):
    cyc = C.c_longlong()
    n = 4000
    assert lib.tgs_debug_pipeline(n, mode, C.byref(cyc)) == 0
    print(f"mode {mode} (mma={mode&1} ld={mode>>1&1} fence={mode>>2&1}): {cyc.value / n:8.1f} cycles/chunk")
for variant, name in ((0, "SS none"), (4, "SS elect"), (1, "A in TMEM"), (2, "SS swz32")):
    for ncols in (16, 32, 64):
        for per, wait in ((1, 1), (8, 0), (64, 0)):
            cyc = C.c_longlong()
            n = 2048
            assert lib.tgs_debug_mma_rate(n, per | (variant << 16), wait, ncols, C.byref(cyc)) == 0
            print(f"{name:10s} N={ncols} commit every {per} wait={wait}: {cyc.value / n:8.1f} cycles/mma", flush=True)
