"""Build tools/debug/libtgs_debug.so (TOOLS ONLY: tcgen05 microbenchmarks, not the product ABI).

    python tools/debug/build.py
    from tools.debug.build import load; lib = load()
"""
import ctypes as C
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
LIB = os.path.join(HERE, "libtgs_debug.so")
SRC = os.path.join(HERE, "tgs_debug.cu")


def build(force: bool = False) -> str:
    sys.path.insert(0, ROOT)
    from paper_2605_17855_b200 import build as b
    deps = [SRC, os.path.join(HERE, "tgs_debug.h")] + [os.path.join(b.CSRC, f) for f in os.listdir(b.CSRC)]
    if not force and os.path.exists(LIB) and all(os.path.getmtime(d) <= os.path.getmtime(LIB) for d in deps):
        return LIB
    cmd = [b.NVCC, *b.ARCH, "-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC", "--expt-relaxed-constexpr",
           "-shared", SRC, "-o", LIB, "-lcudart"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("nvcc failed on tools/debug/tgs_debug.cu")
    return LIB


def load():
    path = build()
    lib = C.CDLL(path)
    P = C.c_void_p
    lib.tgs_debug_mma.argtypes = [P, P, P]
    lib.tgs_debug_pipeline.argtypes = [C.c_int, C.c_int, C.POINTER(C.c_longlong)]
    lib.tgs_debug_mma_rate.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, C.POINTER(C.c_longlong)]
    for f in (lib.tgs_debug_mma, lib.tgs_debug_pipeline, lib.tgs_debug_mma_rate):
        f.restype = C.c_int
    return lib


if __name__ == "__main__":
    print(build(force=True))
