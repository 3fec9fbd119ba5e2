"""Build a variant of libtgs.so with extra nvcc flags on one source (A/B experiments).

    python tools/build_variant.py NAME tgs_raster_tensor.cu -DTGS_RASTER_N=16 -DTGS_RASTER_TS=4
    TGS_LIB=paper_2605_17855_b200/variants/libtgs_NAME.so python tools/profile_frame.py ...

The other objects come from the regular in-tree build (paper_2605_17855_b200/_obj)."""
import glob
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_17855_b200 import build as B  # noqa: E402


def main():
    name, srcs, *extra = sys.argv[1:]
    srcs = srcs.split(",")  # one or more sources (comma-separated) rebuilt with the extra flags
    B.build()
    out_dir = os.path.join(B.HERE, "variants")
    os.makedirs(out_dir, exist_ok=True)
    vobjs = []
    for src in srcs:  # a source may be an absolute path (e.g. an older revision of a csrc file)
        obj = os.path.join(out_dir, f"{name}_{os.path.basename(src)}.o")
        cmd = [B.NVCC, *B.ARCH, *B.NVFLAGS, "-I", B.CSRC, *extra, "-c", os.path.join(B.CSRC, src), "-o", obj]
        subprocess.run(cmd, check=True)
        vobjs.append(obj)
    names = {os.path.basename(s) for s in srcs}
    objs = [o for o in sorted(glob.glob(os.path.join(B.OBJ, "*.o"))) if os.path.basename(o)[:-2] not in names]
    lib = os.path.join(out_dir, f"libtgs_{name}.so")
    subprocess.run([B.NVCC, *B.ARCH, "-shared", "-o", lib, *vobjs, *objs, "-lcudart"], check=True)
    print(lib)


if __name__ == "__main__":
    main()
