"""Executed warp-instructions and stall samples of the tensor rasterizer per warp role, from an
ncu report captured with --import-source on (-lineinfo): source lines of raster_tensor_kernel are
attributed to the producer / MMA / epilogue branches by the line ranges given on the command line.

    python tools/ncu_roles.py report.ncu-rep producer=401-723 mma=724-808 epilogue=809-1010
"""
import csv
import io
import subprocess
import sys


def main(rep, ranges):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    roles = {}
    for spec in ranges:
        name, rng = spec.split("=")
        a, b = (int(x) for x in rng.split("-"))
        roles[name] = (a, b)
    tot = {k: [0, 0] for k in list(roles) + ["other"]}
    fname, hdr = None, None
    for r in csv.reader(io.StringIO(out)):
        if not r:
            continue
        if r[0] == "File Path":
            fname = r[1].split("/")[-1]
        elif r[0] == "Line No":
            hdr = r
        elif hdr and r[0].isdigit() and len(r) == len(hdr) and r[2] == "-":
            d = dict(zip(hdr[4:], r[4:]))
            s = int(d.get("Warp Stall Sampling (All Samples)", "0") or 0)
            ins = int(d.get("Instructions Executed", "0") or 0)
            ln = int(r[0])
            key = "other"
            if fname and fname.startswith("tgs_raster_tensor"):
                for k, (a, b) in roles.items():
                    if a <= ln <= b:
                        key = k
            tot[key][0] += ins
            tot[key][1] += s
    ti = sum(v[0] for v in tot.values()) or 1
    ts = sum(v[1] for v in tot.values()) or 1
    for k, (i, s) in tot.items():
        print(f"{k:10s} instructions {i:12.4e} ({100 * i / ti:5.1f}%)  stall samples {s:8d} ({100 * s / ts:5.1f}%)")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2:])
