"""Per-CUDA-source-line stall samples and executed instructions from an ncu report captured with
--import-source on (compile with -lineinfo).  Usage: python tools/ncu_lines.py report.ncu-rep [n]"""
import csv
import io
import subprocess
import sys


def main(rep, ntop=40):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    rows, fname, hdr = [], None, None
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
            stalls = {k[6:]: int(v) for k, v in d.items() if k.startswith("stall_") and "Not Issued" not in k
                      and v.isdigit() and int(v) > 0}
            rows.append((s, ins, fname, int(r[0]), r[1].strip()[:70], stalls))
    tot = sum(r[0] for r in rows)
    toti = sum(r[1] for r in rows)
    print(f"total samples {tot}  instructions {toti:.3e}")
    for s, ins, f, ln, src, st in sorted(rows, reverse=True)[:ntop]:
        top = ", ".join(f"{k}={v}" for k, v in sorted(st.items(), key=lambda x: -x[1])[:3])
        print(f"{100*s/tot:5.1f}% {ins/toti*100:5.1f}%i {f}:{ln:<5d} {src:70s} {top}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 40)
