"""Summarise an ncu report: duration, issue efficiency, pipe utilisation, stall reasons, the
instruction mix and the top stall sites.  Usage: python tools/ncu_summary.py report.ncu-rep [n]"""
import collections
import csv
import io
import subprocess
import sys


def page(rep, *args):
    out = subprocess.run(["ncu", "-i", rep, *args, "--csv"], capture_output=True, text=True).stdout
    return list(csv.reader(io.StringIO(out)))


def main(rep, ntop=12):
    raw = page(rep, "--page", "raw")
    hdr, vals = raw[0], raw[2]
    d = dict(zip(hdr, vals))
    keys = ["gpu__time_duration.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
            "sm__warps_active.avg.pct_of_peak_sustained_active",
            "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
            "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
            "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
            "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
            "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_sector_hit_rate.pct",
            "launch__registers_per_thread", "launch__grid_size", "launch__block_size"]
    for k in keys:
        print(f"{k:70s} {d.get(k)}")
    st = []
    for h, v in zip(hdr, vals):
        if h.startswith("smsp__average_warps_issue_stalled_") and h.endswith("per_issue_active.ratio"):
            try:
                st.append((float(v), h[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]))
            except ValueError:
                pass
    print("stalls per issue:", ", ".join(f"{n}={v:.2f}" for v, n in sorted(st, reverse=True) if v > 0.05))
    src = page(rep, "--page", "source", "--print-source", "sass")
    sh = src[1]
    ix = {h: i for i, h in enumerate(sh)}
    rows = src[2:]

    def f(r, k):
        try:
            return float(r[ix[k]])
        except (ValueError, KeyError):
            return 0.0

    cnt, smp = collections.Counter(), collections.Counter()
    for r in rows:
        toks = r[1].split()
        op = toks[1] if toks and toks[0].startswith("@") else (toks[0] if toks else "?")
        cnt[op] += f(r, "Instructions Executed")
        smp[op] += f(r, "Warp Stall Sampling (All Samples)")
    tot = sum(cnt.values())
    print(f"executed warp-instructions {tot:.4g}; stall samples {sum(smp.values()):.0f}")
    for op, c in cnt.most_common(ntop):
        print(f"  {op:34s} {c:12.0f} {100 * c / tot:5.1f}%  samples {smp[op]:.0f}")
    print("top stall sites:")
    for r in sorted(rows, key=lambda r: -f(r, "Warp Stall Sampling (All Samples)"))[:ntop]:
        rs = sorted(((f(r, k), k[6:]) for k in sh if k.startswith("stall_") and "Not Issued" not in k),
                    reverse=True)[:3]
        print(f"  {r[0][-5:]} {r[1][:56]:56s} {f(r, 'Warp Stall Sampling (All Samples)'):6.0f} "
              + " ".join(f"{n}={v:.0f}" for v, n in rs if v > 0))


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 12)
