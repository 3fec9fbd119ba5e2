"""Per-launch table from an ncu --csv --log-file launch list (last N launches).
Usage: python tools/launch_table.py launches.csv [N]"""
import collections
import csv
import sys


def main(path, last=40):
    lines = [l for l in open(path) if l.startswith('"')]
    rows = list(csv.DictReader(lines))
    by = collections.OrderedDict()
    for r in rows:
        by.setdefault((int(r["ID"]), r["Kernel Name"]), {})[r["Metric Name"]] = r["Metric Value"]
    items = list(by.items())[-last:]
    tot = 0.0
    for (i, n), m in items:
        t = float(m.get("gpu__time_duration.sum", 0)) / 1000
        tot += t
        extra = " ".join(f"{k.split('__')[1].split('.')[0]}={m[k]}" for k in m if k != "gpu__time_duration.sum")
        print(f"{i:5d} {n.split('(')[0][:48]:48s} {t:9.1f} us  {extra}")
    print(f"sum {tot:.1f} us")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 40)
