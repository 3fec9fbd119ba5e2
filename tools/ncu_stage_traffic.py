"""Per-stage DRAM traffic and device time of one tensor G=2 frame from an ncu metrics CSV
(ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --csv ...
 python tools/profile_frame.py 2 --backend tensor).  Writes profiles/<round>/ncu_traffic.json with
the bytes per stage (the `traffic` field bench.py reports beside the roofline) and prints a table.

    python tools/ncu_stage_traffic.py gpurun_out/metrics.csv profiles/r01/ncu_traffic.json
"""
import collections
import csv
import json
import sys

STAGE = {"preprocess_kernel": "preprocess", "hist_kernel": "sort", "scatter_kernel": "sort",
         "digits_kernel": "sort", "onesweep_kernel": "sort",
         "scan_reduce_kernel": "binning", "scan_small_kernel": "binning", "scan_apply_kernel": "binning",
         "scan_onepass_kernel": "binning",
         "rank_gather_kernel": "binning", "rows_count_kernel": "binning", "rows_meta_kernel": "binning",
         "rows_place_kernel": "binning", "cols_count_kernel": "binning", "offsets_kernel": "binning",
         "cols_place_kernel": "binning", "unit_order_kernel": "binning",
         "raster_tensor_kernel": "raster", "raster_scalar_kernel": "raster"}


def frame_stages(order, start, stop):
    stage_of_scan = "sort"
    agg = collections.defaultdict(lambda: [0.0, 0.0, 0.0])
    for l in order[start:stop]:
        base = l["name"].split("(")[0].split("::")[-1].split("<")[0]
        st = STAGE.get(base, "other")
        if base == "rank_gather_kernel":
            stage_of_scan = "binning"
        if st is None:
            st = stage_of_scan
        a = agg[st]
        a[0] += l.get("gpu__time_duration.sum", 0.0) / 1e3
        a[1] += l.get("dram__bytes_read.sum", 0.0)
        a[2] += l.get("dram__bytes_write.sum", 0.0)
    return agg


def main(src, dst):
    rows = [r for r in csv.reader(open(src)) if len(r) > 10 and r[0].isdigit()]
    launches = collections.OrderedDict()
    for r in rows:
        launches.setdefault(int(r[0]), {"name": r[4]})[r[-3]] = float(r[-1].replace(",", ""))
    order = list(launches.values())
    starts = [i for i, l in enumerate(order) if "preprocess_kernel" in l["name"]] + [len(order)]
    # the last frame of each rasteriser (tensor frames feed bench.py's roofline traffic)
    last = {}
    for a, b in zip(starts[:-1], starts[1:]):
        kind = "tensor" if any("raster_tensor" in l["name"] for l in order[a:b]) else "scalar"
        last[kind] = (a, b)
    out = {}
    for kind in ("tensor", "scalar"):
        if kind not in last:
            continue
        agg = frame_stages(order, *last[kind])
        if kind == "tensor":
            out = {k: int(v[1] + v[2]) for k, v in agg.items()}
        print(f"{kind} frame")
        print(f"{'stage':12s} {'us':>10s} {'read MB':>10s} {'write MB':>10s}")
        for k, (us, rd, wr) in agg.items():
            print(f"{k:12s} {us:10.1f} {rd / 1e6:10.1f} {wr / 1e6:10.1f}")
    json.dump(out, open(dst, "w"), indent=1)


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
