"""north_star (4) evidence: each Gaussian is gathered ONCE per 2x2 group, not once per member tile.

Renders the C3 bench frame (3M splats, 1080p, orbit camera 5) with the tensor rasteriser and reports
* ReuseReport (reference load_reduction, metrics.cpp:45-57): N_group group entries vs N_total tile
  appearances — the loads a per-tile rasteriser would make;
* OpReport of the frame: chunks / rows the producer actually staged (each staged row = one gather of
  one splat for a whole group);
* gathered rows per group entry walked and per tile appearance walked.
The DRAM / L2 side comes from the ncu capture of the same kernel (tools/profile_pass.sh).

    python tools/reuse_evidence.py > profiles/r02/reuse_evidence_<tag>.txt
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_17855_b200 import gsr  # noqa: E402


def main():
    ctx = gsr.Context(0)
    ds = ctx.upload(gsr.gen_synthetic_scene(3, 3_000_000, 1.0, (0.01, 0.05)))
    cam = gsr.orbit_cameras(256, 1920, 1080)[5]
    opt = gsr.RenderOptions(gsr.Backend.tensor, gsr.PrecisionMode.fp32, 2)
    for _ in range(3):
        res = ctx.render(ds, cam, opt)
    rep = ctx.reuse_report()
    ops = res.ops
    rows = ops.used_lanes // (128 * 12)  # rows carried by MMAs (each row counted per member-tile MMA pair)
    print(f"entries (N_group) {rep['n_group']}  tile appearances (N_total) {rep['n_total']}  "
          f"load_reduction {rep['load_reduction']:.4f}")
    print(f"chunks staged {ops.chunk_loads}  MMAs {ops.fragment_ops // 16}  "
          f"rows carried by MMAs {rows}  skipped (tile,row) pairs {ops.skipped_pairs}")
    print(f"per-tile loading would gather {rep['n_total']} records; the grouped kernel stages each kept "
          f"splat once per group: at most {rep['n_group']} gathers (entries walked before retirement "
          f"and culled rows are fewer)")
    print(f"mask popcount histogram {rep['mask_popcount_hist'][:5]}")


if __name__ == "__main__":
    main()
