#!/usr/bin/env python3
"""Benchmark of the B200-native forward render path (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
    python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 bench.py --gpus N ...

Workload (BASELINE configs 3 + 5): the 3M-splat synthetic scene (reference generator, seed 3,
scales 0.01-0.05), 1920x1080, tensorized grouped rasterizer G=2 fp32, cameras from the 256-camera
orbit.  A step = one full frame per rank (preprocess -> bin -> sort -> raster);
rank r renders orbit camera (step*N + r) mod 256.  Per-GPU work is fixed as N grows ("weak"),
frames are independent (camera-batch partitioning, no collective on the data path); value =
frames rendered by all ranks / max-over-ranks device time.

Also reported (JSON keys): per-stage ms, raster ms/frame of the tensor kernel and of the in-repo
CUDA-core baseline kernel (G=1) on the same frames, e2e through the C ABI with host buffers,
roofline of the dominant kernel, the reference's CPU path timed on this host (cpu_baseline).
`--impl reference` times the reference's own CPU implementation (oracle/_ref built from
/root/reference/proj/src) on a bounded sample per step (one 1/8 band of the frame).
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "frames/sec & raster ms/frame @1080p 3M Gaussians; tensor-pipe util; multi-view fps 1–8 GPU"
W, H, N_SPLATS, SEED = 1920, 1080, 3_000_000, 3
N_CAMS = 256
LANES = int(os.environ.get("TGS_BENCH_LANES", "3"))  # frames in flight per GPU (one context/stream each), as tgs_render_batch pipelines


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled while the timed region runs."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.samples = []
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                     timeout=5).stdout.strip()
                if out:
                    self.samples.append([x.strip() for x in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4)
                          if len(s) > 4 + i and s[4 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples)}


def cpu_reference_sample(rec, cam_ns, group, backend, band_index, n_bands=8):
    """One bounded sample of the reference's CPU path: a band of ~1/n_bands of the group rows,
    through the reference's stage API (project_scene over all splats, then build_group_entries /
    sort_entries / rasterize_* on the band).  Returns (frame_fraction, seconds, stage ms)."""
    from oracle.oracle import Ref
    ref = Ref()
    tiles_y = (cam_ns.height + 15) // 16
    groups_y = (tiles_y + group - 1) // group
    rows = [round(i * groups_y / n_bands) for i in range(n_bands + 1)]
    g0, g1 = rows[band_index % n_bands], rows[band_index % n_bands + 1]
    y0, y1 = g0 * group * 16, min(cam_ns.height, g1 * group * 16)
    workers = ref.hardware_concurrency()
    t0 = time.perf_counter()
    _, ms = ref.time_stages(rec, cam_ns, band_y0=y0, band_h=y1 - y0, backend=backend, group_size=group,
                            workers=workers)
    dt = time.perf_counter() - t0
    return (y1 - y0) / cam_ns.height, dt, ms, workers


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return 0
    from oracle.oracle import Ref
    from paper_2605_17855_b200.gsr import orbit_cameras
    from types import SimpleNamespace
    if not Ref.available():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/libgsr_ref.so not built "
                          "(needs /root/reference at build time)"}))
        return 0
    ref = Ref()
    rec = ref.gen_scene(SEED, N_SPLATS, 1.0, 0.01, 0.05, 0)
    cams = orbit_cameras(N_CAMS, W, H)
    fracs, secs = [], []
    workers = 1
    for i in range(args.warmup + args.steps):
        c = cams[i % N_CAMS]
        cns = SimpleNamespace(view=c.view, focal_x=c.focal_x, focal_y=c.focal_y, width=W, height=H,
                              near=c.near, far=c.far)
        frac, dt, ms, workers = cpu_reference_sample(rec, cns, 2, 1, i)
        if i >= args.warmup:
            fracs.append(frac)
            secs.append(dt)
    value = sum(fracs) / sum(secs)
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "frames/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000 * sum(secs) / len(secs),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic (reference generator, seed 3)",
        "config": {"workload": "C3/C5: 3M splats, 1920x1080, orbit cameras, tensor G=2 fp32 "
                   "(reference CPU path; each step one 1/8 band of a frame)", "global_batch": 1,
                   "seq_len": 0, "parallelism": "cpu"},
        "cpu_baseline": {"value": value, "unit": "frames/s", "cores": workers, "kind": "reference",
                         "sample": "per step one 1/8-height band of a 3M/1080p frame: project_scene on all "
                                   "splats + build_group_entries/sort_entries/rasterize_groups_tensor on the band"},
        "e2e": {"value": value, "unit": "frames/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--quick", action="store_true", help="skip e2e/baseline extras (profiling runs)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    if args.impl == "reference":
        return run_reference(args)

    rank, world, local = dist_env()
    import torch
    import torch.distributed as dist
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    from paper_2605_17855_b200 import gsr, _lib
    ctx = gsr.Context(local)
    scene = gsr.gen_synthetic_scene(SEED, N_SPLATS, 1.0, (0.01, 0.05))
    ds = ctx.upload(scene)
    cams = gsr.orbit_cameras(N_CAMS, W, H)
    opt_t = gsr.RenderOptions(gsr.Backend.tensor, gsr.PrecisionMode.fp32, 2)
    opt_s = gsr.RenderOptions(gsr.Backend.scalar, gsr.PrecisionMode.fp32, 1)
    stream = torch.cuda.ExternalStream(ctx.stream, device=torch.device("cuda", local))

    # capacity sizing over every camera this rank will render (untimed), then warm-up
    from paper_2605_17855_b200 import multigpu
    mine = [cams[c] for c in multigpu.camera_schedule(N_CAMS, world, rank, args.warmup + args.steps)]
    for c in {id(c): c for c in mine}.values():
        ctx.enqueue(ds, c, opt_t)
        ctx.sync()
    for i in range(args.warmup):
        ctx.enqueue(ds, mine[i], opt_t)
    ctx.sync()

    # ---- timed region: K frames on this rank, pipelined over LANES contexts (one stream each,
    # camera i on lane i % LANES, like tgs_render_batch), CUDA events on every lane's stream ------
    lanes = [ctx] + [gsr.Context(local) for _ in range(LANES - 1)]
    lane_ds = [ds] + [c.upload(scene) for c in lanes[1:]]
    lane_streams = [torch.cuda.ExternalStream(c.stream, device=torch.device("cuda", local)) for c in lanes]
    for k, c in enumerate(lanes[1:], 1):  # capacity sizing + schedule warm-up of the extra lanes
        for i in range(args.warmup):
            c.enqueue(lane_ds[k], mine[i], opt_t)
            c.sync()
    ev0 = [torch.cuda.Event(enable_timing=True) for _ in lanes]
    ev1 = [torch.cuda.Event(enable_timing=True) for _ in lanes]
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        for e, s in zip(ev0, lane_streams):
            e.record(s)
        for i in range(args.steps):
            k = i % LANES
            lanes[k].enqueue(lane_ds[k], mine[args.warmup + i], opt_t)
        for e, s in zip(ev1, lane_streams):
            e.record(s)
        st_last = ctx.sync()
        for c in lanes[1:]:
            c.sync()
        torch.cuda.synchronize()
    ms_local = max(ev0[0].elapsed_time(e) for e in ev1)
    ms = multigpu.max_over_ranks(ms_local, device=torch.device("cuda", local))
    if world > 1:
        dist.barrier()
    frames = args.steps * world
    value = frames / (ms / 1000.0)

    # ---- per-stage ms (synced frames; the pipeline's own CUDA events), tensor vs baseline ----
    def stage_profile(opt, n=8):
        rows = []
        for i in range(n):
            ctx.enqueue(ds, mine[args.warmup + i % args.steps], opt)
            s = ctx.sync()
            rows.append((s.ms_preprocess, s.ms_binning, s.ms_sort, s.ms_raster, s.ms_total, s.entries))
        med = [statistics.median(r[k] for r in rows) for k in range(6)]
        return {"preprocess": med[0], "binning": med[1], "sort": med[2], "raster": med[3], "total": med[4],
                "entries": int(med[5])}

    st_t = stage_profile(opt_t)
    st_s = stage_profile(opt_s)
    speedup = st_s["raster"] / st_t["raster"] if st_t["raster"] > 0 else None
    # the same comparison with the tile cull off in both rasterisers (the reference's 3-sigma-square
    # work): isolates the tensorised contraction from the cull, which helps the per-pixel baseline more
    ctx.set_tile_cull(False)
    st_t_nc = stage_profile(opt_t)
    st_s_nc = stage_profile(opt_s)
    ctx.set_tile_cull(True)
    speedup_nc = st_s_nc["raster"] / st_t_nc["raster"] if st_t_nc["raster"] > 0 else None

    # ---- walked / contributing pairs of the tensor frames (oracle-equivalent counting pass) --
    ctx.enqueue(ds, mine[args.warmup], opt_t)
    ctx.sync()
    walked, blended = ctx.count_pairs()

    # ---- roofline of the dominant kernel ----------------------------------------------------
    peaks = {}
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        pass
    hbm = float(peaks.get("hbm_gbs", 6650.0))
    tflops = float(peaks.get("bf16_tflops", 1590.0))
    peak_src = "measured" if peaks else "fallback"
    stages = {k: st_t[k] for k in ("preprocess", "binning", "sort", "raster")}
    dom = max(stages, key=stages.get)
    n_vis = int(st_last.visible)
    ent = st_t["entries"]
    # algorithmic bytes per launch of each HBM-bound stage: preprocess reads the
    # 56-B SH0 record and writes the 64-B projected record (+ rect, key, value); the depth presort
    # moves (key, value) pairs 4 times; binning writes every 4-B list entry once and reads the
    # rank-ordered rect (8 B) twice plus the rank->index map (4 B)
    alg_bytes = {"preprocess": (56 + 64) * N_SPLATS, "sort": 4 * 16 * n_vis, "binning": 4 * ent + 20 * n_vis}
    traffic = None
    try:
        traffic = json.load(open(os.path.join(ROOT, "profiles", "r01", "ncu_traffic.json"))).get(dom)
    except Exception:
        pass
    if dom == "raster":
        # tensor pipe: 12 useful flops per walked (pixel, splat) pair (6-term contraction)
        achieved = 12.0 * walked / (st_t["raster"] / 1e3) / 1e12
        roof = {"bound": "tensor", "achieved": achieved, "peak": tflops, "unit": "TFLOP/s",
                "frac": achieved / tflops, "traffic": traffic, "kernel": "raster_tensor_kernel<4>",
                "algorithmic": "12 flops per walked pixel-splat pair (6-term contraction)"}
    else:
        achieved = alg_bytes[dom] / (stages[dom] / 1e3) / 1e9
        roof = {"bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s", "frac": achieved / hbm,
                "traffic": traffic, "kernel": {"binning": "rows_count/place + cols_count/place + scans",
                                               "sort": "depth presort (digit histograms + 4 one-sweep passes)",
                                               "preprocess": "preprocess_kernel"}[dom],
                "algorithmic_bytes": alg_bytes[dom]}
    roof["peak_source"] = peak_src
    # raster pipes (the kernel the paper targets): FP32 / MUFU work per the survey's model
    sm_mhz = clk.summary().get("sm_mhz") or 1965.0
    lanes = 148 * 128 * sm_mhz * 1e6
    fp32_ops = 8.0 * blended + 2.0 * walked
    raster_pipes = {
        "walked_pairs": walked, "blended_pairs": blended,
        "fp32_frac": fp32_ops / (st_t["raster"] / 1e3) / lanes,
        "mufu_frac": blended / (st_t["raster"] / 1e3) / (148 * 16 * sm_mhz * 1e6),
        "tensor_frac": 32.0 * walked / (st_t["raster"] / 1e3) / (tflops * 1e12),
    }

    # ---- e2e through the C ABI with host buffers (gsr::render call shape) --------------------
    e2e = None
    if not args.quick:
        lib = _lib.load()
        rec = torch.from_numpy(scene.records).pin_memory()
        out = torch.empty((H, W, 3), dtype=torch.float32).pin_memory()
        import ctypes as C
        st = _lib.tgs_stats()
        n_e2e = max(3, min(args.steps, 10))
        oc = opt_t.to_c()
        for i in range(2):
            lib.tgs_render_records(ctx.h, C.cast(rec.data_ptr(), _lib.F32P), len(scene), 0,
                                   C.byref(mine[i].to_c()), C.byref(oc), C.cast(out.data_ptr(), _lib.F32P),
                                   C.byref(st))
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for i in range(n_e2e):
            rc = lib.tgs_render_records(ctx.h, C.cast(rec.data_ptr(), _lib.F32P), len(scene), 0,
                                        C.byref(mine[args.warmup + i % args.steps].to_c()), C.byref(oc),
                                        C.cast(out.data_ptr(), _lib.F32P), C.byref(st))
            assert rc == 0, _lib.last_error()
        dt = multigpu.max_over_ranks(time.perf_counter() - t0, device=torch.device("cuda", local))
        e2e = {"value": n_e2e * world / dt, "unit": "frames/s",
               "h2d_bytes_per_step": int(scene.records.nbytes + 88),
               "d2h_bytes_per_step": int(W * H * 3 * 4),
               "api": "tgs_render_records (scene records + camera in, RGB float image out; pinned host buffers)"}

    # ---- CPU baseline: the reference's own CPU path on this host (rank 0, N=1) ---------------
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline and not args.quick:
        try:
            from oracle.oracle import Ref
            from types import SimpleNamespace
            if Ref.available():
                c = mine[args.warmup]
                cns = SimpleNamespace(view=c.view, focal_x=c.focal_x, focal_y=c.focal_y, width=W, height=H,
                                      near=c.near, far=c.far)
                fr, sec, nb = 0.0, 0.0, 0
                workers = 1
                while sec < 10.0 and nb < 8:
                    f, dt, _, workers = cpu_reference_sample(scene.records, cns, 2, 1, nb)
                    fr += f
                    sec += dt
                    nb += 1
                cpu = {"value": fr / sec, "unit": "frames/s", "cores": workers, "kind": "reference",
                       "sample": f"{nb} of 8 horizontal bands of one 3M/1080p frame (G=2 tensor fp32) "
                                 "through the reference stage API (oracle/_ref), ~10 s of CPU work"}
        except Exception as e:  # reported, never fatal for the GPU number
            cpu = {"value": None, "unit": "frames/s", "cores": 0, "kind": "reference", "sample": f"failed: {e}"}

    # our kernels per frame: preprocess 1; depth presort: digit histograms + 4 one-sweep passes;
    # binning: rows count (with the rank gather), scan,
    # rows meta, rows place, cols count, scan, offsets, cols place; unit order 1; raster 1
    launches_per_frame = 1 + 5 + 8 + 1 + 1
    line = {
        "metric": METRIC, "value": value, "unit": "frames/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f32 (fp16 hi/lo tensor-core contraction)",
        "data": "synthetic (reference generator gen_synthetic_scene seed 3, scales 0.01-0.05)",
        "config": {"workload": "C3/C5: 3M splats, 1920x1080, 256-camera orbit, one frame per rank per step, "
                               "tensor G=2 fp32 mode", "global_batch": world, "seq_len": 0,
                   "parallelism": f"camera-batch x{world}, {LANES} frames in flight per GPU", "l2": "inputs > L2 (scene 168 MB + lists >= 240 MB)"},
        "raster_ms_per_frame": st_t["raster"], "baseline_raster_ms_per_frame": st_s["raster"],
        "raster_speedup_vs_cuda_core": speedup,
        "raster_no_tile_cull": {"tensor_ms": st_t_nc["raster"], "cuda_core_ms": st_s_nc["raster"],
                                "speedup": speedup_nc},
        "stage_ms": st_t, "baseline_stage_ms": st_s,
        "roofline": roof, "raster_pipes": raster_pipes,
        "cpu_baseline": cpu, "e2e": e2e,
        "clocks": clk.summary(), "gpu_launches": launches_per_frame * args.steps,
    }
    if rank == 0:
        print(json.dumps(line))
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
