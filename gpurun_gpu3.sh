export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider --timeout 300 2>&1 | tail -8
timeout 300 python tools/profile_frame.py 3 2>&1 | tail -4
timeout 900 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --quick > gpurun_out/bench_r01c.json 2> gpurun_out/bench_r01c.err; tail -3 gpurun_out/bench_r01c.err; python -c "import json; d=json.load(open('gpurun_out/bench_r01c.json')); print({k: d[k] for k in ('value','raster_ms_per_frame','baseline_raster_ms_per_frame','raster_speedup_vs_cuda_core','stage_ms')})"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:raster_tensor -s 1 -c 1 -o gpurun_out/prof_tensor_r01c python tools/profile_frame.py 2 > gpurun_out/ncu_t.log 2>&1; tail -1 gpurun_out/ncu_t.log
