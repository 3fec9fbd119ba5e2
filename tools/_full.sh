# full GPU pass: tests, smoke, bench (cameras), bench (bands), 2-rank functional bench on one GPU
T=${1:-full}
O=gpurun_out/$T
mkdir -p $O
timeout 1200 python -m pytest tests -m gpu -x -q > $O/gpu_tests.log 2>&1; tail -3 $O/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; tail -2 $O/smoke.log
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err; tail -2 $O/bench.err
timeout 600 python bench.py --mode bands --steps 5 --warmup 3 > $O/bench_bands.json 2> $O/bench_bands.err; tail -2 $O/bench_bands.err
TGS_BENCH_BACKEND=gloo timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29531 bench.py --gpus 2 --steps 6 --warmup 3 --quick > $O/bench_2rank.json 2> $O/bench_2rank.err; tail -2 $O/bench_2rank.err
TGS_BENCH_BACKEND=gloo timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29532 bench.py --gpus 2 --mode bands --steps 3 --warmup 3 > $O/bench_bands_2rank.json 2> $O/bench_bands_2rank.err; tail -2 $O/bench_bands_2rank.err
ls -la $O
timeout 900 python bench.py --mode configs --steps 10 --warmup 3 > $O/bench_configs.jsonl 2> $O/bench_configs.err; tail -2 $O/bench_configs.err
