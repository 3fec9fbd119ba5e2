# One profiling pass for a round tag: stage traffic, bench launch list, ncu captures, bench line.
#   /usr/local/graft/bin/gpurun --timeout 1800 -- 'bash tools/profile_pass.sh r01j'
T=${1:-r01x}
O=gpurun_out/$T
mkdir -p $O
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file $O/frame_metrics.csv python tools/profile_frame.py 3 --backend both > /dev/null 2>&1
python tools/ncu_stage_traffic.py $O/frame_metrics.csv $O/ncu_traffic.json > $O/stage_traffic.txt
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/bench_launches.csv python bench.py --steps 2 --warmup 3 --quick --no-cpu-baseline > /dev/null 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:raster_tensor -s 2 -c 1 -o $O/ncu_raster python tools/profile_frame.py 3 --backend tensor > /dev/null 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:cols_place -s 2 -c 1 -o $O/ncu_cols_place python tools/profile_frame.py 3 --backend tensor > /dev/null 2>&1
python bench.py > $O/bench.json 2> $O/bench.err
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
ls $O
