# One profiling pass for a round tag: stage traffic, bench launch list, ncu captures of the top
# kernels (raster, group placement, preprocess, one-sweep), reuse evidence, bench line, smoke.
#   /usr/local/graft/bin/gpurun --timeout 2400 -- 'bash tools/profile_pass.sh r02x'
T=${1:-r02x}
O=gpurun_out/$T
mkdir -p $O
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file $O/frame_metrics.csv python tools/profile_frame.py 3 --backend both > /dev/null 2>&1
python tools/ncu_stage_traffic.py $O/frame_metrics.csv $O/ncu_traffic.json > $O/stage_traffic.txt
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/bench_launches.csv python bench.py --steps 2 --warmup 3 --quick --no-cpu-baseline > /dev/null 2>&1
for k in raster_tensor cols_place preprocess onesweep; do
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:$k -s 2 -c 1 -o $O/ncu_$k python tools/profile_frame.py 3 --backend tensor > /dev/null 2>&1
done
python tools/reuse_evidence.py > $O/reuse_evidence.txt 2>&1
python bench.py > $O/bench.json 2> $O/bench.err
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
ls $O
