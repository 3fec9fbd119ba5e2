# quick GPU iteration: smoke, GPU tests, A/B timing of the tensor raster (+ PROF role timing)
T=${1:-it}
O=gpurun_out/$T
mkdir -p $O
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 900 python -m pytest tests -m gpu -x -q > $O/gpu_tests.log 2>&1
timeout 300 python tools/ab_raster.py tensor 20 > $O/ab.txt 2>&1
timeout 300 python tools/ab_raster.py scalar 20 --group 1 --backend scalar >> $O/ab.txt 2>&1
TGS_LIB=paper_2605_17855_b200/variants/libtgs_prof.so timeout 300 python tools/ab_raster.py prof 3 2>&1 | grep -E "RPROF|AB" | tail -3 >> $O/ab.txt
tail -3 $O/smoke.log; tail -3 $O/gpu_tests.log; cat $O/ab.txt
for v in $VARIANTS; do TGS_LIB=paper_2605_17855_b200/variants/libtgs_$v.so timeout 300 python tools/ab_raster.py $v 20 2>&1 | grep AB >> $O/ab.txt; done
cat $O/ab.txt | tail -8
