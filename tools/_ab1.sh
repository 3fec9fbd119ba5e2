mkdir -p gpurun_out/r02c
for n in pf4 spw2 spw2pf4; do
 TGS_LIB=paper_2605_17855_b200/variants/libtgs_$n.so timeout 300 python tools/ab_raster.py $n 20 >> gpurun_out/r02c/ab.txt 2>&1
 TGS_LIB=paper_2605_17855_b200/variants/libtgs_${n}_prof.so timeout 300 python tools/ab_raster.py ${n}_prof 1 2>&1 | grep -E "RPROF|AB|RUNIT" | head -4 >> gpurun_out/r02c/ab.txt
done
timeout 300 python tools/ab_raster.py base 20 >> gpurun_out/r02c/ab.txt 2>&1
cat gpurun_out/r02c/ab.txt
