# ncu captures of the binning kernels (one launch each, third frame)
T=${1:-r02x}
O=gpurun_out/$T
mkdir -p $O
for k in ${KERNELS:-cols_place rows_place cols_count rows_count}; do
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:$k -s 2 -c 1 -o $O/ncu_$k python tools/profile_frame.py 3 --backend tensor > /dev/null 2>&1
done
ls $O
