#!/bin/bash
# ncu --set full of one big merge_pipe_kernel launch (cfg2 level) for the default library and the variants
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for L in paper_2209_06909_b200/libpowersort_b200.so paper_2209_06909_b200/libps_var_*.so; do
  n=$(basename $L .so)
  PS_LIB=$PWD/$L ncu --set full --import-source on --clock-control none -k regex:merge_pipe_kernel --launch-skip 4 -c 1 -o gpurun_out/pipe_$n python tools/one_sort.py ${1:-cfg2} > /dev/null 2>&1
done
ls gpurun_out/*.ncu-rep
