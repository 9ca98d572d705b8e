#!/bin/bash
# A/B of the libps_var_*.so variants: GPU parity tests through each variant, then quick timings
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
cfgs=${1:-"cfg2 cfg3 cfg5"}
: > gpurun_out/ab.txt
for L in paper_2209_06909_b200/libpowersort_b200.so paper_2209_06909_b200/libps_var_*.so; do
  echo "== $L" >> gpurun_out/ab.txt
  ( PS_LIB=$PWD/$L timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -m gpu -x -q 2>&1 | tail -3 ) >> gpurun_out/ab.txt
done
for rep in 1 2; do
for L in paper_2209_06909_b200/libpowersort_b200.so paper_2209_06909_b200/libps_var_*.so; do
  echo "== $L" >> gpurun_out/ab.txt
  PS_LIB=$PWD/$L timeout 600 python tools/quick_time.py $cfgs 2>&1 | grep "count=0" >> gpurun_out/ab.txt
done
done
cat gpurun_out/ab.txt
