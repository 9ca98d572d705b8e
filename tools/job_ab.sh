#!/bin/bash
# A/B: quick_time of the default library and every libps_var_*.so on the given configs; gpu tests first
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
cfgs=${1:-"cfg2 cfg3 cfg4 cfg5"}
if [ -z "$NOTEST" ]; then ( timeout 900 python -m pytest tests -m gpu -x -q ) > gpurun_out/pytest_gpu.log 2>&1; tail -1 gpurun_out/pytest_gpu.log; fi
: > gpurun_out/ab.txt
for rep in 1 2; do
for L in paper_2209_06909_b200/libpowersort_b200.so paper_2209_06909_b200/libps_var_*.so; do
  echo "== $L" >> gpurun_out/ab.txt
  PS_LIB=$PWD/$L timeout 600 python tools/quick_time.py $cfgs 2>&1 | grep "count=0" >> gpurun_out/ab.txt
done
done
