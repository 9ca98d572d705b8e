#!/bin/bash
# on the GPU box: stage profile of cfg2 for every variant library
for f in paper_2209_06909_b200/libps_var_*.so; do
  echo "== $f" >> gpurun_out/variants.txt
  PS_LIB=$PWD/$f python tools/stage_profile.py ${1:-cfg2} 2>&1 | grep -E "stage  1[123]|stage   [3-7]|sum of|parity" >> gpurun_out/variants.txt
done
