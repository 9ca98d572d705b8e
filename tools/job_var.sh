#!/bin/bash
# A/B of variant libraries: cfg5 at 2^28 stage profile (big pipe stages) + cfg2/cfg4 marginals
cd "$(dirname "$0")/.."
out=gpurun_out/var.txt; : > $out
for f in paper_2209_06909_b200/libpowersort_b200.so paper_2209_06909_b200/libps_var_*.so; do
  echo "== $f" >> $out
  PS_LIB=$PWD/$f timeout 300 python tools/stage_profile.py cfg5 268435456 nocount 2>&1 | grep -E "GB/s|sum of|parity" | sort -k9 -n -r | head -14 >> $out
  for c in ${CFGS:-cfg2 cfg4}; do PS_LIB=$PWD/$f timeout 300 python tools/marginal.py $c >> $out 2>&1; done
done
