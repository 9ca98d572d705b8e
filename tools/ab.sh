#!/bin/bash
# A/B of two library builds: marginals per config (gpurun_out/ab.txt); usage: tools/ab.sh libB.so "cfgs"
out=gpurun_out/ab.txt; : > $out
for c in $2; do for st in -3 all; do
  for L in paper_2209_06909_b200/libpowersort_b200.so $1; do
    if [ $st = all ]; then PS_LIB=$L python tools/marginal.py $c | sed "s|^|$(basename $L) |" >> $out 2>&1;
    else PS_LIB=$L PS_DEBUG_STAGES=$st python tools/marginal.py $c | sed "s|^|$(basename $L) |" >> $out 2>&1; fi
  done
done; done
