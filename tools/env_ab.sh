#!/bin/bash
# A/B of an environment knob: marginals per config with and without it (gpurun_out/envab.txt)
# usage: tools/env_ab.sh "VAR=value" "cfgs" "stages"
out=gpurun_out/envab.txt; : > $out
for c in $2; do for st in ${3:--1 all}; do
  for E in "PS_NONE=1" "$1"; do
    if [ $st = all ]; then env $E python tools/marginal.py $c | sed "s|^|$E |" >> $out 2>&1;
    else env $E PS_DEBUG_STAGES=$st python tools/marginal.py $c | sed "s|^|$E |" >> $out 2>&1; fi
  done
done; done
