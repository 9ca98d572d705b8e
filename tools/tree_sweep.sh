#!/bin/bash
# A/B sweep of the one-CTA tree crossover and per-phase marginals (outputs in gpurun_out/)
out=gpurun_out/tree_sweep.txt
: > $out
for c in cfg2 cfg3; do
  for t in 1024 20000; do
    for st in -1 -2 -3 all; do
      if [ $st = all ]; then PS_TREE_SMALL_R=$t python tools/marginal.py $c | sed "s/^/R=$t /" >> $out 2>&1;
      else PS_TREE_SMALL_R=$t PS_DEBUG_STAGES=$st python tools/marginal.py $c | sed "s/^/R=$t /" >> $out 2>&1; fi
    done
  done
done
for c in cfg1 cfg4; do for st in -1 -2 -3 all; do
  if [ $st = all ]; then python tools/marginal.py $c >> $out 2>&1; else PS_DEBUG_STAGES=$st python tools/marginal.py $c >> $out 2>&1; fi
done; done
