#!/bin/bash
# GPU job: parity tests + per-phase marginals of every config (outputs in gpurun_out/)
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo rc=$? >> gpurun_out/pytest_gpu.log
out=gpurun_out/marginals.txt
: > $out
for c in ${CFGS:-cfg1 cfg2 cfg3 cfg4}; do for st in -1 -2 -3 all; do
  if [ $st = all ]; then python tools/marginal.py $c >> $out 2>&1; else PS_DEBUG_STAGES=$st python tools/marginal.py $c >> $out 2>&1; fi
done; done
