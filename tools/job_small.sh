#!/bin/bash
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo rc=$? >> gpurun_out/pytest_gpu.log
out=gpurun_out/small_ab.txt; : > $out
for c in cfg4 cfg1 cfg2 cfg3; do for E in PS_OLD_SMALL=1 PS_NONE=1; do env $E python tools/marginal.py $c | sed "s|^|$E |" >> $out; done; done
python tools/stage_profile.py cfg4 > gpurun_out/stage_cfg4.txt 2>&1
