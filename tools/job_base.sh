#!/bin/bash
# Baseline at HEAD in a fresh container: gpu tests, quick timings, cfg1 launch list
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
( time timeout 1500 python -m pytest tests -m gpu -q -x ) > gpurun_out/pytest_gpu.log 2>&1
tail -3 gpurun_out/pytest_gpu.log
timeout 600 python tools/quick_time.py cfg1 cfg2 cfg4 cfg3 cfg5 > gpurun_out/quick.txt 2>&1; cat gpurun_out/quick.txt
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cfg1.csv python tools/one_sort.py cfg1 > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cfg2.csv python tools/one_sort.py cfg2 > /dev/null 2>&1
