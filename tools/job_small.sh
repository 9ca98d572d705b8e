#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
( timeout 900 python -m pytest tests/test_reference_suite.py -q -rA ) > gpurun_out/pytest_refsuite.log 2>&1
tail -3 gpurun_out/pytest_refsuite.log
for c in cfg1 cfg4; do python tools/stage_profile.py $c > gpurun_out/stages_$c.txt 2>&1; done
for c in cfg1 cfg4; do PS_LIB=$PWD/paper_2209_06909_b200/libpowersort_b200_debug.so python tools/marginal.py $c; done > gpurun_out/marginal.txt 2>&1
for s in -3 -2 -1 0; do PS_LIB=$PWD/paper_2209_06909_b200/libpowersort_b200_debug.so PS_DEBUG_STAGES=$s python tools/marginal.py cfg1; done >> gpurun_out/marginal.txt 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cfg1.csv python tools/one_sort.py cfg1 > /dev/null 2>&1
python tools/host_time.py cfg1 > gpurun_out/host_time_cfg1.txt 2>&1
