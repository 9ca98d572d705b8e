#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
( timeout 900 python -m pytest tests/test_multigpu.py -m gpu -x -q ) > gpurun_out/pytest_mgpu.log 2>&1
tail -1 gpurun_out/pytest_mgpu.log
python tools/xmerge_time.py 134217728 2 4 8 2>&1
ncu --set full --import-source on --clock-control none -k regex:xs_merge_kernel -s 1 -c 1 -o gpurun_out/xm_full2 python tools/xmerge_time.py 134217728 8 > /dev/null 2>&1
