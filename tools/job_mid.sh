#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
( timeout 1500 python -m pytest tests -m gpu -x -q ) > gpurun_out/pytest_gpu.log 2>&1; tail -1 gpurun_out/pytest_gpu.log
python tools/quick_time.py cfg1 cfg4 cfg2 cfg3 2>&1
PS_WARP_SMALL=1 PS_LIB=$PWD/paper_2209_06909_b200/libpowersort_b200_debug.so python tools/quick_time.py cfg1 cfg4 cfg2 cfg3 2>&1 | sed 's/^/warp /'
python tools/stage_profile.py cfg4 | head -9
