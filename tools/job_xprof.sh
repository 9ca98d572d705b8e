#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/xm_launches.csv python tools/xmerge_time.py 134217728 8 > /dev/null 2>&1
ncu --set full --import-source on --clock-control none -k regex:xs_merge_kernel -s 1 -c 1 -o gpurun_out/xm_full python tools/xmerge_time.py 134217728 8 > /dev/null 2>&1
ls -la gpurun_out
