#!/bin/bash
# GPU job: ncu --set full of one launch.  usage: tools/job_ncu.sh CFG KERNEL_REGEX SKIP TAG
python tools/one_sort.py $1 && ncu --set full --import-source on --clock-control none -k regex:$2 --launch-skip $3 -c 1 -o gpurun_out/prof_$4 python tools/one_sort.py $1 > gpurun_out/ncu_$4.log 2>&1
