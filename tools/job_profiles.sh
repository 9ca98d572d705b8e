#!/bin/bash
# GPU job: the round's committed profiles (run after the plain commands passed)
tag=${1:-r01}
python tools/one_sort.py cfg2 || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${tag}_launches_cfg2.csv python tools/one_sort.py cfg2 > /dev/null 2>&1
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:merge_pipe_kernel --csv --log-file gpurun_out/${tag}_pipe_dram_cfg2.csv python tools/one_sort.py cfg2 > /dev/null 2>&1
ncu --set full --import-source on --clock-control none -k regex:merge_pipe_kernel --launch-skip 3 -c 1 -o gpurun_out/${tag}_pipe_full python tools/one_sort.py cfg2 > /dev/null 2>&1
