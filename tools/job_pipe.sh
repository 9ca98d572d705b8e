#!/bin/bash
# GPU job: parity tests, cfg2 stage profile, ncu of one big pipe stage (+ smem attribution)
tag=${1:-x}
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo rc=$? >> gpurun_out/pytest_gpu.log
python tools/stage_profile.py cfg2 > gpurun_out/stage_cfg2.txt 2>&1
python bench.py --no-cpu > gpurun_out/bench_cfg2.json 2> gpurun_out/bench_cfg2.err
python tools/one_sort.py cfg2 && ncu --set full --import-source on --clock-control none -k regex:merge_pipe_kernel --launch-skip 3 -c 1 -o gpurun_out/prof_pipe_$tag python tools/one_sort.py cfg2 > gpurun_out/ncu_pipe.log 2>&1
