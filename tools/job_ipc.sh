#!/bin/bash
# multi-GPU plumbing after the IPC change: the multigpu GPU tests + the distributed bench with 2 ranks on one GPU
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_multigpu.py -q -x > gpurun_out/pytest_mgpu.log 2>&1; tail -3 gpurun_out/pytest_mgpu.log
bash tools/job_mgpu2.sh
