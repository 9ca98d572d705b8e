#!/bin/bash
# multi-GPU path on one GPU: shard-merge tests, 2-process gloo bench (ranks share the GPU)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
( timeout 900 python -m pytest tests/test_multigpu.py -m gpu -x -q -rA ) > gpurun_out/pytest_mgpu.log 2>&1
tail -3 gpurun_out/pytest_mgpu.log
PS_BENCH_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --config cfg5 --keys 268435456 --steps 3 --warmup 1 > gpurun_out/bench_mgpu2.log 2>&1
tail -c 1500 gpurun_out/bench_mgpu2.log
python tools/xmerge_time.py > gpurun_out/xmerge_time.txt 2>&1
cat gpurun_out/xmerge_time.txt
