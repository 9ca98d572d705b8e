#!/bin/bash
# the distributed bench path (DistributedSorter) with 2 ranks sharing the one GPU (gloo barriers)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
PS_BENCH_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --config cfg5 --keys 268435456 --steps 3 --warmup 1 > gpurun_out/bench_mgpu2.log 2>&1
echo rc=$?
grep '^{' gpurun_out/bench_mgpu2.log | tail -1
tail -5 gpurun_out/bench_mgpu2.log | grep -v '^{'
