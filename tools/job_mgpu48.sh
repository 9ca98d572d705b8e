#!/bin/bash
# the distributed bench path at world sizes 4 and 8 with every rank on the box's one GPU (gloo barriers):
# a functional check of the sharded strong-scaling step (not a scaling number)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for N in 4 8; do
  PS_BENCH_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2954$N bench.py --gpus $N --config cfg5 --keys 134217728 --steps 2 --warmup 1 > gpurun_out/bench_mgpu$N.log 2>&1
  echo "N=$N rc=$?"
  grep '^{' gpurun_out/bench_mgpu$N.log | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['n_gpus'], d['value'], d['ms_per_step'], d['parallelism'])"
done
