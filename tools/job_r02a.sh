#!/bin/bash
# round-2 check: gpu tests, default bench (cfg5), reference arm, cfg2 bench
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
nvidia-smi -q | grep -iE "product name|clocks|Max" | head -20 > gpurun_out/smi.txt
( time timeout 1500 python -m pytest tests -m gpu -x -q -rA --durations=20 ) > gpurun_out/pytest_gpu.log 2>&1
( time timeout 900 python bench.py --steps 10 --warmup 3 ) > gpurun_out/bench_cfg5.log 2>&1
( time timeout 900 python bench.py --config cfg2 --steps 20 --warmup 5 ) > gpurun_out/bench_cfg2.log 2>&1
( time timeout 1200 python bench.py --impl reference --steps 10 --warmup 3 ) > gpurun_out/bench_ref.log 2>&1
