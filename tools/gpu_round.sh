#!/bin/bash
# One GPU session: tests, the default bench (cfg5) and the reference arm.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
( time python -m pytest tests -m gpu -x -q -rA ) > gpurun_out/pytest_gpu.log 2>&1
( time python bench.py --steps 20 --warmup 5 ) > gpurun_out/bench_cfg5.log 2>&1
( time python bench.py --impl reference --steps 20 --warmup 5 ) > gpurun_out/bench_ref.log 2>&1
