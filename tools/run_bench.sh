#!/bin/bash
# helper for gpurun: gpu tests + benches of all configs (outputs in gpurun_out/)
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo rc=$? >> gpurun_out/pytest_gpu.log
python bench.py --no-cpu > gpurun_out/bench_cfg2.json 2> gpurun_out/bench_cfg2.err
for c in cfg1 cfg3 cfg4; do python bench.py --config $c --no-cpu --steps 5 > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; done
