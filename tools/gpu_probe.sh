nproc > gpurun_out/probe.txt; free -g >> gpurun_out/probe.txt; lscpu | head -20 >> gpurun_out/probe.txt; nvidia-smi >> gpurun_out/probe.txt
( time python -m pytest tests -m gpu -x -q ) > gpurun_out/pytest_gpu.log 2>&1
( time python bench.py --config cfg5 --steps 3 --warmup 1 --no-cpu ) > gpurun_out/bench_cfg5.log 2>&1
