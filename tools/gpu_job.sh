cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python tools/quick_time.py cfg2 cfg3 cfg4 cfg5 > gpurun_out/quick.txt 2>&1
( timeout 900 python -m pytest tests -m gpu -x -q ) > gpurun_out/pytest_gpu.log 2>&1
