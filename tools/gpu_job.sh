cd $GRAFT_REPO_ROOT
python tools/quick_time.py cfg1 cfg2 cfg3 cfg4 cfg5 > gpurun_out/quick.txt 2>&1
( time python -m pytest tests -m gpu -x -q ) > gpurun_out/pytest_gpu.log 2>&1
