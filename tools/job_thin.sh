PS_THIN_CUTS=1 timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_thin.log 2>&1; echo rc=$? >> gpurun_out/pytest_thin.log
out=gpurun_out/thin_ab.txt; : > $out
for c in cfg3 cfg4 cfg2; do for T in 1000000000 12000 1; do PS_THIN_CUTS=$T python tools/marginal.py $c | sed "s|^|T=$T |" >> $out; done; done
