out=gpurun_out/sweep.txt; : > $out
for c in cfg2 cfg3 cfg4; do for T in 6000 9000 12000 20000; do PS_THIN_CUTS=$T python tools/marginal.py $c | sed "s|^|THIN=$T |" >> $out; done; done
for c in cfg4 cfg1; do for T in 4096 16384 32768 131072; do PS_TINY_MIN=$T python tools/marginal.py $c | sed "s|^|TINY=$T |" >> $out; done; done
