#!/bin/bash
# ncu DRAM / L2-write traffic of every merge_pipe_kernel launch of one sort (cfg2, cfg5) -> profiles/r02_pipe_traffic_*.json
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
M=dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_srcunit_tex_op_write.sum,gpu__time_duration.sum
for c in cfg2 cfg5; do
  ncu --metrics $M --clock-control none -k regex:merge_pipe_kernel --csv --log-file gpurun_out/pipe_dram_$c.csv python tools/one_sort.py $c > gpurun_out/ncu_$c.log 2>&1
  python tools/pipe_traffic.py gpurun_out/pipe_dram_$c.csv gpurun_out/r02_pipe_traffic_$c.json "$c (k=4)"
done
