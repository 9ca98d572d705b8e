#!/bin/bash
# GPU job: refresh the round's committed evidence (outputs in gpurun_out/).
# 1) gpu tests  2) ncu launch list / pipe DRAM traffic / one full pipe capture
# 3) benches of every config (bench.py reads the fresh traffic json), reference arm
tag=${1:-r01}
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo rc=$? >> gpurun_out/pytest_gpu.log
python tools/one_sort.py cfg2 || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${tag}_launches_cfg2.csv python tools/one_sort.py cfg2 > /dev/null 2>&1
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:merge_pipe_kernel --csv --log-file gpurun_out/${tag}_pipe_dram_cfg2.csv python tools/one_sort.py cfg2 > /dev/null 2>&1
python tools/pipe_traffic.py gpurun_out/${tag}_pipe_dram_cfg2.csv profiles/${tag}_pipe_traffic_cfg2.json > gpurun_out/traffic.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:merge_pipe_kernel --launch-skip 4 -c 1 -o gpurun_out/${tag}_pipe_full python tools/one_sort.py cfg2 > /dev/null 2>&1
python bench.py > gpurun_out/bench_cfg2.json 2> gpurun_out/bench_cfg2.err
python bench.py --k 2 --no-cpu > gpurun_out/bench_cfg2k2.json 2> gpurun_out/bench_cfg2k2.err
for c in cfg1 cfg3 cfg4; do python bench.py --config $c --no-cpu --steps 5 > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; done
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
cp profiles/${tag}_pipe_traffic_cfg2.json gpurun_out/ 2>/dev/null
