#!/bin/bash
# Final evidence of the round at HEAD: gpu tests, smoke, benches of every config, reference arm,
# launch list + full ncu capture of one cfg5 level, DRAM/L2 traffic of the pipe launches, phase counters.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
( time timeout 1500 python -m pytest tests -m gpu -q -rA ) > gpurun_out/pytest_gpu.log 2>&1
tail -1 gpurun_out/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -1 gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench_cfg5.json 2> gpurun_out/bench_cfg5.err
for c in cfg1 cfg2 cfg3 cfg4; do timeout 600 python bench.py --config $c --steps 20 --warmup 5 > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; done
timeout 600 python bench.py --config cfg2 --k 2 --no-cpu --steps 20 --warmup 5 > gpurun_out/bench_cfg2k2.json 2> gpurun_out/bench_cfg2k2.err
timeout 1500 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cfg5.csv python tools/one_sort.py cfg5 > /dev/null 2>&1
bash tools/job_traffic.sh > gpurun_out/traffic.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:merge_pipe_kernel --launch-skip 4 -c 1 -o gpurun_out/pipe_cfg5_level python tools/one_sort.py cfg5 > /dev/null 2>&1
for c in cfg1 cfg2 cfg3 cfg4; do timeout 300 python tools/stage_profile.py $c > gpurun_out/stages_$c.txt 2>&1; done
for f in gpurun_out/bench_*.json; do python -c "import json,sys; d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', '%.3e'%d['value'], d.get('ms_per_step'), (d.get('roofline') or {}).get('frac_of_8TBps'), (d.get('e2e') or {}).get('value'))"; done
