#!/bin/bash
# Round evidence at HEAD: gpu tests, smoke, default bench (cfg5), every other config, the reference arm,
# the launch list of one cfg5 sort.  Outputs in gpurun_out/.
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
for f in gpurun_out/bench_*.json; do python -c "import json,sys; d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', '%.3e'%d['value'], d.get('ms_per_step'), (d.get('roofline') or {}).get('frac_of_8TBps'), (d.get('e2e') or {}).get('value'))"; done
