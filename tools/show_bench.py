import glob, json, sys
for f in sorted(glob.glob('gpurun_out/bench_cfg*.json')):
    for line in open(f):
        try: d = json.loads(line)
        except Exception: print(f, line[:300]); continue
        print(f, 'value %.3e' % d['value'], 'ms/step %.3f' % d['ms_per_step'])
        r = d.get('roofline') or {}
        print('  roofline achieved %.0f GB/s frac %.3f pass %.0f' % (r.get('achieved', 0), r.get('frac') or 0, r.get('merge_pass_gbs_incl_partition', 0)))
        if d.get('phases_per_step'): print('  phases', {k: round(v['ms'], 3) for k, v in d['phases_per_step'].items()})
        if d.get('e2e'): print('  e2e %.3e  %.3f ms' % (d['e2e']['value'], d['e2e'].get('ms_per_step', 0)))
