"""Per-launch DRAM traffic of merge_pipe_kernel from an ncu csv (dram bytes +
duration per launch) -> profiles/<tag>_pipe_traffic.json, read by bench.py for
roofline.traffic.  usage: python tools/pipe_traffic.py CSV OUT_JSON"""
import collections, csv, json, sys

rows = list(csv.reader(open(sys.argv[1])))
hdr, per = None, collections.defaultdict(dict)
for r in rows:
    if 'Kernel Name' in r:
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        v = float(d['Metric Value'].replace(',', ''))
        unit = d.get('Metric Unit', '')
        if d['Metric Name'].startswith('dram__bytes'):
            v *= {'byte': 1, 'Kbyte': 1e3, 'Mbyte': 1e6, 'Gbyte': 1e9}.get(unit, 1)
        per[d['ID']][d['Metric Name']] = v
launches = [{'id': int(k), 'dram_read': v.get('dram__bytes_read.sum', 0), 'dram_write': v.get('dram__bytes_write.sum', 0),
             'us': v.get('gpu__time_duration.sum', 0) / 1e3} for k, v in sorted(per.items(), key=lambda kv: int(kv[0]))]
tot = sum(l['dram_read'] + l['dram_write'] for l in launches)
out = {'kernel': 'merge_pipe_kernel<int>', 'workload': 'cfg2 (n=2^24, k=4), one sort, ncu --clock-control none',
       'launches': len(launches), 'dram_bytes_total': tot, 'dram_bytes_per_launch': tot / max(len(launches), 1),
       'per_launch': launches}
json.dump(out, open(sys.argv[2], 'w'), indent=1)
print('launches', len(launches), 'dram bytes total %.1f MB, per launch %.1f MB' % (tot / 1e6, tot / 1e6 / max(len(launches), 1)))
