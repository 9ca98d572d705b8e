"""Per-launch DRAM traffic of merge_pipe_kernel from an ncu csv (dram bytes,
L2 write sectors from the SMs and duration per launch) -> JSON read by
bench.py for roofline.traffic.  The DRAM write counter only sees the lines
evicted while the launch runs; the L2 write sectors (lts__t_sectors_srcunit_
tex_op_write, 32 B each) count every byte the kernel writes, all of which
reaches DRAM eventually, so dram_read + l2_write is the traffic with the
write-back included.
usage: python tools/pipe_traffic.py CSV OUT_JSON [workload]"""
import collections, csv, json, sys

rows = list(csv.reader(open(sys.argv[1])))
workload = sys.argv[3] if len(sys.argv) > 3 else 'cfg2 (n=2^24, k=4)'
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
        if d['Metric Name'] == 'gpu__time_duration.sum':
            v *= {'nsecond': 1, 'usecond': 1e3, 'msecond': 1e6}.get(unit, 1)
        per[d['ID']][d['Metric Name']] = v
launches = [{'id': int(k), 'dram_read': v.get('dram__bytes_read.sum', 0), 'dram_write': v.get('dram__bytes_write.sum', 0),
             'l2_write': 32 * v.get('lts__t_sectors_srcunit_tex_op_write.sum', 0),
             'us': v.get('gpu__time_duration.sum', 0) / 1e3} for k, v in sorted(per.items(), key=lambda kv: int(kv[0]))]
tot = sum(l['dram_read'] + l['dram_write'] for l in launches)
totwb = sum(l['dram_read'] + l['l2_write'] for l in launches)
n = max(len(launches), 1)
out = {'kernel': 'merge_pipe_kernel', 'workload': workload + ', one sort, ncu --clock-control none',
       'launches': len(launches), 'dram_bytes_total': tot, 'dram_bytes_per_launch': tot / n,
       'traffic_incl_writeback_total': totwb, 'traffic_incl_writeback_per_launch': totwb / n,
       'per_launch': launches}
json.dump(out, open(sys.argv[2], 'w'), indent=1)
print('launches', len(launches), 'dram bytes total %.1f MB, per launch %.1f MB; incl. write-back %.1f MB per launch' % (
    tot / 1e6, tot / 1e6 / n, totwb / 1e6 / n))
