"""Per-launch time and DRAM bytes from an ncu --csv launch list captured with
gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum.
usage: python tools/launch_dram.py gpurun_out/pre_cfg2.csv"""
import collections, csv, sys

rows = list(csv.reader(open(sys.argv[1])))
hdr, L = None, collections.OrderedDict()
for r in rows:
    if 'Kernel Name' in r:
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        key = d['ID']
        e = L.setdefault(key, {'name': d['Kernel Name'].split('(')[0][:50], 'grid': d.get('Grid Size', '')})
        v = float(d['Metric Value'].replace(',', ''))
        e[d['Metric Name']] = v
for k, e in L.items():
    t = e.get('gpu__time_duration.sum', 0) / 1e3
    rd = e.get('dram__bytes_read.sum', 0) / 1e6
    wr = e.get('dram__bytes_write.sum', 0) / 1e6
    print('%4s %8.1f us  rd %8.1f MB  wr %8.1f MB  %7.0f GB/s  %-14s %s' % (k, t, rd, wr, (rd + wr) / t * 1e3 / 1e3 if t else 0, e['grid'], e['name']))
