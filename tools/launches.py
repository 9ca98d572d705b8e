"""Summarise an ncu --metrics gpu__time_duration.sum launch list (csv log).
usage: python tools/launches.py gpurun_out/launches.csv [--seq]"""
import collections, csv, sys

rows = list(csv.reader(open(sys.argv[1])))
hdr, out = None, []
for r in rows:
    if 'Kernel Name' in r:
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        if d.get('Metric Name') == 'gpu__time_duration.sum':
            out.append((d['ID'], d['Kernel Name'].split('(')[0][:60], d.get('Grid Size', ''),
                        float(d['Metric Value'].replace(',', '')) / 1000.0))
if '--seq' in sys.argv:
    for i, k, g, v in out:
        print('%5s %9.1f us  %-16s %s' % (i, v, g, k))
agg = collections.defaultdict(lambda: [0, 0.0])
for _, k, _, v in out:
    agg[k][0] += 1
    agg[k][1] += v
print('%d launches, %.1f us' % (len(out), sum(v for *_, v in out)))
for k, (c, v) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print('%4d %10.1f us  %s' % (c, v, k))
