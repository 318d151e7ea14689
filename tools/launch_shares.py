#!/usr/bin/env python
"""Per-kernel share of an ncu --metrics gpu__time_duration.sum CSV launch list."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = None
agg = collections.defaultdict(lambda: [0, 0.0])
for r in rows:
    if 'Kernel Name' in r:
        hdr = r
        continue
    if hdr is None or len(r) != len(hdr):
        continue
    d = dict(zip(hdr, r))
    if d.get('Metric Name') != 'gpu__time_duration.sum':
        continue
    name = d['Kernel Name'].split('(')[0].replace('void ', '').replace('(anonymous namespace)::', '')[:70]
    v = float(d['Metric Value'].replace(',', ''))
    v *= {'nsecond': 1e-6, 'usecond': 1e-3, 'msecond': 1.0, 'second': 1e3}.get(d['Metric Unit'], 1e-6)
    agg[name][0] += 1
    agg[name][1] += v
tot = sum(a[1] for a in agg.values())
print(f"{sum(a[0] for a in agg.values())} launches, {tot:.1f} ms total device time (serialised, cold cache)")
for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{t:10.1f} ms {100 * t / tot:5.1f}% {n:6d}  {k}")
