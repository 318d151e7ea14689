#!/usr/bin/env python
"""Stall-reason totals of an ncu report, split by PC range: ncu_stalls.py REP [lo-hi ...] (hex suffixes)."""
import csv
import subprocess
import sys

rep = sys.argv[1]
out = subprocess.run(['ncu', '-i', rep, '--page', 'source', '--csv', '--print-source', 'sass'],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr, rows = rows[1], rows[2:]
cols = [i for i, h in enumerate(hdr) if h.startswith('stall_') and 'Not Issued' not in h]
ranges = [tuple(int(x, 16) for x in a.split('-')) for a in sys.argv[2:]] or [(0, 1 << 64)]
for lo, hi in ranges:
    tot = {hdr[i]: 0 for i in cols}
    n = 0
    for r in rows:
        a = int(r[0], 16) & 0xfffff
        if lo <= a < hi:
            n += int(r[2] or 0)
            for i in cols:
                tot[hdr[i]] += int(r[i] or 0)
    s = sum(tot.values()) or 1
    print(f'[{lo:x},{hi:x}) samples {n}: ' + ', '.join(f'{k[6:]} {v / s * 100:.0f}%' for k, v in
                                                   sorted(tot.items(), key=lambda x: -x[1]) if v / s > 0.02))
