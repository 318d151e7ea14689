#!/usr/bin/env python
"""Summarise ncu reports: duration, pipe utilisations, issue activity, top stall PCs."""
import csv
import subprocess
import sys

WANT = ['gpu__time_duration.sum', 'sm__pipe_tensor_cycles_active_realtime.avg.pct',
        'sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active',
        'sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active',
        'sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active', 'smsp__issue_active.avg.pct',
        'dram__bytes_read.sum', 'dram__bytes_write.sum', 'launch__grid_size', 'launch__registers_per_thread',
        'sm__cycles_elapsed.avg.per_second', 'lts__t_sectors.avg.pct']


def raw(rep):
    out = subprocess.run(['ncu', '-i', rep, '--page', 'raw', '--csv'], capture_output=True, text=True).stdout
    r = list(csv.reader(out.splitlines()))
    return [(a, b, c) for a, b, c in zip(r[0], r[1], r[2])]


def top(rep, n):
    out = subprocess.run(['ncu', '-i', rep, '--page', 'source', '--csv', '--print-source', 'sass'],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))[2:]
    tot = sum(int(r[2] or 0) for r in rows)
    print(f'   samples {tot}')
    for r in sorted(rows, key=lambda r: -int(r[2] or 0))[:n]:
        print(f'   {r[0][-5:]} {int(r[2]) / tot * 100:5.1f}% {r[1][:90]}')


for rep in sys.argv[1:]:
    print('==', rep)
    for a, b, c in raw(rep):
        if any(a.startswith(k) or k in a for k in WANT):
            print('  ', a, b, c)
    top(rep, 12)
