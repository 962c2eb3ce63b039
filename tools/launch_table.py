#!/usr/bin/env python3
"""Per-kernel durations of one variant run from an ncu launch list (the first
run after the first L2 flush): python tools/launch_table.py launches.csv"""
import csv
import sys

lines = open(sys.argv[1]).readlines()
i = next(i for i, l in enumerate(lines) if l.startswith('"ID"'))
rows = list(csv.reader(lines[i:]))
seen, total = 0, 0.0
for r in rows[1:]:
    if "init_kernel" in r[4]:
        continue
    if "flush" in r[4]:
        seen += 1
        if seen > 1:
            break
        continue
    us = float(r[-1]) / 1000
    total += us
    print(f"{r[4][:64]:64s} {r[8]:>14s} {us:8.2f} us")
print(f"{'sum':64s} {'':>14s} {total:8.2f} us")
