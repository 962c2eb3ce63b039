#!/usr/bin/env python3
"""Hottest SASS instructions (warp-stall samples) of an ncu report:
    python tools/ncu_hot.py report.ncu-rep [top]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[1]
i_src, i_s = hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)")
recs = [(int(r[i_s] or 0), idx, r[0], r[i_src]) for idx, r in enumerate(rows[2:]) if len(r) > i_s]
tot = sum(r[0] for r in recs) or 1
print(f"total samples {tot}")
for s, idx, addr, src in sorted(recs, reverse=True)[:top]:
    print(f"{100 * s / tot:5.1f}%  #{idx:5d}  {src.strip()[:90]}")
