#!/usr/bin/env python3
"""Print `duration_us  kernel` rows from an ncu --csv launch list on stdin
(the kernel names hold commas, so `cut` cannot split them)."""
import csv
import sys

rows = [r for r in csv.reader(l for l in sys.stdin if l.startswith('"'))]
if rows:
    h = rows[0]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    for r in rows[1:]:
        if len(r) > vi and r[h.index("Metric Name")] == "gpu__time_duration.sum":
            v = float(r[vi].replace(",", ""))
            v = v / 1000.0 if r[ui] in ("nsecond", "ns") else v
            print(f"{v:9.2f} us  {r[ki][:110]}")
