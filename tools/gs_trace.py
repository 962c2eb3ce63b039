#!/usr/bin/env python3
"""GRAMSCHM panel-kernel timeline (PF_GS_TRACE=1): per CTA b, the time it
starts, finishes applying earlier panels, and publishes its own panel."""
import os
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
os.environ["PF_GS_TRACE"] = "1"
from paper_1810_10496_b200.backend.b200 import B200Backend, family  # noqa: E402

m, n = (int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "2048,2048").split(","))
fam = family("GRAMSCHM")
v = next(i for i in range(len(fam.knobs)) if fam.key(i) == "stage=2,vec=1")
be = B200Backend(device=0)
ws = be.workspace("GRAMSCHM", (m, n), True, -1)
ws.run(v, samples=2, batch=1, restore=True, flush=False)
R = ws.outputs()[1].reshape(n, n)
row = R[n - 1, : 3 * ((n - 1) // 3)].reshape(-1, 3).astype(np.float64)
t0 = row[0, 0]
row = (row - t0) % (1 << 24)
prev_pub = None
for b in range(0, row.shape[0]):
    s, a, p = row[b]
    gap = f"{p - prev_pub:7.2f}" if prev_pub is not None else "      -"
    if b < 6 or b % 16 == 0 or b > row.shape[0] - 4:
        print(f"cta {b:4d}  start {s:9.2f}  applied {a:9.2f}  published {p:9.2f}  factor {p - a:7.2f}  period {gap} us")
    prev_pub = p
per = np.diff(row[:, 2])
fac = row[:, 2] - row[:, 1]
wait = row[1:, 1] - row[:-1, 2]
print(f"mean period {per.mean():.2f} us, mean factor {fac.mean():.2f} us, mean (applied_b - published_b-1) {wait.mean():.2f} us")

st = R[n - 2, :64].reshape(16, 4).astype(np.float64)
st = (st - st[0, 3]) % 167772.16  # microseconds (10 ns resolution, mod 2^24)
print("CTA 5 own-panel steps (us): pivot start | pivot done | last warp past barrier | last warp updated")
for kk in range(16):
    print(f"  step {kk:2d}: {st[kk, 3]:8.2f} {st[kk, 0]:8.2f} {st[kk, 1]:8.2f} {st[kk, 2]:8.2f}")
