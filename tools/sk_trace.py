#!/usr/bin/env python3
"""Timeline of the cluster split-K kernel (PF_SK_TRACE=1 must be set):
python tools/sk_trace.py GEMM 512,512,512 [array index of D] [S]

Prints, per event, the min / median / max over CTAs of the %globaltimer stamp
relative to the earliest kernel entry (ns)."""

from __future__ import annotations

import os
import statistics
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

from paper_1810_10496_b200.backend.b200 import B200Backend, family  # noqa: E402

EVENTS = ["entry", "setup", "loads issued", "first tile landed", "mma committed", "accum ready",
          "partials exchanged", "slice stored", "exit",
          "k-block 1 landed", "k-block 2 landed", "k-block 3 landed", "k-block 3+ landed",
          "k-block 0 converted", "k-block 1 converted", "k-block 2 converted"]


def main() -> int:
    assert os.environ.get("PF_SK_TRACE") == "1"
    bench, dims = sys.argv[1], tuple(int(x) for x in sys.argv[2].split(","))
    out_idx = int(sys.argv[3]) if len(sys.argv) > 3 else 2
    S = int(sys.argv[4]) if len(sys.argv) > 4 else 4  # the launch's split factor (tc_splitk_factor)
    fam = family(bench)
    v = next(i for i in range(len(fam.knobs)) if fam.key(i) == "stage=2")
    be = B200Backend(device=0)
    ws = be.workspace(bench, dims, True, -1)
    for _ in range(3):
        ws.run(v, samples=1, batch=1, restore=True, flush=True)
    m, n = dims[0], dims[1]
    d = ws.download(out_idx).astype(np.float32).view(np.uint32).reshape(m, n)
    rows = []
    for r0 in [t + r * (128 // S) for t in range(0, m, 128) for r in range(S)]:
        for c0 in range(0, n, 64):
            w = d[r0, c0:c0 + 32].astype(np.uint64)
            t = w[0::2] | (w[1::2] << np.uint64(32))
            if t[0] > 10**15 and all(t[i] >= t[0] for i in range(9)):
                rows.append(t)
    t0 = min(int(r[0]) for r in rows)
    print(f"{len(rows)} CTA traces")
    for e, name in enumerate(EVENTS):
        xs = [int(r[e]) - t0 for r in rows]
        print(f"{name:20s} min {min(xs):7d}  med {statistics.median(xs):9.0f}  max {max(xs):7d} ns")
    be.close()
    return 0


if __name__ == "__main__":
    sys.exit(main())
