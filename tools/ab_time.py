#!/usr/bin/env python3
"""Median device time of one variant under the current environment (A/B runs
of the PF_* switches): python tools/ab_time.py BENCH d0,d1,.. KEY [samples]"""

from __future__ import annotations

import statistics
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

from paper_1810_10496_b200.backend.b200 import B200Backend, family  # noqa: E402


def main() -> int:
    bench, dims, key = sys.argv[1], tuple(int(x) for x in sys.argv[2].split(",")), sys.argv[3]
    samples = int(sys.argv[4]) if len(sys.argv) > 4 else 20
    fam = family(bench)
    v = next(i for i in range(len(fam.knobs)) if fam.key(i) == key)
    be = B200Backend(device=0)
    ws = be.workspace(bench, dims, True, -1)
    ws.run(v, samples=3, batch=1, restore=True, flush=True)
    ms = ws.run(v, samples=samples, batch=1, restore=True, flush=True)
    print(f"{bench} {dims} {key}: median {statistics.median(ms) * 1e3:.2f} us  min {min(ms) * 1e3:.2f} us")
    be.close()
    return 0


if __name__ == "__main__":
    sys.exit(main())
