#!/usr/bin/env python3
"""Run one variant of one benchmark a few times (for ncu captures).

    ncu --set full -k regex:s2_fused -c 2 python tools/profile_kernels.py ATAX 16384,16384 stage=2
"""

from __future__ import annotations

import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

from paper_1810_10496_b200.backend.b200 import B200Backend, family  # noqa: E402


def main() -> int:
    bench, dims, key = sys.argv[1], tuple(int(x) for x in sys.argv[2].split(",")), sys.argv[3]
    reps = int(sys.argv[4]) if len(sys.argv) > 4 else 3
    fam = family(bench)
    v = next(i for i in range(len(fam.knobs)) if fam.key(i) == key)
    be = B200Backend(device=0)
    ws = be.workspace(bench, dims, True, -1)
    ms = ws.run(v, samples=reps, batch=1, restore=True, flush=True)
    print(bench, dims, key, "ms:", [round(x, 4) for x in ms])
    return 0


if __name__ == "__main__":
    sys.exit(main())
