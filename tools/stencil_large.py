#!/usr/bin/env python3
"""Stencils at sizes whose output does not fit in the 126 MB L2 (VERDICT r1
"honest stencil rooflines"): event-timed median of the stage-1/stage-2
variants, L2 flushed before every sample, algorithmic bytes / time against
the measured HBM peak.  One JSON line per (bench, dims, variant).

    python tools/stencil_large.py [--samples 7] [--cases 2DCONV:8192,8192 3DCONV:512,512,512]

The DRAM-counter side (dram__bytes_read/write.sum) comes from an ncu
capture of the same command (tools/gpu_stencil_r02.sh)."""

from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

from paper_1810_10496_b200.backend.b200 import Workspace, alg_work, family  # noqa: E402

DEFAULT = ["2DCONV:4096,4096", "2DCONV:8192,8192", "2DCONV:16384,16384",
           "3DCONV:256,256,256", "3DCONV:384,384,384", "3DCONV:512,512,512"]


def peak_gbs() -> tuple[float, str]:
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        return float(json.loads(p.read_text())["hbm_gbs"]), "MEASURED_PEAKS.json"
    return 7672.0, "B200_PROFILING.md fallback"


def main() -> int:
    ap = argparse.ArgumentParser()
    ap.add_argument("--samples", type=int, default=7)
    ap.add_argument("--cases", nargs="*", default=DEFAULT)
    ap.add_argument("--stages", default="1,2")
    args = ap.parse_args()
    stages = {int(s) for s in args.stages.split(",")}
    peak, src = peak_gbs()
    for case in args.cases:
        bench, d = case.split(":")
        dims = tuple(int(x) for x in d.split(","))
        fam = family(bench)
        ws = Workspace(0, bench, dims)
        ws.generate(True, 1729, -1)
        nbytes, flops = alg_work(bench, dims)
        for v in range(len(fam.knobs)):
            if fam.knobs[v][0] not in stages:
                continue
            ms = ws.run(v, samples=args.samples, batch=1, restore=True, flush=True)
            med = statistics.median(ms)
            gbs = nbytes / (med * 1e-3) / 1e9
            print(json.dumps({"bench": bench, "dims": list(dims), "variant": fam.key(v), "ms_median": med,
                              "ms": [round(x, 5) for x in ms], "alg_bytes": nbytes, "alg_gbs": gbs,
                              "frac_of_hbm": gbs / peak, "peak_gbs": peak, "peak_source": src,
                              "c3_mode": os.environ.get("PF_C3", "")}), flush=True)
        ws.close()
    return 0


if __name__ == "__main__":
    sys.exit(main())
