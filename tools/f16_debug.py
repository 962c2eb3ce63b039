#!/usr/bin/env python3
"""Localise 3xFP16 contraction errors: 2MM's first product C = A B at a few
sizes with stock / wide-range operands, against numpy fp64.  Prints the worst
error ratio and where the bad elements sit (rows / columns / tiles)."""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

from paper_1810_10496_b200.backend.b200 import Workspace, family  # noqa: E402


def wide(rng, shape, decades):
    mag = 10.0 ** rng.uniform(-decades / 2, decades / 2, size=shape)
    return (mag * rng.choice([-1.0, 1.0], size=shape)).astype(np.float32)


def main() -> int:
    fam = family("2MM")
    v = next(i for i in range(len(fam.knobs)) if fam.key(i) == "stage=2")
    rng = np.random.default_rng(3)
    for n in (1792, 2048):
        for mode in ("stock", "A-wide", "B-wide", "both", "B-rowscaled", "B-colscaled"):
            ws = Workspace(0, "2MM", (n, n, n, n))
            ws.generate(True, 1729, -1)
            A = ws.download(0).reshape(n, n)
            B = ws.download(1).reshape(n, n)
            if mode in ("A-wide", "both"):
                A = wide(rng, (n, n), 6)
                ws.upload(0, A)
            if mode in ("B-wide", "both"):
                B = wide(rng, (n, n), 6)
                ws.upload(1, B)
            if mode == "B-rowscaled":  # rows of B (k index) scaled: per-column max unchanged pattern
                B = (B * (2.0 ** rng.integers(-8, 8, size=(n, 1)))).astype(np.float32)
                ws.upload(1, B)
            if mode == "B-colscaled":  # columns of B (n index) scaled: per-column scales differ
                B = (B * (2.0 ** rng.integers(-8, 8, size=(1, n)))).astype(np.float32)
                ws.upload(1, B)
            ws.run(v, samples=1, batch=1, restore=False, flush=False)
            C = ws.download(2).reshape(n, n).astype(np.float64)
            ref = A.astype(np.float64) @ B.astype(np.float64)
            tol = np.maximum(1e-4 * np.abs(ref).max(), 1e-4 * np.abs(ref))
            ratio = np.abs(C - ref) / tol
            bad = ratio > 1
            print(f"n={n} {mode:12s} worst={ratio.max():.3g} bad={int(bad.sum())} "
                  f"nonfinite={int((~np.isfinite(C)).sum())}", flush=True)
            if bad.any():
                rows = np.unique(np.nonzero(bad)[0])
                cols = np.unique(np.nonzero(bad)[1])
                i, j = np.unravel_index(np.argmax(ratio), ratio.shape)
                print(f"   bad rows {len(rows)} (first {rows[:8].tolist()}), bad cols {len(cols)} "
                      f"(first {cols[:8].tolist()}); worst at ({i},{j}) got {C[i, j]:.6g} ref {ref[i, j]:.6g}; "
                      f"ratio got/ref over bad: median {np.median(C[bad] / ref[bad]):.6g}", flush=True)
            ws.close()
    return 0


if __name__ == "__main__":
    sys.exit(main())
