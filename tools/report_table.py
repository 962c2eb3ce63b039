#!/usr/bin/env python3
"""Render variant_report JSON files as one markdown table (later files win per benchmark).

    python tools/report_table.py profiles/table.md report1.json [report2.json ...]
"""

from __future__ import annotations

import json
import math
import sys
from pathlib import Path


def main() -> int:
    out = Path(sys.argv[1])
    benches: dict = {}
    hbm = None
    for f in sys.argv[2:]:
        d = json.loads(Path(f).read_text())
        hbm = d.get("hbm_peak_gbs", hbm)
        benches.update(d["benches"])
    rows = ["| benchmark | dims | baseline ms | best stage-0 (phase-order class) | x | Table-1 order | x | best variant | ms | x | GB/s (% of HBM) | TF/s |",
            "|---|---|---|---|---|---|---|---|---|---|---|---|"]
    geo = {"phase": [], "full": [], "t1": []}
    for b in sorted(benches):
        r = benches[b]
        t1 = r.get("table1") or {}
        t1s = f"{t1.get('speedup'):.2f}" if t1.get("speedup") else "—"
        rows.append(
            f"| {b} | {'x'.join(map(str, r['dims']))} | {r['baseline_ms']:.3f} | `{r['best_phase_variant']}` "
            f"{r['best_phase_ms']:.3f} | {r['speedup_phase']:.2f} | `{t1.get('variant', '—')}` | {t1s} | "
            f"`{r['best_variant']}` | {r['best_ms']:.3f} | {r['speedup_full']:.1f} | {r['best_gbs']:.0f} "
            f"({100 * r['best_hbm_frac']:.0f}%) | {r['best_tflops']:.1f} |")
        geo["phase"].append(r["speedup_phase"])
        geo["full"].append(r["speedup_full"])
        if t1.get("speedup"):
            geo["t1"].append(t1["speedup"])
    g = {k: math.exp(sum(map(math.log, v)) / len(v)) if v else float("nan") for k, v in geo.items()}
    rows.append("")
    rows.append(f"Geomean speedup over the baseline variant ({len(benches)} kernels): phase-order class "
                f"**{g['phase']:.2f}x**, paper Table-1 orders **{g['t1']:.2f}x** ({len(geo['t1'])} kernels), "
                f"with Blackwell staging **{g['full']:.1f}x**. HBM peak {hbm} GB/s (measured).")
    out.write_text("\n".join(rows) + "\n")
    print(out.read_text())
    return 0


if __name__ == "__main__":
    sys.exit(main())
