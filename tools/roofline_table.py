#!/usr/bin/env python3
"""Per-kernel roofline table from a variant report (best variant per benchmark).

    python tools/roofline_table.py profiles/r01_variant_report_v7.json profiles/r01_roofline_v7.md

Bounds: HBM for the BLAS-2 set and the two convolutions
(algorithmic bytes / time vs the measured copy bandwidth); the tensor ceiling for
the contractions: since round 2 the pre-split products run 3xFP16 on
kind::f16 (standard flops / time vs bf16 burst / 3, and vs the MMA-only rate
of the kind::f16 pair pipeline measured with PF_TC_DIAG=5); GEMM 512^3 stays
3xTF32 (bf16 burst / 2 / 3); L2 / latency kernels get no
HBM fraction (FDTD keeps its fields in L2; GRAMSCHM is a chain of 2048
dependent column steps).
"""

from __future__ import annotations

import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
BOUND = {
    "ATAX": "hbm", "BICG": "hbm", "MVT": "hbm", "GESUMMV": "hbm", "2DCONV": "hbm", "3DCONV": "hbm",
    "GEMM": "tensor (latency at 512^3)", "2MM": "tensor", "3MM": "tensor", "SYRK": "tensor", "SYR2K": "tensor",
    "CORR": "tensor + hbm", "COVAR": "tensor + hbm", "FDTD-2D": "l2", "GRAMSCHM": "latency (column chain)",
}
# 2MM 2048^3, kind::f16 pair kernel with operand loads disabled (PF_TC_DIAG=5): 44.1 us per 17.18 GF product on
# the 128 SMs its 64 pair tiles occupy (profiles/r02/mma_only_2MM.csv)
MMA_ONLY_TFLOPS = 389.6
F16_BENCHES = ("2MM", "3MM", "SYRK", "SYR2K", "CORR", "COVAR")


def main() -> int:
    rep = json.loads(Path(sys.argv[1]).read_text())
    peaks = json.loads((ROOT / "MEASURED_PEAKS.json").read_text())
    hbm = float(peaks["hbm_gbs"])
    tc32 = float(peaks["bf16_tflops"]) / 2 / 3
    tc16 = float(peaks["bf16_tflops"]) / 3
    rows = [
        f"# Roofline per benchmark (best variant, config size) — `{Path(sys.argv[1]).name}`",
        "",
        f"HBM peak {hbm:.0f} GB/s (measured copy).  Tensor ceilings from the measured bf16 burst "
        f"{float(peaks['bf16_tflops']):.0f} TF/s: 3xFP16 {tc16:.0f} TF/s (/ 3 MMAs per product; 2MM, 3MM, SYRK, "
        f"SYR2K, CORR, COVAR) and 3xTF32 {tc32:.0f} TF/s (/ 2 for TF32 / 3; GEMM 512^3).  MMA-only rate of the "
        f"kind::f16 pair pipeline {MMA_ONLY_TFLOPS:.0f} TF/s (PF_TC_DIAG=5, on the 128 SMs a 2048^2 product "
        f"occupies).",
        "",
        "| benchmark | bound | best variant | ms | speedup vs baseline | achieved | fraction of bound |",
        "|---|---|---|---|---|---|---|",
    ]
    for b in sorted(rep["benches"]):
        r = rep["benches"][b]
        bound = BOUND.get(b, "?")
        ms = r["best_ms"]
        if bound == "hbm":
            ach, frac = f"{r['best_gbs']:.0f} GB/s", f"{r['best_gbs'] / hbm:.0%} of HBM"
        elif bound.startswith("tensor"):
            tf = r["best_tflops"]
            if b in F16_BENCHES:
                ach, frac = f"{tf:.1f} TF/s", f"{tf / tc16:.0%} of 3xFP16 ({tf / MMA_ONLY_TFLOPS:.0%} of MMA-only)"
            else:
                ach, frac = f"{tf:.1f} TF/s", f"{tf / tc32:.0%} of 3xTF32"
            if b in ("SYRK", "SYR2K"):  # symmetric: half of the standard flops are computed
                frac += "; standard flops, half computed (symmetry)"
        elif bound == "l2":
            ach, frac = f"{r['best_gbs']:.0f} GB/s (L2-resident)", "—"
        else:
            ach, frac = f"{r['best_tflops']:.1f} TF/s", "—"
        rows.append(f"| {b} | {bound} | `{r['best_variant']}` | {ms:.4g} | {r['speedup_full']:.1f}x | {ach} | {frac} |")
    Path(sys.argv[2]).write_text("\n".join(rows) + "\n")
    print("\n".join(rows))
    return 0


if __name__ == "__main__":
    sys.exit(main())
