#!/usr/bin/env python3
"""Time every variant of every benchmark at a size class on one GPU.

For each benchmark: device time (median of samples, CUDA events, L2 flushed
before each sample) of every variant at the measurement size, then

* speedup_phase  = baseline / best stage-0 variant   (the paper's transformations
                   only: store promotion, unrolling, strength reduction, vectors)
* speedup_full   = baseline / best variant           (with Blackwell staging)
* speedup_table1 = baseline / variant selected by the paper's Table-1 order
* roofline of the best variant: algorithmic bytes / time vs the measured HBM
  peak, algorithmic flops / time in TFLOP/s.

Writes a JSON report (default profiles/variant_report.json) and prints a
markdown table.  Variants slower than ``--skip-ms`` after one sample are not
re-sampled (their single sample is kept).
"""

from __future__ import annotations

import argparse
import json
import math
import statistics
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

from paper_1810_10496_b200 import passmodel, registry  # noqa: E402
from paper_1810_10496_b200.backend.b200 import B200Backend, alg_work, family  # noqa: E402
from paper_1810_10496_b200.catalog import parse_phase_order  # noqa: E402

TABLE1 = {
    "2MM": "-cfl-anders-aa -dse -loop-reduce -licm -instcombine",
    "3MM": "-loop-reduce -gvn-hoist -reg2mem -cfl-anders-aa -sroa -licm",
    "ATAX": "-bb-vectorize -loop-reduce -licm -cfl-anders-aa",
    "BICG": "-gvn -loop-reduce -cfl-anders-aa -licm -loop-reduce",
    "CORR": "-cfl-anders-aa -loop-reduce -gvn -sink -loop-extract-single -loop-unswitch -loop-unswitch -ipsccp "
            "-reg2mem -licm -nvptx-lower-alloca",
    "COVAR": "-cfl-anders-aa -loop-unswitch -reassociate -jump-threading -loop-reduce -gvn -loop-unswitch "
             "-reassociate -sink -loop-unswitch -loop-reduce -jump-threading -reg2mem -licm -nvptx-lower-alloca",
    "GEMM": "-cfl-anders-aa -print-memdeps -loop-reduce -licm",
    "GESUMMV": "-instcombine -reg2mem -mem2reg",
    "GRAMSCHM": "-sink -reg2mem -licm -cfl-anders-aa -sroa",
    "MVT": "-gvn -loop-reduce -cfl-anders-aa -licm",
    "SYR2K": "-loop-reduce -loop-unroll -instcombine -loop-reduce -licm -cfl-anders-aa",
    "SYRK": "-licm -cfl-anders-aa -reg2mem -licm -sroa",
}


def geo(xs):
    return math.exp(sum(math.log(x) for x in xs) / len(xs))


def main() -> int:
    ap = argparse.ArgumentParser()
    ap.add_argument("--size", default="config")
    ap.add_argument("--samples", type=int, default=5)
    ap.add_argument("--skip-ms", type=float, default=50.0)
    ap.add_argument("--benches", nargs="*", default=list(registry.BENCHES))
    ap.add_argument("--out", default=str(ROOT / "profiles" / "variant_report.json"))
    args = ap.parse_args()
    peaks = json.loads((ROOT / "MEASURED_PEAKS.json").read_text()) if (ROOT / "MEASURED_PEAKS.json").exists() else {}
    hbm = float(peaks.get("hbm_gbs", 6650.0))
    be = B200Backend(device=0, samples=1, flush_l2=True)
    out = {"size": args.size, "hbm_peak_gbs": hbm, "benches": {}}
    rows = []
    for bench in args.benches:
        t0 = time.time()
        dims = registry.SIZES[bench][args.size]
        fam = family(bench)
        ws = be.workspace(bench, dims, True, -1)
        times = {}
        for v in range(len(fam.knobs)):
            if not be._supported(bench, v, dims):
                continue
            ws.run(v, samples=1, batch=1, restore=True, flush=False)  # untimed: module load, graph capture, scratch
            first = ws.run(v, samples=1, batch=1, restore=True, flush=True)[0]
            if first > args.skip_ms:
                times[v] = first
                continue
            ms = ws.run(v, samples=args.samples, batch=1, restore=True, flush=True)
            times[v] = statistics.median(ms)
        base = times[0]
        stage0 = {v: t for v, t in times.items() if fam.knobs[v][0] == 0}
        best0 = min(stage0, key=stage0.get)
        best = min(times, key=times.get)
        bytes_, flops = alg_work(bench, dims)
        t1 = None
        if bench in TABLE1:
            vt = fam.select(passmodel.interpret(parse_phase_order(TABLE1[bench])))
            t1 = {"variant": fam.key(vt), "ms": times.get(vt), "speedup": base / times[vt] if vt in times else None}
        rec = {
            "dims": list(dims),
            "variants_timed": len(times),
            "distinct_stage_best": {str(s): min((t for v, t in times.items() if fam.knobs[v][0] == s), default=None)
                                    for s in range(fam.max_stage + 1)},
            "baseline_ms": base,
            "best_phase_variant": fam.key(best0), "best_phase_ms": stage0[best0], "speedup_phase": base / stage0[best0],
            "best_variant": fam.key(best), "best_ms": times[best], "speedup_full": base / times[best],
            "table1": t1,
            "best_gbs": bytes_ / (times[best] * 1e-3) / 1e9, "best_hbm_frac": bytes_ / (times[best] * 1e-3) / 1e9 / hbm,
            "best_tflops": flops / (times[best] * 1e-3) / 1e12,
            "alg_bytes": bytes_, "alg_flops": flops,
            "all_ms": {fam.key(v): t for v, t in times.items()},
            "wall_s": time.time() - t0,
        }
        out["benches"][bench] = rec
        rows.append((bench, rec))
        ws.close()
        be._ws.clear()
        print(f"{bench:9s} base {base:10.3f} ms | phase best {stage0[best0]:9.3f} ms ({base / stage0[best0]:6.2f}x) "
              f"| best {times[best]:9.3f} ms ({base / times[best]:7.2f}x) {fam.key(best):28s} "
              f"| {rec['best_gbs']:7.0f} GB/s {rec['best_tflops']:6.1f} TF/s | {rec['wall_s']:.0f}s", flush=True)
    out["geomean_speedup_phase"] = geo([r["speedup_phase"] for _, r in rows])
    out["geomean_speedup_full"] = geo([r["speedup_full"] for _, r in rows])
    t1 = [r["table1"]["speedup"] for _, r in rows if r["table1"] and r["table1"]["speedup"]]
    out["geomean_speedup_table1"] = geo(t1) if t1 else None
    print(f"geomean speedup: phase-class {out['geomean_speedup_phase']:.3f}x | full {out['geomean_speedup_full']:.3f}x"
          f" | Table-1 orders {out['geomean_speedup_table1']}")
    Path(args.out).parent.mkdir(parents=True, exist_ok=True)
    Path(args.out).write_text(json.dumps(out, indent=1, sort_keys=True) + "\n")
    return 0


if __name__ == "__main__":
    sys.exit(main())
