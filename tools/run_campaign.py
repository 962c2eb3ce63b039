#!/usr/bin/env python3
"""Run the full 15-benchmark campaign (BASELINE configs[4] shape):
explore (num_sequences orders per kernel) -> finalize -> reduce -> KB ->
speedup report -> leave-one-out 1-NN/3-NN transfer.

One GPU: ``python tools/run_campaign.py``.  N GPUs (one process each; the
kernels are sharded over the ranks with device affinity):
``python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1
tools/run_campaign.py``."""

from __future__ import annotations

import argparse
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

from paper_1810_10496_b200 import passmodel, registry  # noqa: E402
from paper_1810_10496_b200.catalog import PassCatalog  # noqa: E402
from paper_1810_10496_b200.backend.b200 import B200Backend  # noqa: E402
from paper_1810_10496_b200.campaign import run_campaign  # noqa: E402
from paper_1810_10496_b200.dist import Dist  # noqa: E402
from paper_1810_10496_b200.explorer import ExplorationConfig  # noqa: E402


# seconds per kernel of the round-1 single-GPU full sweep (profiles/r01_campaign_full):
# the LPT weights of the kernel-to-rank assignment
KERNEL_COSTS = {"2DCONV": 3, "3DCONV": 3, "2MM": 27, "3MM": 18, "ATAX": 7, "BICG": 7, "CORR": 165, "COVAR": 169,
                "FDTD-2D": 14, "GEMM": 2, "GESUMMV": 4, "GRAMSCHM": 882, "MVT": 7, "SYR2K": 28, "SYRK": 21}


def main() -> int:
    ap = argparse.ArgumentParser()
    ap.add_argument("--size", default="config")
    ap.add_argument("--num-sequences", type=int, default=1000)
    ap.add_argument("--max-len", type=int, default=256)
    ap.add_argument("--top-k", type=int, default=10)
    ap.add_argument("--final-reps", type=int, default=30)
    ap.add_argument("--final-random-inputs", type=int, default=30)
    ap.add_argument("--loo-trials", type=int, default=100)
    ap.add_argument("--benches", nargs="*", default=list(registry.BENCHES))
    ap.add_argument("--out", default="gpurun_out/campaign")
    ap.add_argument("--samples", type=int, default=5)
    ap.add_argument("--catalog", default="staging", choices=("staging", "table1"),
                    help="staging: the 20 Table-1 passes + the 4 staging passes (passmodel default); "
                         "table1: the paper's 20 Table-1 passes only (BASELINE configs[4])")
    ap.add_argument("--ir", default="structural", choices=registry.IR_SOURCES,
                    help="feature source: PolyBench-shaped IR (default) or IR recovered from the baseline PTX")
    args = ap.parse_args()
    dist = Dist()
    be = B200Backend(device=dist.local, samples=args.samples)
    suite = registry.build_suite(be, args.size, benches=args.benches, ir=args.ir)
    cfg = ExplorationConfig(num_sequences=args.num_sequences, max_len=args.max_len, top_k=args.top_k,
                            final_reps=args.final_reps, final_random_inputs=args.final_random_inputs)
    log = print if dist.rank == 0 else (lambda *a, **k: None)
    catalog = (passmodel.default_catalog() if args.catalog == "staging"
               else PassCatalog.of(*passmodel.TABLE1_PASSES))
    res = run_campaign(suite, be, cfg, catalog=catalog, loo_trials=args.loo_trials, out_dir=args.out, dist=dist,
                       log=log, kernel_costs=KERNEL_COSTS)
    runs = dist.sum(be.device_runs)
    launches = dist.sum(be.kernel_launches)
    seconds = dist.max(res.seconds)
    log(f"done in {seconds:.0f}s on {dist.world} GPU(s); device runs {runs:.0f}, kernel launches {launches:.0f}")
    dist.close()
    return 0


if __name__ == "__main__":
    sys.exit(main())
