#!/usr/bin/env python3
"""Run the full 15-benchmark campaign on one GPU (BASELINE configs[4] shape):
explore (num_sequences orders per kernel) -> finalize -> reduce -> KB ->
speedup report -> leave-one-out 1-NN/3-NN transfer."""

from __future__ import annotations

import argparse
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

from paper_1810_10496_b200 import registry  # noqa: E402
from paper_1810_10496_b200.backend.b200 import B200Backend  # noqa: E402
from paper_1810_10496_b200.campaign import run_campaign  # noqa: E402
from paper_1810_10496_b200.explorer import ExplorationConfig  # noqa: E402


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
    args = ap.parse_args()
    be = B200Backend(device=0, samples=args.samples)
    suite = registry.build_suite(be, args.size, benches=args.benches)
    cfg = ExplorationConfig(num_sequences=args.num_sequences, max_len=args.max_len, top_k=args.top_k,
                            final_reps=args.final_reps, final_random_inputs=args.final_random_inputs)
    res = run_campaign(suite, be, cfg, loo_trials=args.loo_trials, out_dir=args.out)
    print(f"done in {res.seconds:.0f}s; device runs {be.device_runs}, kernel launches {be.kernel_launches}")
    return 0


if __name__ == "__main__":
    sys.exit(main())
