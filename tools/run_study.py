#!/usr/bin/env python3
"""Cross-application matrix + permutation study (paper Fig. 3 / Fig. 5) on one
GPU, from a campaign's knowledge base:

    python tools/run_study.py --kb profiles/r01_campaign_full/kb.json --out gpurun_out/study
"""

from __future__ import annotations

import argparse
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

from paper_1810_10496_b200 import explorer, registry, study  # noqa: E402
from paper_1810_10496_b200.backend.b200 import B200Backend  # noqa: E402


def main() -> int:
    ap = argparse.ArgumentParser()
    ap.add_argument("--kb", required=True)
    ap.add_argument("--size", default="config")
    ap.add_argument("--trials", type=int, default=1000)
    ap.add_argument("--seed", type=int, default=1729)
    ap.add_argument("--bucket-width", type=float, default=0.05)
    ap.add_argument("--samples", type=int, default=5)
    ap.add_argument("--no-reuse", action="store_true", help="re-measure identical artifacts")
    ap.add_argument("--out", default="gpurun_out/study")
    args = ap.parse_args()
    kb = explorer.KnowledgeBase.load(args.kb)
    be = B200Backend(device=0, samples=args.samples)
    suite = registry.build_suite(be, args.size, benches=[b for b in registry.BENCHES if b in kb.entries])
    cfg = explorer.ExplorationConfig(rtol=1e-4, final_reps=1, final_random_inputs=1)
    study.run_study(suite, kb, be, cfg, args.out, trials=args.trials, seed=args.seed,
                    bucket_width=args.bucket_width, reuse=not args.no_reuse)
    print(f"device runs {be.device_runs}, kernel launches {be.kernel_launches}")
    return 0


if __name__ == "__main__":
    sys.exit(main())
