#!/usr/bin/env python3
"""Host timeline of the bench's explore() steps (diagnostic): wraps the
device worker's pf_eval_batch calls and explore_suite with perf_counter
stamps, runs bench.main() with the given arguments, and prints where the
device sat idle inside the steps (before the first batch, between batches,
after the last one)."""
import json
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import bench  # noqa: E402
from paper_1810_10496_b200 import sweep  # noqa: E402
from paper_1810_10496_b200.backend import b200  # noqa: E402

LOG = {"batches": [], "steps": []}
_orig_submit = b200.B200Backend._worker_submit


def _submit(self, items):
    t_sub = time.perf_counter()
    fut = _orig_submit(self, items)
    rec = {"n": len(items), "submit": t_sub}
    LOG["batches"].append(rec)

    def done(f):
        rec["done"] = time.perf_counter()
    fut.add_done_callback(done)
    return fut


_orig_suite = sweep.explore_suite


def _suite(*a, **k):
    t0 = time.perf_counter()
    out = _orig_suite(*a, **k)
    LOG["steps"].append((t0, time.perf_counter()))
    return out


b200.B200Backend._worker_submit = _submit
sweep.explore_suite = _suite
bench.explore_suite = _suite

sys.argv = ["bench.py"] + sys.argv[1:]
rc = bench.main()
out = Path(sys.argv[0]).parent
steps = LOG["steps"]
for i, (s0, s1) in enumerate(steps):
    bs = [b for b in LOG["batches"] if s0 <= b["submit"] <= s1]
    if not bs:
        continue
    first_sub = min(b["submit"] for b in bs)
    last_done = max(b.get("done", s1) for b in bs)
    print(f"step {i:2d}: {1e3 * (s1 - s0):7.1f} ms, {len(bs):2d} batches ({sum(b['n'] for b in bs)} items), "
          f"first submit +{1e3 * (first_sub - s0):5.1f} ms, last batch done {1e3 * (s1 - last_done):5.1f} ms "
          f"before the step ends; submits at "
          + " ".join(f"{1e3 * (b['submit'] - s0):.0f}" for b in bs)
          + " | done at " + " ".join(f"{1e3 * (b.get('done', s1) - s0):.0f}" for b in bs))
json.dump(LOG, open("gpurun_out/batch_gaps.json", "w"))
sys.exit(rc)
