"""bench.py under torchrun with 2 ranks on one GPU (gloo control plane, both
ranks on cuda:0 through the Dist test hooks): every rank must run through
the same sequence of collectives and rank 0 must print one JSON line that
aggregates over both ranks.  Guards the N > 1 path the driver's scaling run
uses (it once called a collective from rank 0's JSON block only)."""

from __future__ import annotations

import json
import os
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu

ROOT = Path(__file__).resolve().parent.parent


def test_bench_two_ranks_one_gpu():
    env = dict(os.environ, PF_DIST_ONE_DEVICE="1", PF_DIST_BACKEND="gloo")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", "29677", "bench.py", "--gpus", "2", "--steps", "1",
           "--warmup", "3", "--num-sequences", "60", "--e2e-steps", "1", "--sweep-orders", "3", "--cpu-orders", "0"]
    r = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=1500)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["value"] > 0 and d["e2e"]["value"] > 0
    assert d["sweep"]["fresh_evaluations"] > 0 and d["gpu_launches"] > 0
