"""Pins ``study.py`` (cross-application matrix, permutation study) against the
reference front door byte for byte.

Run A: the unmodified reference CLI (`/root/reference/pkg/src/phaseforge/
cli.py` ``explore``, ``experiments cross-apply``, ``experiments permute``) on
its deterministic SimulatorBackend.  Run B: ``study.cross_apply_matrix`` and
``study.permutation_study`` on the same simulator (bound to this package's
types through tools/phaseforge_alias.py), the same KB, suite and flags.
``matrix.csv`` and ``permute.csv`` must be identical.  Needs the reference
tree (this container); skipped on the GPU box.
"""

from __future__ import annotations

import json
import os
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
REF_SRC = Path("/root/reference/pkg/src")

pytestmark = pytest.mark.skipif(not REF_SRC.exists(), reason="reference tree not mounted")

IR = "func body {\nentry:\n  load\n  store\n  ret\n}\n"
PASSES = ["licm", "gvn", "instcombine", "loop-unroll", "sroa", "mem2reg", "dse", "sink"]
KERNELS = [
    {"id": "ka", "model": {"baseline_time": 1.0, "seed_salt": 3, "noise_amplitude": 0.002,
                           "motifs": [{"passes": ["licm", "gvn"], "multiplier": 0.6},
                                      {"passes": ["loop-unroll"], "multiplier": 0.8}]}},
    {"id": "kb", "model": {"baseline_time": 2.0, "seed_salt": 11, "noise_amplitude": 0.002,
                           "failure_rates": [0.05, 0.05, 0.0],
                           "motifs": [{"passes": ["sroa", "mem2reg", "licm"], "multiplier": 0.5}]}},
    {"id": "kc", "model": {"baseline_time": 0.5, "seed_salt": 5, "noise_amplitude": 0.002,
                           "motifs": [{"passes": ["instcombine", "dse"], "multiplier": 0.7},
                                      {"passes": ["gvn", "sink"], "multiplier": 0.9}]}},
]
FLAGS = ["--num-sequences", "80", "--max-len", "10", "--final-reps", "3", "--final-random-inputs", "3",
         "--top-k", "4", "--seed", "1729"]

REF_RUN = """
import sys
sys.path.insert(0, {ref!r})
from phaseforge.cli import main
d = {d!r}
flags = {flags!r}
common = ["--suite", d + "/suite.json", "--out-dir", d + "/A"] + flags
assert main(["explore", "--catalog", d + "/catalog.txt"] + common) == 0
assert main(["experiments", "cross-apply", "--kb", d + "/A/kb.json"] + common) == 0
assert main(["experiments", "permute", "--kb", d + "/A/kb.json", "--trials", "40", "--bucket-width", "0.1"]
            + common) == 0
"""

OWN_RUN = """
import sys
sys.path[:0] = [{root!r}, {root!r} + "/tools"]
import phaseforge_alias  # noqa: F401  (reference simulator + CLI bound to this package's types)
import phaseforge
from pathlib import Path
from paper_1810_10496_b200 import explorer, results, study
d = Path({d!r})
kernels = phaseforge.cli._load_suite(d / "suite.json")
kb = explorer.KnowledgeBase.load(d / "A" / "kb.json")
kernels = [k for k in kernels if k.id in kb.entries]
be = phaseforge.backend.SimulatorBackend()
cfg = explorer.ExplorationConfig(num_sequences=80, max_len=10, seed=1729, top_k=4, final_reps=3,
                                 final_random_inputs=3, rtol=0.01, atol=1e-6)
(d / "B").mkdir()
m = study.cross_apply_matrix(kernels, kb, be, cfg, per_kernel_tolerance=False)
results.export_matrix_csv(m, d / "B" / "matrix.csv")
be = phaseforge.backend.SimulatorBackend()
p = study.permutation_study(kernels, kb, be, cfg, trials=40, seed=1729, bucket_width=0.1,
                            per_kernel_tolerance=False)
study.write_permute_csv(p, d / "B" / "permute.csv")
"""


def _run(code: str) -> None:
    env = {k: v for k, v in os.environ.items() if k != "PYTHONPATH"}
    done = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, env=env, timeout=300)
    assert done.returncode == 0, done.stderr[-3000:]


def test_study_matches_reference_cli(tmp_path):
    (tmp_path / "catalog.txt").write_text("\n".join(PASSES) + "\n")
    suite = {"kernels": [dict(k, ir=IR, validation_input="small", measurement_input="full",
                              reference_outputs=[1.0, 2.0, 3.0]) for k in KERNELS]}
    (tmp_path / "suite.json").write_text(json.dumps(suite))
    _run(REF_RUN.format(ref=str(REF_SRC), d=str(tmp_path), flags=FLAGS))
    _run(OWN_RUN.format(root=str(ROOT), d=str(tmp_path)))
    for name in ("matrix.csv", "permute.csv"):
        want = (tmp_path / "A" / name).read_text()
        got = (tmp_path / "B" / name).read_text()
        assert got == want, name
    assert (tmp_path / "A" / "permute.csv").read_text().count("\n") > 3
