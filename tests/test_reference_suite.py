"""The reference's own 180 tests, unmodified, against the restated engine.

tools/phaseforge_alias.py maps ``import phaseforge`` onto
paper_1810_10496_b200 (catalog, irfeat, explorer, advisor, results,
backend.types); the reference's simulator / toolchain / CLI sources -- its
test doubles and front door, out of scope for the B200 build -- execute on
top of the restated types.  Skipped where /root/reference is absent.
"""

from __future__ import annotations

import os
import subprocess
import sys
from pathlib import Path

import pytest

from conftest import ROOT, have_reference

REF_TESTS = Path("/root/reference/pkg/tests")


@pytest.mark.skipif(not have_reference(), reason="reference package not available")
def test_reference_test_suite_passes_on_restated_engine(tmp_path):
    env = dict(os.environ)
    env["PYTHONDONTWRITEBYTECODE"] = "1"
    env["PYTHONPATH"] = os.pathsep.join([str(ROOT), str(ROOT / "tools"), str(REF_TESTS)])
    proc = subprocess.run(
        [sys.executable, "-m", "pytest", "-p", "phaseforge_alias", "-p", "no:cacheprovider", "--rootdir",
         str(tmp_path), "-q", str(REF_TESTS)],
        cwd=tmp_path, env=env, capture_output=True, text=True, timeout=900,
    )
    tail = "\n".join(proc.stdout.splitlines()[-15:])
    assert proc.returncode == 0, tail + proc.stderr[-2000:]
    assert "180 passed" in tail, tail
