"""The reference arm of bench.py (oracle/ref_arm.py, oracle/pf_cpu_runner):
the runner honours the reference runner protocol (toolchain.py:216-273, the
TIME/OUT report of :178-213) with the oracle's outputs, and the unmodified
reference explore() drives it through ToolchainBackend."""

from __future__ import annotations

import subprocess

import numpy as np
import pytest

from oracle import oracle as orc
from oracle import ref_arm
from paper_1810_10496_b200 import registry
from paper_1810_10496_b200.backend.toolchain import parse_report


@pytest.fixture(scope="module")
def runner():
    return ref_arm.build_runner()


@pytest.mark.parametrize("bench", ["GEMM", "ATAX", "CORR", "FDTD-2D"])
def test_runner_report_is_the_oracle(bench, runner, tmp_path):
    art = tmp_path / "a.art"
    art.write_text("x")
    dims = registry.SIZES[bench]["validation"]
    for data, stock, inst in ((registry.describe(bench, dims), True, -1),
                              (registry.describe(bench, dims) + "#3", False, 3)):
        out = subprocess.run([str(runner), str(art), data, "validation"], capture_output=True, text=True, check=True)
        parsed = parse_report(out.stdout)
        assert parsed is not None
        t, values = parsed
        ref = np.concatenate(orc.reference(bench, dims, stock, 1729, inst)).astype(np.float64)
        assert t > 0 and np.allclose(np.array(values), ref, rtol=1e-6, atol=0)
    out = subprocess.run([str(runner), str(art), registry.describe(bench, dims), "measurement"],
                         capture_output=True, text=True, check=True)
    assert parse_report(out.stdout)[1] == ()


def test_runner_rejects_bad_descriptors(runner, tmp_path):
    art = tmp_path / "a.art"
    art.write_text("x")
    for data in ("NOPE:n=4", "GEMM", "GEMM:ni=0,nj=4,nk=4"):
        assert subprocess.run([str(runner), str(art), data, "validation"], capture_output=True).returncode == 2


def test_reference_explore_through_toolchain(runner):
    pf = ref_arm.reference_engine()
    if pf is None:
        pytest.skip("reference package not available")
    work = ref_arm.workdir()
    be = ref_arm.toolchain_backend(pf, work)
    dims = {"GEMM": registry.SIZES["GEMM"]["validation"]}
    cases = ref_arm.kernel_cases(pf, ["GEMM"], dims, work)
    fresh, recs, secs = ref_arm.explore_step(pf, be, cases, ["licm", "gvn", "sroa"], 3, 1729)
    assert recs == 3 and fresh >= 1 and ref_arm.explore_step.valid == fresh and secs > 0
