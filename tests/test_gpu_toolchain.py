"""Process-level drop-in on the B200: ``ToolchainBackend`` over ``pftool``
(one runner process per execution, toolchain.py:216-273) returns the same
validation and random-input outputs as the in-process ``B200Backend``, and
the explore -> finalize loop runs through it."""

from __future__ import annotations

import json

import pytest

from paper_1810_10496_b200 import explorer, passmodel, pftool
from paper_1810_10496_b200.backend.b200 import B200Backend
from paper_1810_10496_b200.backend.toolchain import ToolchainBackend, ToolchainSpec
from paper_1810_10496_b200.backend.types import ExecutionStatus, InputKind, KernelCase
from paper_1810_10496_b200.catalog import PhaseOrder

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def suite(tmp_path_factory):
    out = tmp_path_factory.mktemp("tcsuite")
    be = B200Backend()
    pftool.write_suite(out, "validation", benches=["GEMM", "BICG"], backend=be)
    data = json.loads((out / "suite.json").read_text())
    cases = [KernelCase(k["id"], out / k["source"], k["validation_input"], k["measurement_input"],
                        tuple(k["reference_outputs"]), (out / k["ir_path"]).read_text()) for k in data["kernels"]]
    spec = ToolchainSpec.load(out / "toolchain.json")
    return cases, ToolchainBackend(spec), be


def _same(a, b):
    """Report values round-trip bit-exactly (repr); variants whose column
    reductions use float atomics (fused BLAS-2) may differ run to run in the
    last bits, so the bar is 1e-6 relative, far inside the 1e-4 parity bar."""
    assert len(a) == len(b)
    for x, y in zip(a, b):
        assert abs(x - y) <= 1e-6 * max(abs(x), abs(y), 1e-30), (x, y)


def test_runner_outputs_equal_in_process(suite):
    cases, tc, be = suite
    orders = [PhaseOrder(), PhaseOrder.of("cfl-anders-aa", "licm", "loop-unroll", "bb-vectorize"),
              PhaseOrder.of("cfl-anders-aa", "licm", "loop-interchange", "loop-data-prefetch")]
    for case in cases:
        own = KernelCase(case.id, f"polybench-gpu:{case.id}", case.validation_input, case.measurement_input,
                         case.reference_outputs, case.ir_text)
        for order in orders:
            a, b = tc.compile(case, order), be.compile(own, order)
            assert a.artifact.digest == b.artifact.digest
            ra = tc.execute(case, order, a.artifact, InputKind.VALIDATION)
            rb = be.execute(own, order, b.artifact, InputKind.VALIDATION)
            assert ra.status is rb.status is ExecutionStatus.VALID
            _same(ra.outputs, rb.outputs)
            ra = tc.execute(case, order, a.artifact, InputKind.VALIDATION, random_input_index=3)
            rb = be.execute(own, order, b.artifact, InputKind.VALIDATION, random_input_index=3)
            _same(ra.outputs, rb.outputs)
            m = tc.execute(case, order, a.artifact, InputKind.MEASUREMENT)
            assert m.status is ExecutionStatus.VALID and m.wall_time > 0 and m.outputs == ()


def test_explore_finalize_through_runner(suite):
    cases, tc, _ = suite
    case = cases[0]
    cfg = explorer.ExplorationConfig(num_sequences=6, max_len=12, top_k=2, final_reps=2, final_random_inputs=2,
                                     rtol=1e-4, atol=1e-4 * max(abs(x) for x in case.reference_outputs))
    records = explorer.explore(case, passmodel.default_catalog(), cfg, tc)
    assert len(records) == 6
    assert all(r.status is not explorer.RecordStatus.BROKEN_REPORT for r in records)
    best, t = explorer.finalize(case, records, cfg, tc)
    assert t > 0
