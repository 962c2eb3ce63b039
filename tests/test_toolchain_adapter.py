"""Process-level drop-in: the four compile stages of
``pftool`` behind a ToolchainSpec produce exactly the artifacts
``B200Backend.compile`` produces (same bytes, same digests, same failure
classes).  CPU-only: compile is a variant lookup plus a host-side
``pf_variant_supported`` check.  The runner half is in test_gpu_toolchain.py.

When /root/reference is present (this container, not the GPU box) the stock
reference ``ToolchainBackend`` drives the adapter too.
"""

from __future__ import annotations

import sys
from pathlib import Path
from random import Random

import pytest

from paper_1810_10496_b200 import passmodel, pftool, registry
from paper_1810_10496_b200.backend.b200 import B200Backend
from paper_1810_10496_b200.backend.toolchain import ToolchainBackend, ToolchainSpec, parse_report
from paper_1810_10496_b200.backend.types import CompileStatus, KernelCase
from paper_1810_10496_b200.catalog import PhaseOrder, random_phase_order

REF_TOOLCHAIN = Path("/root/reference/pkg/src/phaseforge/backend/toolchain.py")


def _case(tmp: Path, bench: str, measurement: str = "polybench") -> KernelCase:
    own = registry.kernel_case(bench, measurement)
    src = tmp / f"{bench}.pfk"
    src.write_text(f"{registry.source_of(bench)}\nvalidation {own.validation_input}\n"
                   f"measurement {own.measurement_input}\n")
    return KernelCase(own.id, src, own.validation_input, own.measurement_input, (0.0,), own.ir_text)


def _orders(n: int, seed: int) -> list[PhaseOrder]:
    rng = Random(seed)
    cat = passmodel.default_catalog()
    return [PhaseOrder()] + [random_phase_order(cat, 12, rng) for _ in range(n)]


@pytest.fixture(scope="module")
def spec(tmp_path_factory):
    work = tmp_path_factory.mktemp("pftool")
    return ToolchainSpec.from_json_dict(pftool.toolchain_spec_dict(work_dir=str(work / "work")))


@pytest.mark.parametrize("bench", ["GEMM", "ATAX", "FDTD-2D"])
def test_adapter_artifacts_match_in_process_backend(spec, tmp_path, bench):
    tc = ToolchainBackend(spec)
    b2 = B200Backend()
    case = _case(tmp_path, bench)
    for order in _orders(5, 1729 + len(bench)):
        a = tc.compile(case, order)
        b = b2.compile(registry.kernel_case(bench, "polybench"), order)
        assert a.status is b.status is CompileStatus.OK
        assert a.artifact.digest == b.artifact.digest
        assert a.artifact.content == b.artifact.content


def test_adapter_failure_classes(spec, tmp_path):
    tc = ToolchainBackend(spec)
    case = _case(tmp_path, "ATAX")
    # a stage-2 order (loop-data-prefetch after interchange) on an input the fused
    # kernel refuses: odd column count -> CODEGEN_FAILURE, as in B200Backend.compile
    bad = KernelCase(case.id, case.source, case.validation_input, case.measurement_input, (0.0,), None)
    src = Path(case.source)
    src.write_text(f"{registry.source_of('ATAX')}\nvalidation {registry.describe('ATAX', (33, 33))}\n")
    order = PhaseOrder.of("cfl-anders-aa", "licm", "loop-interchange", "loop-data-prefetch")
    b2 = B200Backend()
    odd = KernelCase(case.id, registry.source_of("ATAX"), registry.describe("ATAX", (33, 33)),
                     registry.describe("ATAX", (33, 33)), (0.0,), None)
    want = b2.compile(odd, order).status
    assert want is CompileStatus.CODEGEN_FAILURE
    assert tc.compile(bad, order).status is want
    # a missing kernel source is a configuration error
    from paper_1810_10496_b200.backend.types import BackendError

    with pytest.raises(BackendError):
        tc.compile(KernelCase("X", tmp_path / "missing.pfk", "a", "b", (0.0,), None), order)


def test_report_grammar_of_runner_output():
    text = f"TIME {0.00125!r}\nOUT 3\n{1.5!r}\n{-2.0!r}\n{3e-07!r}\n"
    assert parse_report(text) == (0.00125, (1.5, -2.0, 3e-07))
    assert parse_report("TIME 0.001\nOUT 0\n") == (0.001, ())
    assert parse_report("TIME 0\nOUT 0\n") is None


def test_pftool_rejects_malformed_input(tmp_path):
    src = tmp_path / "x.pfk"
    src.write_text("not-a-kernel\n")
    assert pftool.main(["frontend", str(src), str(tmp_path / "o.ir")]) == 1
    src.write_text("polybench-gpu:GEMM\n")
    assert pftool.main(["frontend", str(src), str(tmp_path / "o.ir")]) == 0
    assert pftool.main(["opt", str(tmp_path / "o.ir"), str(tmp_path / "p.ir"), "-Not_A_Pass"]) == 1
    assert pftool.main(["opt", str(tmp_path / "o.ir"), str(tmp_path / "p.ir"), "-licm"]) == 0
    assert pftool.main(["bogus"]) == 2


@pytest.mark.skipif(not REF_TOOLCHAIN.exists(), reason="reference tree not mounted")
def test_stock_reference_toolchain_drives_adapter(spec, tmp_path):
    """The unmodified reference ToolchainBackend, its own types, our stages."""
    sys.path.insert(0, str(REF_TOOLCHAIN.parents[2]))
    try:
        saved = {k: v for k, v in sys.modules.items() if k == "phaseforge" or k.startswith("phaseforge.")}
        for k in saved:
            del sys.modules[k]
        import phaseforge.backend.toolchain as rtc  # the reference's own module
        import phaseforge.backend.types as rtypes
        from phaseforge.catalog import PhaseOrder as RPhaseOrder
        from phaseforge.catalog import PassId as RPassId
    finally:
        sys.path.pop(0)
    try:
        rspec = rtc.ToolchainSpec.from_json_dict(pftool.toolchain_spec_dict(work_dir=str(tmp_path / "w")))
        rbe = rtc.ToolchainBackend(rspec)
        own = _case(tmp_path, "GEMM")
        rcase = rtypes.KernelCase(own.id, own.source, own.validation_input, own.measurement_input, (0.0,), None)
        b2 = B200Backend()
        for order in _orders(3, 7):
            rorder = RPhaseOrder(tuple(RPassId(p.name) for p in order.passes))
            got = rbe.compile(rcase, rorder)
            assert got.status is rtypes.CompileStatus.OK
            assert got.artifact.digest == b2.compile(registry.kernel_case("GEMM", "polybench"), order).artifact.digest
    finally:
        for k in [k for k in sys.modules if k == "phaseforge" or k.startswith("phaseforge.")]:
            del sys.modules[k]
        sys.modules.update(saved)
