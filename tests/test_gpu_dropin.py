"""Drop-in property on the B200: an engine with its *own* value types (a second,
independently imported copy of the engine package, standing in for the
reference ``phaseforge`` whose enums are compared by identity) drives
``B200Backend(types=...)`` through explore -> finalize -> reduce_order."""

from __future__ import annotations

import importlib.util
import sys
from pathlib import Path

import numpy as np
import pytest

from paper_1810_10496_b200 import registry

pytestmark = pytest.mark.gpu

PKG = Path(__file__).resolve().parent.parent / "paper_1810_10496_b200"


def _foreign_engine():
    name = "foreign_engine"
    if name in sys.modules:
        return sys.modules[name]
    spec = importlib.util.spec_from_file_location(name, PKG / "__init__.py", submodule_search_locations=[str(PKG)])
    mod = importlib.util.module_from_spec(spec)
    sys.modules[name] = mod
    spec.loader.exec_module(mod)
    return mod


def test_foreign_engine_drives_b200_backend():
    from oracle import oracle as orc
    from paper_1810_10496_b200.backend.b200 import B200Backend

    fe = _foreign_engine()
    ftypes = sys.modules["foreign_engine.backend.types"]
    from paper_1810_10496_b200.backend import types as own

    assert ftypes.ExecutionStatus is not own.ExecutionStatus  # distinct enum classes
    be = B200Backend(device=0, types=ftypes, samples=3)
    bench = "GEMM"
    dims = registry.SIZES[bench]["validation"]
    ref = np.concatenate(orc.reference(bench, dims)).astype(np.float64)
    case = registry.kernel_case(bench, "polybench")
    fcase = fe.KernelCase(case.id, case.source, case.validation_input, case.measurement_input,
                          tuple(ref.tolist()), case.ir_text)
    cfg = fe.ExplorationConfig(num_sequences=60, max_len=24, top_k=3, final_reps=3, final_random_inputs=3,
                               rtol=1e-4, atol=1e-4 * float(np.abs(ref).max()))
    catalog = fe.PassCatalog.of("cfl-anders-aa", "licm", "loop-reduce", "loop-unroll", "reg2mem", "sroa",
                                "slp-vectorizer", "loop-interchange", "loop-data-prefetch", "gvn")
    records = fe.explore(fcase, catalog, cfg, be)
    statuses = {r.status.value for r in records}
    assert "valid" in statuses and statuses <= {"valid", "reused"}
    assert any(r.status.value == "reused" for r in records)  # identical SASS -> REUSED
    best, best_time = fe.finalize(fcase, records, cfg, be)
    reduced = fe.reduce_order(fcase, best, be, 0.05, cfg)
    assert len(reduced) <= len(best)
    base = fe.measure_average(be, fcase, fe.PhaseOrder(), 3, cfg)
    assert best_time < base  # the specialised variant beats the nvcc-shaped baseline
    be.close()


def test_unmodified_reference_engine_drives_b200_backend(reference_engine):
    """The reference's own explore -> finalize -> reduce_order ->
    measure_average (imported unmodified from /root/reference or its pip
    install in baseline/_ref) on B200Backend(types=phaseforge.backend.types):
    the INTEGRATION.md §2 claim, on hardware."""
    from oracle import oracle as orc
    from paper_1810_10496_b200.backend.b200 import B200Backend

    pf = reference_engine
    assert pf.__file__ and "paper_1810_10496_b200" not in pf.__file__
    be = B200Backend(device=0, types=pf.backend.types, samples=3)
    for bench in ("GEMM", "ATAX"):
        dims = registry.SIZES[bench]["validation"]
        ref = np.concatenate(orc.reference(bench, dims)).astype(np.float64)
        case = registry.kernel_case(bench, "polybench")
        rcase = pf.KernelCase(case.id, case.source, case.validation_input, case.measurement_input,
                              tuple(ref.tolist()), case.ir_text)
        cfg = pf.ExplorationConfig(num_sequences=80, max_len=24, top_k=3, final_reps=3, final_random_inputs=3,
                                   rtol=1e-4, atol=1e-4 * float(np.abs(ref).max()))
        catalog = pf.PassCatalog.of("cfl-anders-aa", "licm", "loop-reduce", "loop-unroll", "reg2mem", "sroa",
                                    "slp-vectorizer", "loop-interchange", "loop-data-prefetch", "gvn")
        records = pf.explore(rcase, catalog, cfg, be)
        assert all(type(r.status) is pf.RecordStatus for r in records)
        assert any(r.status is pf.RecordStatus.VALID for r in records)
        assert any(r.status is pf.RecordStatus.REUSED for r in records)
        best, best_time = pf.finalize(rcase, records, cfg, be)
        with be.digest_timing():
            reduced = pf.reduce_order(rcase, best, be, 0.01, cfg)
        assert len(reduced) <= len(best)
        assert be.compile(rcase, reduced).artifact.digest == be.compile(rcase, best).artifact.digest or \
            len(reduced) < len(best)
        base = pf.explorer.measure_average(be, rcase, pf.PhaseOrder(), 3, cfg)
        assert best_time < base, bench
    be.close()
