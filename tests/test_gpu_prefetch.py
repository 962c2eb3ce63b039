"""The batched product path: ``explore`` with the B200 backend's prefetch.

``B200Backend.prefetch_many`` runs the fresh evaluations of a whole order
stream as device batches ahead of ``explore`` (sweep.explore_suite, the path
bench.py times).  The record stream must be the one ``explore`` produces
evaluating candidate by candidate -- same orders, digests, statuses and
eval indices (times are independent device measurements) -- and the
validation outputs served from a batch must be the outputs of a direct run.
"""

from __future__ import annotations

from dataclasses import replace

import numpy as np
import pytest

from paper_1810_10496_b200 import passmodel, registry
from paper_1810_10496_b200.explorer import ExplorationConfig, explore

pytestmark = pytest.mark.gpu

BENCHES = ["ATAX", "GEMM", "FDTD-2D", "SYRK", "GESUMMV"]


def _cases(be):
    return registry.build_suite(be, size="validation", benches=BENCHES)


def _strip(records):
    return [(r.kernel_id, r.order, r.artifact_digest, r.status, r.eval_index) for r in records]


def _cfg(case, seed):
    scale = max(abs(x) for x in case.reference_outputs)
    return ExplorationConfig(num_sequences=150, max_len=64, seed=seed, rtol=1e-4, atol=1e-4 * scale)


def test_prefetched_explore_matches_sequential(gpu_backend):
    from paper_1810_10496_b200.backend.b200 import B200Backend
    from paper_1810_10496_b200.sweep import explore_suite

    cat = passmodel.default_catalog()
    cases = _cases(gpu_backend)
    cfgs = [_cfg(c, 1729 + i) for i, c in enumerate(cases)]
    seq = B200Backend(device=0, samples=1)
    want = {c.id: explore(c, cat, cfg, seq) for c, cfg in zip(cases, cfgs)}
    seq.close()
    be = B200Backend(device=0, samples=1)
    got = explore_suite(cases, cat, cfgs, be)
    assert be.prefetch_batches >= len(cases)  # chunked: at least one batch per kernel
    runs_after_batches = be.device_runs
    for c in cases:
        assert _strip(sorted(got[c.id], key=lambda r: r.eval_index)) == \
            _strip(sorted(want[c.id], key=lambda r: r.eval_index)), c.id
        assert any(r.status.value == "valid" for r in got[c.id])
    assert be.device_runs == runs_after_batches  # every execute() was served from a batch
    assert not be._prefetched and not be._pending  # all consumed
    # a second, warm round (no warm-up runs) gives the same records again
    again = explore_suite(cases, cat, cfgs, be)
    for c in cases:
        assert _strip(again[c.id]) == _strip(got[c.id]) or \
            _strip(sorted(again[c.id], key=lambda r: r.eval_index)) == \
            _strip(sorted(got[c.id], key=lambda r: r.eval_index))
    be.close()


def test_prefetched_validation_outputs_equal_direct_runs(gpu_backend):
    from paper_1810_10496_b200.backend.b200 import B200Backend
    from paper_1810_10496_b200.backend.types import InputKind
    from paper_1810_10496_b200.explorer import draw_orders

    cat = passmodel.default_catalog()
    case = _cases(gpu_backend)[1]  # GEMM: tcgen05 and SIMT variants
    orders = draw_orders(cat, _cfg(case, 7))
    be = B200Backend(device=0, samples=2)
    cands = be.fresh_candidates(case, orders)
    be.prefetch(case, orders)
    direct = B200Backend(device=0, samples=1)
    first = {}
    for o in orders:
        c = be.compile(case, o)
        if c.is_ok and c.artifact.digest not in first:
            first[c.artifact.digest] = o
    assert len(first) == len(cands)
    for digest, o in first.items():
        art = be.compile(case, o).artifact
        got = be.execute(case, o, art, InputKind.VALIDATION)
        ref = direct.execute(case, o, art, InputKind.VALIDATION)
        assert got.status.value == "valid" and got.outputs == ref.outputs
        t = be.execute(case, o, art, InputKind.MEASUREMENT)
        assert t.status.value == "valid" and t.wall_time > 0
    be.close()
    direct.close()


def test_prefetch_with_host_inputs_uses_uploaded_data(gpu_backend):
    """e2e path: the measurement input comes from pinned host memory, uploaded
    asynchronously inside prefetch_many; the measured workspace then holds it."""
    from oracle import oracle as orc
    from paper_1810_10496_b200 import _abi
    from paper_1810_10496_b200.backend.b200 import B200Backend, _Staging
    from paper_1810_10496_b200.explorer import draw_orders

    cat = passmodel.default_catalog()
    small = _cases(gpu_backend)[0]  # ATAX, measured on a larger input than the validation one
    case = registry.kernel_case("ATAX", measurement_dims=(512, 640), reference_outputs=small.reference_outputs)
    _, mdims = registry.parse_descriptor(case.measurement_input)
    host = orc.generate("ATAX", mdims, False, 4242, 3)  # a non-stock input
    be = B200Backend(device=0, samples=1)
    bufs, table = [], {}
    for a, (_, role, _) in enumerate(be.workspace("ATAX", mdims, True, -1).arrays):
        if role == _abi.ROLE_OUT:
            continue
        st = _Staging(_abi.lib(), host[a].nbytes)
        np.ctypeslib.as_array((np.ctypeslib.ctypes.c_float * host[a].size).from_address(st.ptr))[:] = host[a]
        bufs.append(st)
        table[a] = st.ptr
    orders = draw_orders(cat, _cfg(case, 11))
    n = be.prefetch_many([(case, orders)], host_inputs={(case.id, "measurement"): table})
    records = explore(case, cat, _cfg(case, 11), be)
    assert n > 0 and any(r.status.value == "valid" for r in records)
    ws = be.workspace("ATAX", mdims, True, -1)  # tagged as this descriptor's input: not regenerated
    for a in table:
        assert np.array_equal(ws.download(a), host[a])
    be.close()
    for st in bufs:
        st.free()


def test_reference_engine_with_prefetch(gpu_backend, reference_engine):
    """The unmodified reference explore() consumes a prefetched batch."""
    from paper_1810_10496_b200.backend.b200 import B200Backend

    pf = reference_engine
    case = _cases(gpu_backend)[1]
    rcase = pf.KernelCase(case.id, case.source, case.validation_input, case.measurement_input,
                          case.reference_outputs, case.ir_text)
    scale = max(abs(x) for x in case.reference_outputs)
    cfg = pf.ExplorationConfig(num_sequences=120, max_len=48, seed=5, rtol=1e-4, atol=1e-4 * scale)
    cat = pf.PassCatalog.of(*[p.name for p in passmodel.default_catalog().passes])
    from random import Random

    rng = Random(cfg.seed)
    orders = [pf.random_phase_order(cat, cfg.max_len, rng) for _ in range(cfg.num_sequences)]
    be = B200Backend(device=0, samples=1, types=pf.backend.types)
    be.prefetch(rcase, orders)
    be._drain()  # run accounting happens when a batch is collected
    runs = be.device_runs
    records = pf.explore(rcase, cat, cfg, be)
    assert be.device_runs == runs and not be._prefetched
    assert {r.status.value for r in records} <= {"valid", "reused"}
    be.close()
