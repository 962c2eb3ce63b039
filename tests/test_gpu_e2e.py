"""The end-to-end host-buffer path (bench.py's e2e number): inputs uploaded
from host memory inside pf_eval_batch, outputs read back into host buffers,
checked against the oracle; plus device-side compare/checksum helpers."""

from __future__ import annotations

import ctypes

import numpy as np
import pytest

from oracle import oracle as orc
from paper_1810_10496_b200 import registry

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("bench", ["ATAX", "MVT", "GEMM", "FDTD-2D"])
def test_eval_batch_host_buffers_match_oracle(bench, gpu_backend):
    from paper_1810_10496_b200.backend.b200 import family
    from paper_1810_10496_b200.sweep import evaluate_round

    dims = registry.SIZES[bench]["validation"]
    inputs = orc.generate(bench, dims, False, 99, 4)           # a random input instance, on the host
    ref = orc.run(bench, dims, [a.copy() for a in inputs])
    ws = gpu_backend.workspace(bench, dims, True, -1)           # device holds the *stock* input
    fam = family(bench)
    variants = [0, len(fam.knobs) - 1]
    host_in = {ws: {a: inputs[a].ctypes.data for a, (_, role, _) in enumerate(ws.arrays) if role != 2}}
    outs = {a: np.zeros(ws.elems[a], np.float32) for a, (_, _, o) in enumerate(ws.arrays) if o}
    host_out = {ws: {a: buf.ctypes.data for a, buf in outs.items()}}
    for v in variants:
        ms, total = evaluate_round([(ws, v)], host_in=host_in, host_out=host_out)
        assert ms[0] > 0 and total >= ms[0]
        for a, buf in outs.items():
            r = ref[a].astype(np.float64)
            tol = np.maximum(1e-4 * np.abs(r), 1e-4 * np.abs(r).max())
            assert np.all(np.abs(buf - r) <= tol), (bench, fam.key(v), a)
    ws.input_tag = None  # device now holds the uploaded input


def test_device_compare_and_checksum(gpu_backend):
    from paper_1810_10496_b200.backend.b200 import family

    bench, dims = "SYRK", registry.SIZES["SYRK"]["validation"]
    fam = family(bench)
    a = gpu_backend.workspace(bench, dims, True, -1)
    from paper_1810_10496_b200.backend.b200 import Workspace

    b = Workspace(0, bench, dims)
    b.generate(True, gpu_backend.seed, -1)
    a.run(0)
    b.run(len(fam.knobs) - 1)  # tcgen05 variant
    err, bad = b.compare(a, 1e-4, 1e-4)
    assert bad == 0 and err < 1.0
    s_a, abs_a = a.checksum(1)
    s_b, abs_b = b.checksum(1)
    assert abs(s_a - s_b) <= 1e-4 * abs_a
    b.close()
