"""CPU oracle: the C restatement against the independent numpy restatement.

Both are test infrastructure (oracle/).  Kernel arithmetic parity with
PolyBench/GPU is UNPINNED (no PolyBench/GPU source in /root/reference);
agreement of two independent restatements is the pin.
"""

from __future__ import annotations

import numpy as np
import pytest

from oracle import oracle as orc
from oracle import polybench_np as npo
from paper_1810_10496_b200 import registry

orc.set_threads(4)


@pytest.mark.parametrize("bench", registry.BENCHES)
@pytest.mark.parametrize("stock,instance", [(True, -1), (False, 0), (False, 5)])
def test_generators_bit_exact_between_restatements(bench, stock, instance):
    dims = registry.SIZES[bench]["validation"]
    a = orc.generate(bench, dims, stock, 1729, instance)
    b = npo.generate(bench, dims, stock, 1729, instance)
    assert len(a) == len(b)
    for x, y in zip(a, b):
        assert x.dtype == np.float32 and np.array_equal(x, y)


@pytest.mark.parametrize("bench", registry.BENCHES)
@pytest.mark.parametrize("stock,instance", [(True, -1), (False, 2)])
def test_kernels_agree_between_restatements(bench, stock, instance):
    dims = registry.SIZES[bench]["validation"]
    ra = orc.reference(bench, dims, stock, 1729, instance)
    rb = npo.reference(bench, dims, stock, 1729, instance)
    for x, y in zip(ra, rb):
        y64 = y.astype(np.float64)
        tol = np.maximum(1e-6 * np.abs(y64), 1e-6 * float(np.abs(y64).max()))
        assert np.all(np.abs(x.astype(np.float64) - y64) <= tol), bench


def test_random_inputs_differ_per_instance_and_seed():
    a = orc.generate("GEMM", (8, 8, 8), False, 1729, 0)[0]
    b = orc.generate("GEMM", (8, 8, 8), False, 1729, 1)[0]
    c = orc.generate("GEMM", (8, 8, 8), False, 7, 0)[0]
    assert not np.array_equal(a, b) and not np.array_equal(a, c)
    assert a.min() >= 0.0 and a.max() < 1.0


def test_known_values():
    # hand-checked entries of the frozen spec (oracle/SPEC.md)
    A, B, C = orc.generate("GEMM", (4, 4, 4))
    assert A[1 * 4 + 3] == np.float32(3 / 4) and B[2 * 4 + 3] == np.float32(7 / 4) and C[0] == np.float32(0.5)
    x = orc.generate("ATAX", (4, 4))[1]
    assert x[3] == np.float32(3 * np.pi)
    a3 = orc.generate("3DCONV", (4, 4, 4))[0]
    assert a3[(1 * 4 + 2) * 4 + 3] == 1 + 4 + 9
    out = orc.reference("GEMM", (2, 2, 2))[0]
    A, B, C = [t.astype(np.float64).reshape(2, 2) for t in orc.generate("GEMM", (2, 2, 2))]
    assert np.allclose(out.reshape(2, 2), 2123 * C + 32412 * A @ B, rtol=1e-7)
