"""The two tensor-core arithmetic modes of the stage-2 contractions.

* 3xFP16 (default for products that run pre-split, tc_f16.cuh): operands are
  scaled by a power of two and split into fp16 hi / lo images.  Its scaling
  is exercised here with inputs spanning many decades and both signs (the
  PolyBench inputs are all O(1)), against an fp64 numpy product, at sizes
  where the f16 path is taken (SYRK from n = 256; plain products from ~1.6k).
* 3xTF32 (PF_TC_F16=0, with CORR/COVAR's two-launch fp32 statistics) stays
  available for A/B runs: the tensor-core parity tests are re-run in a
  subprocess with it selected.

Tolerance as everywhere: |t - r| <= max(1e-4 max|r|, 1e-4 |r|).
"""

from __future__ import annotations

import os
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = Path(__file__).resolve().parent.parent
RTOL = 1e-4


def _check(got, ref):
    ref = ref.astype(np.float64)
    tol = np.maximum(RTOL * np.abs(ref).max(), RTOL * np.abs(ref))
    err = np.abs(got.astype(np.float64) - ref)
    worst = float((err / tol).max())
    assert worst <= 1.0, f"max error / tolerance = {worst:.3g}"
    return worst


def _wide(rng, shape, decades=8):
    mag = 10.0 ** rng.uniform(-decades / 2, decades / 2, size=shape)
    return (mag * rng.choice([-1.0, 1.0], size=shape)).astype(np.float32)


def _stage2(bench):
    from paper_1810_10496_b200.backend.b200 import family

    fam = family(bench)
    return next(v for v in range(len(fam.knobs)) if fam.key(v) == "stage=2")


def _run(bench, dims, inputs, arrays):
    """Stage-2 run on uploaded inputs; returns the requested arrays (by index)."""
    from paper_1810_10496_b200.backend.b200 import Workspace

    ws = Workspace(0, bench, dims)
    try:
        ws.generate(True, 1729, -1)
        for a, x in inputs.items():
            ws.upload(a, x)
        ws.run(_stage2(bench), samples=1, batch=1, restore=False, flush=False)
        return [ws.download(a) for a in arrays]
    finally:
        ws.close()


@pytest.mark.parametrize("n,m", [(384, 320), (1024, 520)])
def test_syrk_wide_range(n, m):
    rng = np.random.default_rng(n + m)
    A = _wide(rng, (n, m))
    C = _wide(rng, (n, n), decades=2)
    (out,) = _run("SYRK", (n, m), {0: A, 1: C}, [1])
    out = out.reshape(n, n)
    a64 = A.astype(np.float64)
    ref = 12435.0 * (a64 @ a64.T) + 4546.0 * C.astype(np.float64)
    _check(out, ref)


def test_2mm_wide_range_f16_path():
    n = 1792  # plain products fill the GPU without split-K from here: the 3xFP16 path
    rng = np.random.default_rng(3)
    A = _wide(rng, (n, n), 6)
    B = _wide(rng, (n, n), 6)
    D = _wide(rng, (n, n), 4)
    outs = [o.reshape(n, n) for o in _run("2MM", (n, n, n, n), {0: A, 1: B, 3: D}, [2, 4])]  # C = A B, E = C D
    C_ref = A.astype(np.float64) @ B.astype(np.float64)
    _check(outs[0], C_ref)
    E_ref = outs[0].astype(np.float64) @ D.astype(np.float64)  # second product on the device's C
    _check(outs[1], E_ref)


def test_syr2k_wide_range():
    n, m = 512, 448
    rng = np.random.default_rng(7)
    A = _wide(rng, (n, m), 6)
    B = _wide(rng, (n, m), 3)  # different magnitudes: one shared scale for both pairs
    C = _wide(rng, (n, n), 2)
    (out,) = _run("SYR2K", (n, m), {0: A, 1: B, 2: C}, [2])
    out = out.reshape(n, n)
    a, b = A.astype(np.float64), B.astype(np.float64)
    ref = 12435.0 * (a @ b.T + b @ a.T) + 4546.0 * C.astype(np.float64)
    _check(out, ref)


def test_tf32_mode_and_unfused_statistics_still_match():
    env = dict(os.environ, PF_TC_F16="0")
    env.pop("PF_PARITY_LOG", None)
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-m", "gpu", "-p", "no:cacheprovider",
                        "tests/test_gpu_parity.py", "-k", "tensor_core"],
                       cwd=ROOT, env=env, capture_output=True, text=True, timeout=1200)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]


def test_2mm_long_k_two_pass_split():
    """K > kStripMaxK (2944): the MN-major operand takes the two-pass split
    (column maxima of row blocks, then transposed 64 x 64 tiles)."""
    ni, nj, nk = 1792, 1792, 3008
    rng = np.random.default_rng(11)
    A = _wide(rng, (ni, nk), 4)
    B = _wide(rng, (nk, nj), 4)
    D = _wide(rng, (nj, ni), 2)
    C, E = (o.reshape(ni, -1) for o in _run("2MM", (ni, nj, nk, ni), {0: A, 1: B, 3: D}, [2, 4]))
    _check(C, A.astype(np.float64) @ B.astype(np.float64))
    _check(E, C.astype(np.float64) @ D.astype(np.float64))


@pytest.mark.parametrize("bench", ["CORR", "COVAR"])
@pytest.mark.parametrize("dims", [(384, 3008), (512, 700)])
def test_corrcov_both_statistics_paths(bench, dims):
    """n <= kCSMaxRows: the column-strip kernel; n > kCSMaxRows: column
    partials + statistics + tile centring; both against the C oracle on the
    stock input."""
    from oracle import oracle as orc
    from paper_1810_10496_b200.backend.b200 import Workspace

    orc.set_threads(0)
    ref = orc.reference(bench, dims, True, 1729, -1)
    ws = Workspace(0, bench, dims)
    try:
        ws.generate(True, 1729, -1)
        ws.run(_stage2(bench), samples=1, batch=1, restore=True, flush=False)
        outs = [ws.download(a) for a, (_, _, o) in enumerate(ws.arrays) if o]
    finally:
        ws.close()
    assert len(outs) == len(ref)
    for got, r in zip(outs, ref):
        _check(got, np.asarray(r))


def test_2mm_stream_k():
    """Pair tiles over several waves with a partial last one (2304^2: 81 tiles
    on 74 SM pairs): the stream-K pair kernel (tc_sk2.cuh) splits tiles across
    pairs and adds the partial tiles onto a zeroed D."""
    n = 2304
    rng = np.random.default_rng(13)
    A = _wide(rng, (n, n), 4)
    B = _wide(rng, (n, n), 4)
    D = _wide(rng, (n, n), 2)
    C, E = (o.reshape(n, n) for o in _run("2MM", (n, n, n, n), {0: A, 1: B, 3: D}, [2, 4]))
    _check(C, A.astype(np.float64) @ B.astype(np.float64))
    _check(E, C.astype(np.float64) @ D.astype(np.float64))
