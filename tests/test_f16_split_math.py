"""The 3xFP16 operand split (csrc/tc_f16.cuh) restated in numpy: the error
bounds DESIGN.md §5 states for it, checked on CPU.

Per operand row: s = 2^(15 - e) with max|x| = f 2^e, f in [0.5, 1);
hi = fp16_rn(x s), lo = fp16_rn(x s - hi).  Claims:
  * x s is exact and max|x s| lies in [2^14, 2^15) (no fp16 overflow);
  * |x s - (hi + lo)| <= 2^-22 |x s| for |x| >= 2^-17 max|x|;
  * below that, the absolute error stays under 2^-39 max|x| (in x units);
  * a product accumulated as lo*hi + hi*lo + hi*hi matches the fp64 product
    to well inside the 1e-4 tolerance, including rows spanning many decades.
"""

from __future__ import annotations

import numpy as np


def row_scale(x: np.ndarray) -> np.ndarray:
    amax = np.abs(x).max(axis=1, keepdims=True)
    _, e = np.frexp(amax)
    return np.where(amax > 0, np.ldexp(1.0, 15 - e), 1.0).astype(np.float32)


def split(x: np.ndarray):
    s = row_scale(x)
    y = (x * s).astype(np.float32)
    hi = y.astype(np.float16)
    lo = (y - hi.astype(np.float32)).astype(np.float16)
    return s, y, hi, lo


def wide(rng, shape, decades):
    mag = 10.0 ** rng.uniform(-decades / 2, decades / 2, size=shape)
    return (mag * rng.choice([-1.0, 1.0], size=shape)).astype(np.float32)


def test_scale_is_exact_and_in_range():
    rng = np.random.default_rng(0)
    x = wide(rng, (64, 512), 10)
    s, y, hi, lo = split(x)
    assert np.all(np.log2(s) == np.round(np.log2(s)))  # powers of two
    assert np.array_equal(y.astype(np.float64), x.astype(np.float64) * s.astype(np.float64))  # exact
    ymax = np.abs(y).max(axis=1)
    assert np.all(ymax >= 2.0**14) and np.all(ymax < 2.0**15)
    assert np.all(np.isfinite(hi)) and np.all(np.isfinite(lo))


def test_split_error_bounds():
    rng = np.random.default_rng(1)
    x = wide(rng, (64, 2048), 12)
    s, y, hi, lo = split(x)
    err = np.abs(y.astype(np.float64) - hi.astype(np.float64) - lo.astype(np.float64))
    rowmax = np.abs(x).max(axis=1, keepdims=True).astype(np.float64)
    big = np.abs(x) >= 2.0**-17 * rowmax
    assert np.all(err[big] <= 2.0**-22 * np.abs(y.astype(np.float64))[big])
    # in x units: the small elements (lo in fp16 subnormals) below 2^-39 of the row max,
    # every element below 2^-22 of it
    err_x = err / s.astype(np.float64)
    assert np.all(err_x[~big] <= (2.0**-39 * rowmax * np.ones_like(err_x))[~big])
    assert np.all(err_x <= 2.0**-22 * rowmax)


def test_three_product_gemm_holds_fp32_tolerance():
    rng = np.random.default_rng(2)
    M, N, K = 96, 80, 1024
    A = wide(rng, (M, K), 8)
    Bt = wide(rng, (N, K), 8)  # op(B)^T: one row per output column
    sa, _, ah, al = split(A)
    sb, _, bh, bl = split(Bt)
    f = lambda u: u.astype(np.float64)  # noqa: E731  (products of two fp16 are exact in fp64)
    acc = f(al) @ f(bh).T + f(ah) @ f(bl).T + f(ah) @ f(bh).T
    got = acc / (f(sa) * f(sb).T)
    ref = f(A) @ f(Bt).T
    tol = np.maximum(1e-4 * np.abs(ref).max(), 1e-4 * np.abs(ref))
    assert np.all(np.abs(got - ref) <= tol)
    # and it is far tighter than the tolerance: ~2^-21 of the row-scale products
    assert np.abs(got - ref).max() <= 1e-5 * np.abs(ref).max()
