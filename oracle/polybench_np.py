"""Second, independent restatement of the 15 PolyBench/GPU kernels in numpy.

CPU ORACLE (test infrastructure only).  Written against oracle/SPEC.md
without sharing code with polybench_cpu.c: vectorised numpy generators and
fp64 numpy kernels.  Agreement of the two restatements at small sizes
(tests/test_oracle.py) is the pin for kernel semantics, because the
reference carries no PolyBench/GPU code or kernel golden values (SURVEY §8c:
parity unpinned).
"""

from __future__ import annotations

import numpy as np

MASK = np.uint64(0xFFFFFFFFFFFFFFFF)
STOCK_SEED = 1729
STOCK_INSTANCE = -2
BIDX = {b: i for i, b in enumerate((
    "2DCONV", "3DCONV", "2MM", "3MM", "ATAX", "BICG", "CORR", "COVAR", "FDTD-2D",
    "GEMM", "GESUMMV", "GRAMSCHM", "MVT", "SYR2K", "SYRK",
))}


def _mix(z):
    z = np.asarray(z, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
    return z ^ (z >> np.uint64(31))


def _u64(x: int) -> np.uint64:
    return np.uint64(x & 0xFFFFFFFFFFFFFFFF)


def key(seed: int, bench: str, array: int, instance: int) -> np.uint64:
    with np.errstate(over="ignore"):
        k = _mix(_u64(seed) + _u64(0x9E3779B97F4A7C15))
        k = _mix(k ^ (_u64(BIDX[bench] + 1) * _u64(0x100000001B3)))
        k = _mix(k ^ (_u64(array + 1) * _u64(0xC2B2AE3D27D4EB4F)))
        k = _mix(k ^ (_u64(instance + 2) * _u64(0x165667B19E3779F9)))
    return np.uint64(k)


def uniform(k: np.uint64, n: int) -> np.ndarray:
    idx = np.arange(n, dtype=np.uint64)
    with np.errstate(over="ignore"):
        h = _mix(k + idx * np.uint64(0x9E3779B97F4A7C15))
    return (h >> np.uint64(40)).astype(np.float32) * np.float32(1.0 / 16777216.0)


def _grid(rows: int, cols: int):
    i = np.arange(rows, dtype=np.int64)[:, None]
    j = np.arange(cols, dtype=np.int64)[None, :]
    return np.broadcast_to(i, (rows, cols)), np.broadcast_to(j, (rows, cols))


def _ratio(a, b, add, n) -> np.ndarray:
    """fp32((fp32(a) * fp32(b) + add) / n) with one rounding per operation."""
    p = np.float32(a).astype(np.float32) * np.asarray(b).astype(np.float32) if np.isscalar(a) else \
        np.asarray(a).astype(np.float32) * np.asarray(b).astype(np.float32)
    return ((p + np.float32(add)) / np.float32(n)).astype(np.float32)


def _pi(n: int) -> np.ndarray:
    return (np.arange(n, dtype=np.float64) * np.pi).astype(np.float32)


def generate(bench: str, dims, stock: bool = True, seed: int = 1729, instance: int = -1) -> list[np.ndarray]:
    """Input/zeroed arrays in the library's array order (flattened float32)."""
    d = [int(x) for x in dims]
    if not stock:
        return _random(bench, d, seed, instance)
    if bench == "2DCONV":
        ni, nj = d
        return [uniform(key(STOCK_SEED, bench, 0, STOCK_INSTANCE), ni * nj), np.zeros(ni * nj, np.float32)]
    if bench == "3DCONV":
        ni, nj, nk = d
        i, j, k = np.meshgrid(np.arange(ni), np.arange(nj), np.arange(nk), indexing="ij")
        return [(i % 12 + 2 * (j % 7) + 3 * (k % 13)).astype(np.float32).ravel(), np.zeros(ni * nj * nk, np.float32)]
    if bench == "2MM":
        ni, nj, nk, nl = d
        i, k = _grid(ni, nk)
        A = _ratio(i, k, 0, ni)
        k2, j = _grid(nk, nj)
        B = _ratio(k2, j + 1, 0, nj)
        j2, l = _grid(nj, nl)
        D = _ratio(j2, l + 2, 0, nk)
        return [A.ravel(), B.ravel(), np.zeros(ni * nj, np.float32), D.ravel(), np.zeros(ni * nl, np.float32)]
    if bench == "3MM":
        ni, nj, nk, nl, nm = d
        i, k = _grid(ni, nk)
        k2, j = _grid(nk, nj)
        j3, m = _grid(nj, nm)
        m4, l = _grid(nm, nl)
        return [_ratio(i, k, 0, ni).ravel(), _ratio(k2, j + 1, 0, nj).ravel(), _ratio(j3, m + 3, 0, nl).ravel(),
                _ratio(m4, l + 2, 0, nk).ravel(), np.zeros(ni * nj, np.float32), np.zeros(nj * nl, np.float32),
                np.zeros(ni * nl, np.float32)]
    if bench == "ATAX":
        nx, ny = d
        i, j = _grid(nx, ny)
        return [_ratio(i, j, 0, nx).ravel(), _pi(ny), np.zeros(ny, np.float32), np.zeros(nx, np.float32)]
    if bench == "BICG":
        nx, ny = d
        i, j = _grid(nx, ny)
        return [_ratio(i, j, 0, nx).ravel(), _pi(nx), _pi(ny), np.zeros(ny, np.float32), np.zeros(nx, np.float32)]
    if bench in ("CORR", "COVAR"):
        m, n = d
        i, j = _grid(n + 1, m + 1)
        data = _ratio(i, j, 0, m + 1 if bench == "CORR" else m).ravel()
        extra = [np.zeros(m + 1, np.float32)] * (2 if bench == "CORR" else 1)
        return [data] + [e.copy() for e in extra] + [np.zeros((m + 1) * (m + 1), np.float32)]
    if bench == "FDTD-2D":
        nx, ny, tmax = d
        i, j = _grid(nx, ny)
        return [np.arange(tmax, dtype=np.float32), _ratio(i, j + 1, 1, nx).ravel(), _ratio(i - 1, j + 2, 2, nx).ravel(),
                _ratio(i - 9, j + 4, 3, nx).ravel()]
    if bench == "GEMM":
        ni, nj, nk = d
        i, k = _grid(ni, nk)
        k2, j = _grid(nk, nj)
        i3, j3 = _grid(ni, nj)
        return [_ratio(i, k, 0, ni).ravel(), _ratio(k2, j, 1, nj).ravel(), _ratio(i3, j3, 2, nj).ravel()]
    if bench == "GESUMMV":
        (n,) = d
        i, j = _grid(n, n)
        A = _ratio(i, j, 0, n).ravel()
        x = (np.arange(n).astype(np.float32) / np.float32(n)).astype(np.float32)
        return [A, A.copy(), x, np.zeros(n, np.float32), np.zeros(n, np.float32)]
    if bench == "GRAMSCHM":
        m, n = d
        return [_gram_input(uniform(key(STOCK_SEED, bench, 0, STOCK_INSTANCE), m * n), m, n),
                np.zeros(n * n, np.float32), np.zeros(m * n, np.float32)]
    if bench == "MVT":
        (n,) = d
        i, j = _grid(n, n)
        idx = np.arange(n).astype(np.float32)
        f = lambda off: ((idx + np.float32(off)) / np.float32(n)).astype(np.float32)
        return [_ratio(i, j, 0, n).ravel(), f(0), f(1), f(3), f(4)]
    if bench == "SYR2K":
        n, m = d
        i, k = _grid(n, m)
        i2, j2 = _grid(n, n)
        return [_ratio(i, k, 1, n).ravel(), _ratio(i, k, 2, n).ravel(), _ratio(i2, j2, 2, n).ravel()]
    if bench == "SYRK":
        n, m = d
        i, k = _grid(n, m)
        i2, j2 = _grid(n, n)
        return [_ratio(i, k, 0, n).ravel(), _ratio(i2, j2, 2, n).ravel()]
    raise KeyError(bench)


def _gram_input(u: np.ndarray, m: int, n: int) -> np.ndarray:
    a = u.reshape(m, n).copy()
    r = np.arange(min(m, n))
    a[r, r] = (a[r, r] + np.float32(n)).astype(np.float32)
    return a.ravel()


_ZEROED = {
    "2DCONV": {1}, "3DCONV": {1}, "2MM": {2, 4}, "3MM": {4, 5, 6}, "ATAX": {2, 3}, "BICG": {3, 4},
    "CORR": {1, 2, 3}, "COVAR": {1, 2}, "FDTD-2D": set(), "GEMM": set(), "GESUMMV": {3, 4},
    "GRAMSCHM": {1, 2}, "MVT": set(), "SYR2K": set(), "SYRK": set(),
}


def _random(bench: str, d, seed: int, instance: int) -> list[np.ndarray]:
    shapes = [a.size for a in generate(bench, d, True)]
    out = []
    for a, n in enumerate(shapes):
        if a in _ZEROED[bench]:
            out.append(np.zeros(n, np.float32))
            continue
        u = uniform(key(seed, bench, a, instance), n)
        if bench == "GRAMSCHM" and a == 0:
            u = _gram_input(u, d[0], d[1])
        out.append(u)
    return out


def run(bench: str, dims, arrays: list[np.ndarray]) -> list[np.ndarray]:
    """Reference semantics in fp64; returns the PolyBench compare set (float32)."""
    d = [int(x) for x in dims]
    f64 = [a.astype(np.float64) for a in arrays]
    if bench == "2DCONV":
        ni, nj = d
        A = f64[0].reshape(ni, nj)
        c = {k: float(np.float32(v)) for k, v in dict(c11=0.2, c21=0.5, c31=-0.8, c12=-0.3, c22=0.6, c32=-0.9,
                                                         c13=0.4, c23=0.7, c33=0.10).items()}
        B = np.zeros((ni, nj))
        B[1:-1, 1:-1] = (c["c11"] * A[:-2, :-2] + c["c12"] * A[1:-1, :-2] + c["c13"] * A[2:, :-2]
                         + c["c21"] * A[:-2, 1:-1] + c["c22"] * A[1:-1, 1:-1] + c["c23"] * A[2:, 1:-1]
                         + c["c31"] * A[:-2, 2:] + c["c32"] * A[1:-1, 2:] + c["c33"] * A[2:, 2:])
        return [B.astype(np.float32).ravel()]
    if bench == "3DCONV":
        ni, nj, nk = d
        A = f64[0].reshape(ni, nj, nk)
        B = np.zeros_like(A)
        s = slice(1, -1)
        m1, p1 = slice(0, -2), slice(2, None)
        B[s, s, s] = (2 * A[m1, m1, m1] + 4 * A[p1, m1, m1] + 5 * A[m1, m1, m1] + 7 * A[p1, m1, m1]
                      - 8 * A[m1, m1, m1] + 10 * A[p1, m1, m1] - 3 * A[s, m1, s] + 6 * A[s, s, s] - 9 * A[s, p1, s]
                      + 2 * A[m1, m1, p1] + 4 * A[p1, m1, p1] + 5 * A[m1, s, p1] + 7 * A[p1, s, p1]
                      - 8 * A[m1, p1, p1] + 10 * A[p1, p1, p1])
        return [B.astype(np.float32).ravel()]
    if bench == "2MM":
        ni, nj, nk, nl = d
        C = (f64[0].reshape(ni, nk) @ f64[1].reshape(nk, nj)).astype(np.float32).astype(np.float64)
        return [(C @ f64[3].reshape(nj, nl)).astype(np.float32).ravel()]
    if bench == "3MM":
        ni, nj, nk, nl, nm = d
        E = (f64[0].reshape(ni, nk) @ f64[1].reshape(nk, nj)).astype(np.float32).astype(np.float64)
        F = (f64[2].reshape(nj, nm) @ f64[3].reshape(nm, nl)).astype(np.float32).astype(np.float64)
        return [(E @ F).astype(np.float32).ravel()]
    if bench == "ATAX":
        nx, ny = d
        A = f64[0].reshape(nx, ny)
        tmp = (A @ f64[1]).astype(np.float32).astype(np.float64)
        return [(A.T @ tmp).astype(np.float32)]
    if bench == "BICG":
        nx, ny = d
        A = f64[0].reshape(nx, ny)
        return [(A.T @ f64[1]).astype(np.float32), (A @ f64[2]).astype(np.float32)]
    if bench == "MVT":
        (n,) = d
        A = f64[0].reshape(n, n)
        return [(f64[1] + A @ f64[3]).astype(np.float32), (f64[2] + A.T @ f64[4]).astype(np.float32)]
    if bench == "GESUMMV":
        (n,) = d
        A, B, x = f64[0].reshape(n, n), f64[1].reshape(n, n), f64[2]
        return [(43532.0 * (A @ x) + 12313.0 * (B @ x)).astype(np.float32)]
    if bench == "GEMM":
        ni, nj, nk = d
        C = 2123.0 * f64[2].reshape(ni, nj) + 32412.0 * (f64[0].reshape(ni, nk) @ f64[1].reshape(nk, nj))
        return [C.astype(np.float32).ravel()]
    if bench == "SYRK":
        n, m = d
        A = f64[0].reshape(n, m)
        return [(4546.0 * f64[1].reshape(n, n) + 12435.0 * (A @ A.T)).astype(np.float32).ravel()]
    if bench == "SYR2K":
        n, m = d
        A, B = f64[0].reshape(n, m), f64[1].reshape(n, m)
        return [(4546.0 * f64[2].reshape(n, n) + 12435.0 * (A @ B.T + B @ A.T)).astype(np.float32).ravel()]
    if bench in ("COVAR", "CORR"):
        m, n = d
        fn = float(np.float32(3214212.01))
        data = f64[0].reshape(n + 1, m + 1)[1:, 1:]
        mean = (data.sum(axis=0) / fn).astype(np.float32).astype(np.float64)
        sym = np.zeros((m + 1, m + 1))
        if bench == "COVAR":
            cen = (data - mean).astype(np.float32).astype(np.float64)
            sym[1:, 1:] = cen.T @ cen
            return [sym.astype(np.float32).ravel()]
        std = np.sqrt(((data - mean) ** 2).sum(axis=0) / fn).astype(np.float32)
        std = np.where(std <= np.float32(0.005), np.float32(1.0), std).astype(np.float64)
        z = ((data - mean) / (np.sqrt(fn) * std)).astype(np.float32).astype(np.float64)
        g = z.T @ z
        sym[1:, 1:] = g
        sym[m, 1:] = g[m - 1, :] if False else sym[m, 1:]
        # corr_kernel: diagonal 1 for j1 < m, off-diagonal mirrored, symmat[m][m] = 1
        idx = np.arange(1, m + 1)
        sym[idx, idx] = 1.0
        return [sym.astype(np.float32).ravel()]
    if bench == "FDTD-2D":
        nx, ny, tmax = d
        fict = arrays[0]
        ex, ey, hz = (f64[k].reshape(nx, ny).copy() for k in (1, 2, 3))
        r = lambda a: a.astype(np.float32).astype(np.float64)
        for t in range(tmax):
            ey[1:, :] = r(ey[1:, :] - 0.5 * (hz[1:, :] - hz[:-1, :]))
            ey[0, :] = float(fict[t])
            ex[:, 1:] = r(ex[:, 1:] - 0.5 * (hz[:, 1:] - hz[:, :-1]))
            hz[:-1, :-1] = r(hz[:-1, :-1] - 0.7 * (ex[:-1, 1:] - ex[:-1, :-1] + ey[1:, :-1] - ey[:-1, :-1]))
        return [ex.astype(np.float32).ravel(), ey.astype(np.float32).ravel(), hz.astype(np.float32).ravel()]
    if bench == "GRAMSCHM":
        m, n = d
        A = f64[0].reshape(m, n).copy()
        R = np.zeros((n, n))
        Q = np.zeros((m, n))
        for k in range(n):
            R[k, k] = np.float32(np.sqrt(A[:, k] @ A[:, k]))
            Q[:, k] = (A[:, k] / R[k, k]).astype(np.float32)
            if k + 1 < n:
                rk = (Q[:, k] @ A[:, k + 1:]).astype(np.float32).astype(np.float64)
                R[k, k + 1:] = rk
                A[:, k + 1:] = (A[:, k + 1:] - np.outer(Q[:, k], rk)).astype(np.float32)
        return [A.astype(np.float32).ravel(), R.astype(np.float32).ravel(), Q.astype(np.float32).ravel()]
    raise KeyError(bench)


def reference(bench: str, dims, stock: bool = True, seed: int = 1729, instance: int = -1) -> list[np.ndarray]:
    return run(bench, dims, generate(bench, dims, stock, seed, instance))
