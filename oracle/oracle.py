"""ctypes wrapper over liborc.so -- the CPU ORACLE (test infrastructure only).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
``--impl reference`` leg import this module.  The product path
(paper_1810_10496_b200) never does.

See polybench_cpu.c for the parity status ("parity unpinned" for kernel
arithmetic: PolyBench/GPU is not in /root/reference) and oracle/SPEC.md for
the frozen kernel definitions.
"""

from __future__ import annotations

import ctypes
import subprocess
from ctypes import POINTER, c_float, c_int, c_int64, c_uint64
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
LIB = HERE / "liborc.so"

BENCHES = (
    "2DCONV", "3DCONV", "2MM", "3MM", "ATAX", "BICG", "CORR", "COVAR", "FDTD-2D",
    "GEMM", "GESUMMV", "GRAMSCHM", "MVT", "SYR2K", "SYRK",
)
NARRAYS = {
    "2DCONV": 2, "3DCONV": 2, "2MM": 5, "3MM": 7, "ATAX": 4, "BICG": 5, "CORR": 4, "COVAR": 3,
    "FDTD-2D": 4, "GEMM": 3, "GESUMMV": 5, "GRAMSCHM": 3, "MVT": 5, "SYR2K": 3, "SYRK": 2,
}
# indices of the arrays each benchmark reports (PolyBench/GPU compareResults)
OUTPUTS = {
    "2DCONV": (1,), "3DCONV": (1,), "2MM": (4,), "3MM": (6,), "ATAX": (2,), "BICG": (3, 4),
    "CORR": (3,), "COVAR": (2,), "FDTD-2D": (1, 2, 3), "GEMM": (2,), "GESUMMV": (3,),
    "GRAMSCHM": (0, 1, 2), "MVT": (1, 2), "SYR2K": (2,), "SYRK": (1,),
}

_lib = None


def build() -> Path:
    subprocess.run(["make", "-s", "-C", str(HERE)], check=True)
    return LIB


def lib():
    global _lib
    if _lib is None:
        if not LIB.exists():
            build()
        h = ctypes.CDLL(str(LIB))
        I64P = POINTER(c_int64)
        h.orc_array_elems.restype = c_int64
        h.orc_array_elems.argtypes = [c_int, I64P, c_int]
        h.orc_array_role.restype = c_int
        h.orc_array_role.argtypes = [c_int, c_int]
        h.orc_generate.restype = c_int
        h.orc_generate.argtypes = [c_int, I64P, c_int, c_int, c_uint64, c_int64, POINTER(c_float)]
        h.orc_run.restype = c_int
        h.orc_run.argtypes = [c_int, I64P, POINTER(POINTER(c_float))]
        h.orc_set_threads.restype = c_int
        h.orc_set_threads.argtypes = [c_int]
        h.orc_get_threads.restype = c_int
        _lib = h
    return _lib


def _dims(dims) -> ctypes.Array:
    a = (c_int64 * 6)()
    for i, v in enumerate(dims):
        a[i] = int(v)
    return a


def set_threads(n: int = 0) -> int:
    return lib().orc_set_threads(n)


def generate(bench: str, dims, stock: bool = True, seed: int = 1729, instance: int = -1) -> list[np.ndarray]:
    """All arrays of ``bench`` as the device generator would produce them."""
    b = BENCHES.index(bench)
    d = _dims(dims)
    out = []
    for a in range(NARRAYS[bench]):
        n = lib().orc_array_elems(b, d, a)
        arr = np.empty(n, dtype=np.float32)
        rc = lib().orc_generate(b, d, a, int(stock), seed, instance, arr.ctypes.data_as(POINTER(c_float)))
        if rc:
            raise RuntimeError(f"orc_generate failed for {bench} array {a}")
        out.append(arr)
    return out


def run(bench: str, dims, arrays: list[np.ndarray]) -> list[np.ndarray]:
    """Run the kernel in place on ``arrays`` (float32); returns them."""
    b = BENCHES.index(bench)
    ptrs = (POINTER(c_float) * len(arrays))(*[a.ctypes.data_as(POINTER(c_float)) for a in arrays])
    if lib().orc_run(b, _dims(dims), ptrs):
        raise RuntimeError(f"orc_run failed for {bench}")
    return arrays


def reference(bench: str, dims, stock: bool = True, seed: int = 1729, instance: int = -1) -> list[np.ndarray]:
    """Output arrays (PolyBench compare set) for the given input instance."""
    arrays = run(bench, dims, generate(bench, dims, stock, seed, instance))
    return [arrays[i] for i in OUTPUTS[bench]]


__all__ = ["BENCHES", "OUTPUTS", "build", "generate", "lib", "reference", "run", "set_threads"]
