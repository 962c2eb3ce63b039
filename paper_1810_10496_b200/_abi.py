"""ctypes bindings to ``libpfgpu.so`` (declared in ``include/pfgpu.h``).

This is the in-process replacement for the reference's two process
boundaries (compile stages, `backend/toolchain.py:113-119`; runner,
`toolchain.py:250-258`).  The library is loaded from the package directory
only -- there is no CPU fallback: if the shared object is missing the import
of the B200 backend fails loudly.
"""

from __future__ import annotations

import ctypes
import os
import threading
from ctypes import POINTER, c_char_p, c_double, c_float, c_int, c_int64, c_size_t, c_uint64, c_void_p
from pathlib import Path

LIB_PATH = Path(__file__).resolve().parent / "libpfgpu.so"

PF_OK = 0
PF_EINVAL = -1
PF_ECUDA = -2
PF_ENOMEM = -3
PF_ENOTBUILT = -4

ROLE_IN, ROLE_INOUT, ROLE_OUT = 0, 1, 2
MAX_DIMS = 6
NKNOBS = 5

BENCH_NAMES = (
    "2DCONV", "3DCONV", "2MM", "3MM", "ATAX", "BICG", "CORR", "COVAR", "FDTD-2D",
    "GEMM", "GESUMMV", "GRAMSCHM", "MVT", "SYR2K", "SYRK",
)


class PfError(RuntimeError):
    def __init__(self, code: int, message: str):
        super().__init__(f"libpfgpu error {code}: {message}")
        self.code = code


_lock = threading.Lock()
_lib = None


def _declare(lib) -> None:
    I64P = POINTER(c_int64)
    sig = {
        "pf_abi_version": (c_int, []),
        "pf_last_error": (c_char_p, []),
        "pf_device_count": (c_int, [POINTER(c_int)]),
        "pf_device_reset": (c_int, [c_int]),
        "pf_device_info": (c_int, [c_int, c_char_p, c_size_t, POINTER(c_int), I64P, POINTER(c_int), POINTER(c_int)]),
        "pf_bench_count": (c_int, []),
        "pf_bench_info": (c_int, [c_int, c_char_p, c_size_t, POINTER(c_int), POINTER(c_int)]),
        "pf_bench_dim_name": (c_int, [c_int, c_int, c_char_p, c_size_t]),
        "pf_array_info": (c_int, [c_int, c_int, c_char_p, c_size_t, POINTER(c_int), POINTER(c_int)]),
        "pf_array_elems": (c_int, [c_int, I64P, c_int, I64P]),
        "pf_alg_work": (c_int, [c_int, I64P, POINTER(c_double), POINTER(c_double)]),
        "pf_variant_count": (c_int, [c_int]),
        "pf_variant_knobs": (c_int, [c_int, c_int, POINTER(c_int)]),
        "pf_variant_launches": (c_int, [c_int, c_int, I64P, I64P]),
        "pf_variant_supported": (c_int, [c_int, c_int, I64P]),
        "pf_ws_create": (c_int, [c_int, c_int, I64P, POINTER(c_void_p)]),
        "pf_ws_destroy": (c_int, [c_void_p]),
        "pf_ws_generate": (c_int, [c_void_p, c_int, c_uint64, c_int64]),
        "pf_ws_upload": (c_int, [c_void_p, c_int, c_void_p, c_int64]),
        "pf_ws_download": (c_int, [c_void_p, c_int, c_void_p, c_int64]),
        "pf_ws_upload_async": (c_int, [c_void_p, c_int, c_void_p, c_int64]),
        "pf_ws_restore": (c_int, [c_void_p]),
        "pf_ws_array_ptr": (c_int, [c_void_p, c_int, POINTER(c_void_p)]),
        "pf_run": (c_int, [c_void_p, c_int, c_int, c_int, c_int, c_int, POINTER(c_float)]),
        "pf_run_e2e": (c_int, [c_void_p, c_int, c_int, POINTER(c_void_p), POINTER(c_void_p), POINTER(c_float)]),
        "pf_eval_batch": (c_int, [c_void_p, c_int, c_int, c_int, POINTER(c_float), POINTER(c_float)]),
        "pf_compare": (c_int, [c_void_p, c_void_p, c_double, c_double, POINTER(c_double), I64P]),
        "pf_checksum": (c_int, [c_void_p, c_int, POINTER(c_double), POINTER(c_double)]),
        "pf_host_alloc": (c_int, [c_size_t, POINTER(c_void_p)]),
        "pf_host_free": (c_int, [c_void_p]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args


def lib():
    """Load (once) and return the shared library; raises if it is not built."""
    global _lib
    with _lock:
        if _lib is None:
            path = Path(os.environ.get("PFGPU_LIB", LIB_PATH))
            if not path.exists():
                raise ImportError(
                    f"libpfgpu.so not found at {path}; build it with `make` or __graft_entry__.build()"
                )
            handle = ctypes.CDLL(str(path))
            _declare(handle)
            _lib = handle
        return _lib


def check(rc: int) -> None:
    if rc != PF_OK:
        msg = lib().pf_last_error()
        raise PfError(rc, msg.decode() if msg else "")


class PfEval(ctypes.Structure):
    """Mirror of ``struct pf_eval`` (include/pfgpu.h)."""

    _fields_ = [("ws", c_void_p), ("variant", c_int), ("host_in", c_void_p), ("host_out", c_void_p),
                ("batch", c_int), ("no_flush", c_int)]


def dims_array(dims) -> ctypes.Array:
    arr = (c_int64 * MAX_DIMS)()
    for i, v in enumerate(dims):
        arr[i] = int(v)
    return arr


def exported_symbols() -> list[str]:
    """Function names declared in include/pfgpu.h (for the load/export test)."""
    header = Path(__file__).resolve().parent.parent / "include" / "pfgpu.h"
    names = []
    for line in header.read_text().splitlines():
        line = line.strip()
        if line.startswith(("int pf_", "const char* pf_")) and "(" in line:
            names.append(line.split("(")[0].split()[-1].lstrip("*"))
    return names


__all__ = [
    "BENCH_NAMES",
    "LIB_PATH",
    "PfError",
    "check",
    "dims_array",
    "exported_symbols",
    "lib",
]
