"""Backends: the drop-in boundary types and the B200 (libpfgpu) backend."""

from .types import (
    Artifact,
    Backend,
    BackendError,
    CompileOutcome,
    CompileStatus,
    ExecutionOutcome,
    ExecutionStatus,
    InputKind,
    KernelCase,
)

__all__ = [
    "Artifact",
    "Backend",
    "BackendError",
    "CompileOutcome",
    "CompileStatus",
    "ExecutionOutcome",
    "ExecutionStatus",
    "InputKind",
    "KernelCase",
]


def __getattr__(name):
    # B200Backend needs libpfgpu.so; import it lazily so the pure-Python
    # engine stays importable on a machine without the built library.
    if name == "B200Backend":
        from .b200 import B200Backend

        return B200Backend
    raise AttributeError(name)
