"""Shared pytest configuration.

* ``gpu`` marker: tests that need a B200 (run by the driver with ``-m gpu``).
* ``reference`` helpers: the upstream ``phaseforge`` package is imported from
  /root/reference when present (this container only) for exact-parity tests;
  those tests skip on the GPU box, where /root/reference does not exist.
"""

from __future__ import annotations

import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))

REFERENCE_SRC = Path("/root/reference/pkg/src")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and libpfgpu.so")
    config.addinivalue_line("markers", "slow: long-running")


def have_reference() -> bool:
    return (REFERENCE_SRC / "phaseforge" / "__init__.py").exists()


@pytest.fixture(scope="session")
def phaseforge():
    """The unmodified reference package, imported read-only from /root/reference."""
    if not have_reference():
        pytest.skip("reference package not available (GPU box)")
    sys.dont_write_bytecode = True
    if str(REFERENCE_SRC) not in sys.path:
        sys.path.append(str(REFERENCE_SRC))
    import phaseforge  # noqa: WPS433

    return phaseforge


BASELINE_REF = ROOT / "baseline" / "_ref"


def reference_engine_path() -> Path | None:
    """Where the unmodified reference package can be imported from: the
    read-only source tree (this container) or its pip install under
    baseline/_ref (git-ignored, travels to the GPU box with the snapshot)."""
    if have_reference():
        return REFERENCE_SRC
    if (BASELINE_REF / "phaseforge" / "__init__.py").exists():
        return BASELINE_REF
    return None


@pytest.fixture(scope="session")
def reference_engine():
    """The unmodified reference ``phaseforge`` package (test oracle and
    drop-in driver; never imported by the product)."""
    path = reference_engine_path()
    if path is None:
        pytest.skip("reference package not available (neither /root/reference nor baseline/_ref)")
    sys.dont_write_bytecode = True
    if str(path) not in sys.path:
        sys.path.append(str(path))
    import phaseforge  # noqa: WPS433

    return phaseforge


@pytest.fixture(scope="session")
def gpu_backend():
    from paper_1810_10496_b200.backend.b200 import B200Backend, device_count

    if device_count() < 1:
        pytest.fail("no CUDA device visible for a gpu-marked test")
    be = B200Backend(device=0, samples=3)
    yield be
    be.close()
