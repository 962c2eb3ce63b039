"""pytest plugin: make ``import phaseforge`` resolve to this repository's
restated engine, so the reference's own unmodified tests
(/root/reference/pkg/tests) run against it.

The engine modules (catalog, irfeat, explorer, advisor, results,
backend.types, backend.toolchain) come from ``paper_1810_10496_b200``.  The
reference's simulator and CLI sources (out of scope for the B200 build, and
used by the reference tests as their test double / front door) are executed
from /root/reference inside the aliased package, so their relative imports
bind to the restated types -- a foreign-type mix would fail the engine's
enum identity checks.  Usage (see tests/test_reference_suite.py):

    PYTHONPATH=<repo>:<repo>/tools python -m pytest -p phaseforge_alias \\
        -p no:cacheprovider /root/reference/pkg/tests/test_explorer.py ...
"""

from __future__ import annotations

import importlib.util
import sys
import types
from pathlib import Path

REF = Path("/root/reference/pkg/src/phaseforge")


def _install() -> None:
    if "phaseforge" in sys.modules and getattr(sys.modules["phaseforge"], "__restated__", False):
        return
    from paper_1810_10496_b200 import advisor, catalog, explorer, irfeat, results
    from paper_1810_10496_b200.backend import toolchain as btoolchain
    from paper_1810_10496_b200.backend import types as btypes

    pkg = types.ModuleType("phaseforge")
    pkg.__path__ = []
    pkg.__restated__ = True
    bpkg = types.ModuleType("phaseforge.backend")
    bpkg.__path__ = []
    sys.modules["phaseforge"] = pkg
    sys.modules["phaseforge.backend"] = bpkg
    for name, mod in (("catalog", catalog), ("irfeat", irfeat), ("explorer", explorer), ("advisor", advisor),
                      ("results", results)):
        sys.modules[f"phaseforge.{name}"] = mod
        setattr(pkg, name, mod)
    sys.modules["phaseforge.backend.types"] = btypes
    bpkg.types = btypes

    def load(name: str, path: Path):
        spec = importlib.util.spec_from_file_location(name, path)
        mod = importlib.util.module_from_spec(spec)
        sys.modules[name] = mod
        spec.loader.exec_module(mod)
        return mod

    bpkg.simulator = load("phaseforge.backend.simulator", REF / "backend" / "simulator.py")
    sys.modules["phaseforge.backend.toolchain"] = btoolchain
    bpkg.toolchain = btoolchain
    for mod in (btypes, bpkg.simulator, bpkg.toolchain):
        for k in dir(mod):
            if not k.startswith("_"):
                setattr(bpkg, k, getattr(mod, k))
    pkg.backend = bpkg
    pkg.cli = load("phaseforge.cli", REF / "cli.py")
    for mod in (catalog, irfeat, explorer, advisor, results, bpkg):
        for k in dir(mod):
            if not k.startswith("_") and not hasattr(pkg, k):
                setattr(pkg, k, getattr(mod, k))
    pkg.__version__ = "0.1.0"


_install()
