"""The PTX -> IR-subset feature generator (tools/gen_ir.py):
the committed texts parse under the reference grammar, give non-degenerate
feature vectors, keep PolyBench's structural identities, and are exactly what
the generator produces from the current kernel sources."""

from __future__ import annotations

import shutil
import subprocess
import sys
from pathlib import Path

import pytest

from paper_1810_10496_b200 import registry
from paper_1810_10496_b200.irfeat import cosine_distance, extract_features, parse_ir

ROOT = Path(__file__).resolve().parent.parent


@pytest.mark.parametrize("bench", registry.BENCHES)
def test_generated_ir_parses(bench):
    text = registry.ir_text(bench, "ptx")
    fv = extract_features(parse_ir(text))
    assert fv.norm() > 0
    v = dict(zip(("blocks", "insns"), (fv.values[0], fv.values[9])))
    assert v["blocks"] >= 2 and v["insns"] > v["blocks"]
    assert fv.values[16] > 0 and fv.values[17] > 0  # loads and stores survive
    case = registry.kernel_case(bench, ir="ptx")
    assert case.ir_text == text


def test_structural_identities():
    fv = {b: extract_features(parse_ir(registry.ir_text(b, "ptx"))) for b in registry.BENCHES}
    # ATAX, BICG and MVT are the same row-dot + column-dot kernel pair in PolyBench/GPU
    assert cosine_distance(fv["ATAX"], fv["BICG"]) < 1e-12
    assert cosine_distance(fv["ATAX"], fv["MVT"]) < 1e-12
    assert cosine_distance(fv["2DCONV"], fv["GEMM"]) > 1e-3
    with pytest.raises(ValueError):
        registry.ir_text("GEMM", "llvm")


@pytest.mark.skipif(shutil.which("nvcc") is None and not Path("/usr/local/cuda/bin/nvcc").exists(),
                    reason="nvcc not available")
def test_generator_is_reproducible(tmp_path):
    out = tmp_path / "ir"
    env_code = (f"import sys; sys.path.insert(0, {str(ROOT / 'tools')!r}); import gen_ir, pathlib; "
                f"gen_ir.OUT = pathlib.Path({str(out)!r}); sys.exit(gen_ir.main())")
    done = subprocess.run([sys.executable, "-c", env_code], capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert done.returncode == 0, done.stderr[-2000:]
    for bench in registry.BENCHES:
        assert (out / f"{bench}.ir").read_text() == registry.ir_text(bench, "ptx"), bench
