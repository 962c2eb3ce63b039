"""The benchmark registry: the 15 PolyBench/GPU kernels as ``KernelCase``s.

In the reference the registry is a suite JSON loaded by ``cli._load_suite``
(`/root/reference/pkg/src/phaseforge/cli.py:60-101`) into ``KernelCase``
values (`backend/types.py:103-118`) whose ``source`` is a path or simulator
model and whose inputs are opaque strings.  Here:

* ``source``            ``"polybench-gpu:<BENCH>"``
* ``validation_input``  ``"<BENCH>:<dim>=<v>,..."`` (small, never timed)
* ``measurement_input`` the timed size (PolyBench/GPU default or the
  BASELINE.json config size)
* ``reference_outputs`` outputs of the *baseline* (empty-order) variant on the
  validation input, produced on the device by ``build_suite`` -- the analogue
  of PolyBench's own CPU check, whose agreement with the independent CPU
  oracle is established by ``tests/`` (never by the product path);
* ``ir_text``           an IR-subset description of the unoptimised kernel
  CFG (grammar of ``irfeat.parse_ir``), used by the 1-NN/3-NN transfer.
"""

from __future__ import annotations

from dataclasses import dataclass
from pathlib import Path

from .backend.types import KernelCase

BENCHES = (
    "2DCONV", "3DCONV", "2MM", "3MM", "ATAX", "BICG", "CORR", "COVAR", "FDTD-2D",
    "GEMM", "GESUMMV", "GRAMSCHM", "MVT", "SYR2K", "SYRK",
)

DIM_NAMES = {
    "2DCONV": ("ni", "nj"),
    "3DCONV": ("ni", "nj", "nk"),
    "2MM": ("ni", "nj", "nk", "nl"),
    "3MM": ("ni", "nj", "nk", "nl", "nm"),
    "ATAX": ("nx", "ny"),
    "BICG": ("nx", "ny"),
    "CORR": ("m", "n"),
    "COVAR": ("m", "n"),
    "FDTD-2D": ("nx", "ny", "tmax"),
    "GEMM": ("ni", "nj", "nk"),
    "GESUMMV": ("n",),
    "GRAMSCHM": ("m", "n"),
    "MVT": ("n",),
    "SYR2K": ("n", "m"),
    "SYRK": ("n", "m"),
}

# size classes: validation (quick correctness input), polybench (PolyBench/GPU
# 1.0 defaults), config (BASELINE.json configs[0..3]).
SIZES = {
    "2DCONV": {"validation": (128, 128), "polybench": (4096, 4096), "config": (4096, 4096)},
    "3DCONV": {"validation": (32, 32, 32), "polybench": (256, 256, 256), "config": (256, 256, 256)},
    "2MM": {"validation": (128, 128, 128, 128), "polybench": (2048,) * 4, "config": (2048,) * 4},
    "3MM": {"validation": (128,) * 5, "polybench": (512,) * 5, "config": (2048,) * 5},
    "ATAX": {"validation": (256, 256), "polybench": (4096, 4096), "config": (16384, 16384)},
    "BICG": {"validation": (256, 256), "polybench": (4096, 4096), "config": (16384, 16384)},
    "CORR": {"validation": (128, 128), "polybench": (2048, 2048), "config": (2048, 2048)},
    "COVAR": {"validation": (128, 128), "polybench": (2048, 2048), "config": (2048, 2048)},
    "FDTD-2D": {"validation": (64, 64, 10), "polybench": (2048, 2048, 500), "config": (2048, 2048, 500)},
    "GEMM": {"validation": (64, 64, 64), "polybench": (512, 512, 512), "config": (512, 512, 512)},
    "GESUMMV": {"validation": (256,), "polybench": (4096,), "config": (16384,)},
    "GRAMSCHM": {"validation": (128, 128), "polybench": (2048, 2048), "config": (2048, 2048)},
    "MVT": {"validation": (256,), "polybench": (4096,), "config": (16384,)},
    "SYR2K": {"validation": (128, 128), "polybench": (2048, 2048), "config": (2048, 2048)},
    "SYRK": {"validation": (128, 128), "polybench": (1024, 1024), "config": (2048, 2048)},
}

BLAS2 = ("ATAX", "BICG", "MVT", "GESUMMV")
STENCILS = ("2DCONV", "3DCONV", "FDTD-2D")
DENSE = ("2MM", "3MM", "SYRK", "SYR2K", "CORR", "COVAR", "GRAMSCHM")


def bench_index(name: str) -> int:
    return BENCHES.index(name)


def describe(bench: str, dims) -> str:
    """Input descriptor string, e.g. ``GEMM:ni=512,nj=512,nk=512``."""
    names = DIM_NAMES[bench]
    if len(dims) != len(names):
        raise ValueError(f"{bench} expects {len(names)} dims, got {len(dims)}")
    return bench + ":" + ",".join(f"{n}={int(v)}" for n, v in zip(names, dims))


def parse_descriptor(text: str) -> tuple[str, tuple[int, ...]]:
    """Inverse of ``describe``; raises ValueError on anything malformed."""
    bench, sep, rest = text.partition(":")
    if not sep or bench not in DIM_NAMES:
        raise ValueError(f"not a PolyBench/GPU input descriptor: {text!r}")
    fields = dict(item.split("=", 1) for item in rest.split(",") if item)
    try:
        dims = tuple(int(fields[n]) for n in DIM_NAMES[bench])
    except (KeyError, ValueError) as exc:
        raise ValueError(f"bad descriptor {text!r}: {exc}") from exc
    if any(d < 1 for d in dims):
        raise ValueError(f"dims must be positive in {text!r}")
    return bench, dims


def source_of(bench: str) -> str:
    return f"polybench-gpu:{bench}"


def bench_of(kernel: KernelCase) -> str:
    src = kernel.source
    if isinstance(src, str) and src.startswith("polybench-gpu:"):
        return src.split(":", 1)[1]
    bench, _ = parse_descriptor(kernel.validation_input)
    return bench


# ---------------------------------------------------------------- IR-subset texts
# Unoptimised-IR-shaped CFG descriptions (irfeat grammar).  Each kernel is a
# guard block, nested counted loops and straight-line bodies, mirroring the
# PolyBench/GPU kernel sources' structure.

@dataclass(frozen=True)
class _Loop:
    body: dict          # op -> count for the innermost body
    pre: dict = None    # ops before the inner loop (at this nest level)
    post: dict = None   # ops after the inner loop
    inner: "_Loop | None" = None


def _ops(lines: list[str], ops: dict | None) -> None:
    for op in ("addr", "load", "fadd", "iadd", "cmp", "store", "call", "other"):
        lines.extend([f"  {op}"] * (ops or {}).get(op, 0))


def _function(name: str, guard: dict, loop: _Loop | None, tail: dict | None = None,
              guards: int = 1) -> str:
    """entry -> chained bounds guards -> (loop nest | straight-line tail) -> exit."""
    lines = [f"func {name} {{", "entry:"]
    _ops(lines, guard)
    n = [0]

    def fresh(prefix: str) -> str:
        n[0] += 1
        return f"{prefix}{n[0]}"

    for _ in range(guards):
        nxt = fresh("g")
        lines += ["  cmp", f"  condbr {nxt} exit", f"{nxt}:"]

    def emit_loop(lp: _Loop, cont: str) -> None:
        head, body, latch, done = fresh("h"), fresh("b"), fresh("l"), fresh("x")
        _ops(lines, lp.pre)
        lines.extend([f"  br {head}", f"{head}:", "  phi 2", "  phi 2", "  cmp", f"  condbr {body} {done}", f"{body}:"])
        if lp.inner is not None:
            emit_loop(lp.inner, latch)
        else:
            _ops(lines, lp.body)
            lines.append(f"  br {latch}")
        lines.extend([f"{latch}:", "  iadd", f"  br {head}", f"{done}:"])
        _ops(lines, lp.post)
        lines.append(f"  br {cont}")

    if loop is not None:
        emit_loop(loop, "exit")
    else:
        _ops(lines, tail)
        lines.append("  br exit")
    lines += ["exit:", "  ret", "}"]
    return "\n".join(lines) + "\n"


def _mm(name: str, store_in_loop: bool = True, two_products: bool = False) -> str:
    body = {"addr": 4 if two_products else 2, "load": (5 if two_products else 3) if store_in_loop else (4 if two_products else 2),
            "fadd": 5 if two_products else 2, "iadd": 2, "store": 1 if store_in_loop else 0}
    return _function(name, {"iadd": 4, "cmp": 1, "other": 2},
                     _Loop(body=body, pre={"addr": 1, "load": 1, "fadd": 1, "store": 1}), guards=2)


def _mv(name: str, rows: bool, extra: int = 0) -> str:
    body = {"addr": 2 + extra, "load": 3 + extra, "fadd": 2 + 2 * extra, "iadd": 1, "store": 1 + extra}
    return _function(name, {"iadd": 2, "cmp": 1, "other": 1}, _Loop(body=body, pre={"addr": 1}), guards=1)


def _ir_texts() -> dict[str, str]:
    t: dict[str, str] = {}
    t["2DCONV"] = _function("Convolution2D_kernel", {"iadd": 6, "cmp": 1},
                            None, tail={"addr": 9, "load": 9, "fadd": 17, "iadd": 12, "store": 1}, guards=4)
    t["3DCONV"] = _function("convolution3D_kernel", {"iadd": 6, "cmp": 1},
                            None, tail={"addr": 15, "load": 15, "fadd": 29, "iadd": 30, "store": 1}, guards=6)
    t["GEMM"] = _mm("gemm")
    t["2MM"] = _mm("mm2_kernel1") + _mm("mm2_kernel2")
    t["3MM"] = _mm("mm3_kernel1") + _mm("mm3_kernel2") + _mm("mm3_kernel3")
    t["SYRK"] = _mm("syrk_kernel")
    t["SYR2K"] = _mm("syr2k_kernel", two_products=True)
    t["ATAX"] = _mv("atax_kernel1", True) + _mv("atax_kernel2", False)
    t["BICG"] = _mv("bicgKernel1", False) + _mv("bicgKernel2", True)
    t["MVT"] = _mv("mvt_kernel1", True) + _mv("mvt_kernel2", False)
    t["GESUMMV"] = _function("gesummv_kernel", {"iadd": 2, "cmp": 1},
                             _Loop(body={"addr": 3, "load": 6, "fadd": 4, "iadd": 1, "store": 2},
                                   post={"load": 2, "fadd": 3, "store": 1}), guards=1)
    mean = _function("mean_kernel", {"iadd": 3, "cmp": 2},
                     _Loop(body={"addr": 1, "load": 2, "fadd": 1, "iadd": 1, "store": 1},
                           pre={"store": 1}, post={"load": 1, "fadd": 1, "store": 1}), guards=2)
    reduce_ = _function("reduce_kernel", {"iadd": 6, "cmp": 4}, None,
                        tail={"addr": 2, "load": 2, "fadd": 1, "store": 1}, guards=4)
    std = _function("std_kernel", {"iadd": 3, "cmp": 2},
                    _Loop(body={"addr": 1, "load": 4, "fadd": 3, "iadd": 1, "store": 1},
                          pre={"store": 1}, post={"load": 2, "fadd": 2, "call": 1, "cmp": 1, "store": 2}), guards=2)
    sym = _Loop(body={"addr": 3, "load": 3, "fadd": 2, "iadd": 2, "store": 1},
                pre={"store": 1}, post={"load": 1, "store": 1})
    corr = _function("corr_kernel", {"iadd": 3, "cmp": 2},
                     _Loop(body={}, pre={"store": 1}, inner=sym), guards=2)
    covar = _function("covar_kernel", {"iadd": 3, "cmp": 2},
                      _Loop(body={}, inner=sym), guards=2)
    t["CORR"] = mean + std + reduce_.replace("reduce_kernel", "reduce_kernel") + corr
    t["COVAR"] = mean + reduce_ + covar
    t["FDTD-2D"] = (
        _function("fdtd_step1_kernel", {"iadd": 4, "cmp": 2}, None,
                  tail={"addr": 3, "load": 3, "fadd": 2, "iadd": 2, "cmp": 1, "store": 1}, guards=3)
        + _function("fdtd_step2_kernel", {"iadd": 4, "cmp": 3}, None,
                    tail={"addr": 3, "load": 3, "fadd": 2, "iadd": 2, "store": 1}, guards=3)
        + _function("fdtd_step3_kernel", {"iadd": 4, "cmp": 2}, None,
                    tail={"addr": 5, "load": 5, "fadd": 5, "iadd": 4, "store": 1}, guards=3)
    )
    t["GRAMSCHM"] = (
        _function("gramschmidt_kernel1", {"iadd": 1, "cmp": 1},
                  _Loop(body={"addr": 1, "load": 3, "fadd": 2, "iadd": 1, "store": 1},
                        post={"load": 1, "call": 1, "store": 1}), guards=1)
        + _function("gramschmidt_kernel2", {"iadd": 2, "cmp": 1}, None,
                    tail={"addr": 3, "load": 2, "fadd": 1, "store": 1}, guards=1)
        + _function("gramschmidt_kernel3", {"iadd": 2, "cmp": 2},
                    _Loop(body={"addr": 3, "load": 3, "fadd": 2, "iadd": 1, "store": 1},
                          pre={"store": 1},
                          post={"addr": 3, "load": 3, "fadd": 2, "iadd": 1, "store": 1}), guards=2)
    )
    return t


IR_TEXTS = _ir_texts()

# The second feature source: IR-subset text recovered from the -O0 PTX of each
# benchmark's compiled baseline variant (tools/gen_ir.py, committed under ir/).
IR_DIR = Path(__file__).resolve().parent / "ir"
IR_SOURCES = ("structural", "ptx")


def ir_text(bench: str, source: str = "structural") -> str:
    """``structural``: the PolyBench/GPU kernel shapes above (the default, used
    by the golden fixtures); ``ptx``: generated from the baseline variant's PTX."""
    if source == "structural":
        return IR_TEXTS[bench]
    if source == "ptx":
        path = IR_DIR / f"{bench}.ir"
        if not path.exists():
            raise FileNotFoundError(f"{path} missing: run tools/gen_ir.py")
        return path.read_text()
    raise ValueError(f"unknown IR source {source!r} (expected one of {IR_SOURCES})")


def kernel_case(bench: str, size: str = "config", reference_outputs: tuple[float, ...] = (),
                validation_dims=None, measurement_dims=None, ir: str = "structural") -> KernelCase:
    """A ``KernelCase`` for ``bench``; reference outputs are filled by ``build_suite``."""
    sizes = SIZES[bench]
    vdims = validation_dims or sizes["validation"]
    mdims = measurement_dims or sizes[size]
    return KernelCase(
        id=bench,
        source=source_of(bench),
        validation_input=describe(bench, vdims),
        measurement_input=describe(bench, mdims),
        reference_outputs=tuple(reference_outputs),
        ir_text=ir_text(bench, ir),
    )


def build_suite(backend, size: str = "config", benches=BENCHES, ir: str = "structural") -> list[KernelCase]:
    """KernelCases with ``reference_outputs`` = baseline-variant outputs on the
    validation input, computed on the device through ``backend``."""
    cases = []
    for b in benches:
        case = kernel_case(b, size, ir=ir)
        outs = backend.baseline_outputs(case)
        cases.append(KernelCase(case.id, case.source, case.validation_input, case.measurement_input,
                                tuple(outs), case.ir_text))
    return cases


__all__ = [
    "BENCHES",
    "BLAS2",
    "DENSE",
    "DIM_NAMES",
    "IR_TEXTS",
    "SIZES",
    "STENCILS",
    "bench_index",
    "bench_of",
    "build_suite",
    "describe",
    "ir_text",
    "kernel_case",
    "parse_descriptor",
    "source_of",
]
