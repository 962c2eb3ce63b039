"""Process-level adapter: libpfgpu behind the reference runner contract.

``python -m paper_1810_10496_b200.pftool <command> ...`` implements the four
compile-stage commands and the runner that a reference ``ToolchainSpec``
names (`/root/reference/pkg/src/phaseforge/backend/toolchain.py:29-35`), so
the stock ``ToolchainBackend`` -- and the reference CLI's ``--backend
toolchain`` -- can drive the B200 kernels without importing this package:

  frontend <source> <output>         kernel source file -> IR file
  opt      <input> <output> -p1 -p2  append the pass flags (malformed flag: exit 1)
  link     <input> <output>          copy
  codegen  <input> <output>          pass model -> variant -> artifact bytes,
                                     identical to ``B200Backend.compile``'s
  run      <artifact> <data> <kind>  execute; prints the report grammar of
                                     toolchain.py:178-213 (TIME/OUT/values)
  suite    <dir> [--size S]          write kernel sources, suite.json (with
                                     baseline reference outputs, needs a GPU)
                                     and toolchain.json for this adapter

The kernel "source" is a small text file: ``polybench-gpu:<BENCH>`` and the
two input descriptors, so codegen can refuse a variant that does not support
them (CODEGEN_FAILURE, as ``B200Backend.compile`` does).  The runner is one
process and one CUDA context per execution, as in the reference; the
in-process ``B200Backend`` is the fast path.
"""

from __future__ import annotations

import argparse
import json
import os
import shlex
import shutil
import sys
from pathlib import Path

from . import passmodel, registry
from .catalog import PassId, PhaseOrder

IR_MAGIC = "; pfgpu-ir/1"


def _read_source(path: Path) -> dict:
    lines = [ln.strip() for ln in path.read_text().splitlines() if ln.strip()]
    if not lines or not lines[0].startswith("polybench-gpu:"):
        raise ValueError(f"{path}: not a polybench-gpu kernel source")
    bench = lines[0].split(":", 1)[1]
    if bench not in registry.BENCHES:
        raise ValueError(f"{path}: unknown benchmark {bench!r}")
    info = {"bench": bench, "inputs": []}
    for ln in lines[1:]:
        key, _, value = ln.partition(" ")
        if key in ("validation", "measurement"):
            registry.parse_descriptor(value)
            info["inputs"].append(value)
    return info


def _read_ir(path: Path) -> dict:
    text = path.read_text().splitlines()
    if not text or text[0] != IR_MAGIC:
        raise ValueError(f"{path}: not a pfgpu IR file")
    return json.loads("\n".join(text[1:]))


def _write_ir(path: Path, ir: dict) -> None:
    path.write_text(IR_MAGIC + "\n" + json.dumps(ir, sort_keys=True) + "\n")


def cmd_frontend(src: str, out: str) -> int:
    info = _read_source(Path(src))
    _write_ir(Path(out), {**info, "passes": []})
    return 0


def cmd_opt(inp: str, out: str, flags: list[str]) -> int:
    ir = _read_ir(Path(inp))
    for flag in flags:
        if not flag.startswith("-"):
            print(f"pftool opt: expected a pass flag, got {flag!r}", file=sys.stderr)
            return 1
        ir["passes"].append(PassId(flag[1:]).name)  # ValueError (exit 1) on a malformed name
    _write_ir(Path(out), ir)
    return 0


def cmd_link(inp: str, out: str) -> int:
    _read_ir(Path(inp))
    shutil.copyfile(inp, out)
    return 0


def cmd_codegen(inp: str, out: str) -> int:
    from .backend.b200 import _supported_dims, artifact_content, family

    ir = _read_ir(Path(inp))
    bench = ir["bench"]
    order = PhaseOrder(tuple(PassId(p) for p in ir["passes"]))
    variant = family(bench).select(passmodel.interpret(order))
    for text in ir["inputs"]:
        _, dims = registry.parse_descriptor(text)
        if not _supported_dims(bench, variant, dims):
            print(f"{bench} variant {family(bench).key(variant)} does not support {text}", file=sys.stderr)
            return 1
    Path(out).write_bytes(artifact_content(bench, variant))
    return 0


def cmd_run(artifact: str, data: str, kind: str) -> int:
    from .backend.b200 import ARTIFACT_MAGIC, B200Backend, variant_of_artifact
    from .backend.types import InputKind, KernelCase

    content = Path(artifact).read_bytes()
    head = content.split(b"\n", 1)[0].decode(errors="replace").split()
    if not head or head[0] != ARTIFACT_MAGIC or not head[1].startswith("bench="):
        print("pftool run: not a pfgpu artifact", file=sys.stderr)
        return 2
    bench = head[1].split("=", 1)[1]
    variant = variant_of_artifact(bench, content)
    descriptor, _, index = data.partition("#")
    dbench, _ = registry.parse_descriptor(descriptor)
    if dbench != bench:
        print(f"pftool run: data {descriptor!r} is not a {bench} input", file=sys.stderr)
        return 2
    input_kind = InputKind(kind)
    backend = B200Backend(device=int(os.environ.get("PF_DEVICE", "0")))
    case = KernelCase(bench, registry.source_of(bench), descriptor, descriptor, (), None)
    got = backend.execute_variant(case, bench, variant, input_kind, int(index) if index else None)
    if got.status.value != "valid":
        print(f"pftool run: {got.status.value}: {got.log}", file=sys.stderr)
        return 3
    values = got.outputs if input_kind is InputKind.VALIDATION else ()
    sys.stdout.write(f"TIME {got.wall_time!r}\nOUT {len(values)}\n" + "".join(f"{v!r}\n" for v in values))
    return 0


def write_suite(out_dir: str | Path, size: str = "validation", benches=registry.BENCHES, backend=None) -> Path:
    """Kernel sources + ``suite.json`` (reference ``_load_suite`` schema,
    cli.py:60-101) + ``toolchain.json`` naming this adapter.  Reference outputs
    are the baseline variant's validation outputs, so a GPU is needed."""
    from .backend.b200 import B200Backend

    out = Path(out_dir)
    (out / "kernels").mkdir(parents=True, exist_ok=True)
    backend = backend or B200Backend()
    entries = []
    for case in registry.build_suite(backend, size, benches=benches):
        bench = registry.bench_of(case)
        src = out / "kernels" / f"{bench}.pfk"
        src.write_text(f"{registry.source_of(bench)}\nvalidation {case.validation_input}\n"
                       f"measurement {case.measurement_input}\n")
        ir = out / "kernels" / f"{bench}.ir"
        ir.write_text(case.ir_text)
        entries.append({"id": case.id, "source": f"kernels/{bench}.pfk", "ir_path": f"kernels/{bench}.ir",
                        "validation_input": case.validation_input, "measurement_input": case.measurement_input,
                        "reference_outputs": list(case.reference_outputs)})
    (out / "suite.json").write_text(json.dumps({"kernels": entries}, indent=1) + "\n")
    spec = toolchain_spec_dict()
    (out / "toolchain.json").write_text(json.dumps(spec, indent=1) + "\n")
    return out


def toolchain_spec_dict(work_dir: str = "work", exec_timeout: float = 120.0) -> dict:
    """ToolchainSpec JSON (toolchain.py:72-90) whose stages and runner are this tool."""
    root = Path(__file__).resolve().parent.parent
    tool = f"env PYTHONPATH={shlex.quote(str(root))} {shlex.quote(sys.executable)} -m paper_1810_10496_b200.pftool"
    return {"frontend_cmd": f"{tool} frontend {{input}} {{output}}",
            "optimizer_cmd": f"{tool} opt {{input}} {{output}} {{passes}}",
            "linker_cmd": f"{tool} link {{input}} {{output}}",
            "codegen_cmd": f"{tool} codegen {{input}} {{output}}",
            "runner_cmd": f"{tool} run {{artifact}} {{data}} {{kind}}",
            "work_dir": work_dir, "exec_timeout": exec_timeout}


def main(argv: list[str] | None = None) -> int:
    argv = list(sys.argv[1:] if argv is None else argv)
    if not argv:
        print(__doc__, file=sys.stderr)
        return 2
    cmd, rest = argv[0], argv[1:]
    try:
        if cmd == "frontend" and len(rest) == 2:
            return cmd_frontend(*rest)
        if cmd == "opt" and len(rest) >= 2:
            return cmd_opt(rest[0], rest[1], rest[2:])
        if cmd == "link" and len(rest) == 2:
            return cmd_link(*rest)
        if cmd == "codegen" and len(rest) == 2:
            return cmd_codegen(*rest)
        if cmd == "run" and len(rest) == 3:
            return cmd_run(*rest)
        if cmd == "suite":
            ap = argparse.ArgumentParser(prog="pftool suite")
            ap.add_argument("dir")
            ap.add_argument("--size", default="validation")
            ap.add_argument("--benches", nargs="*", default=list(registry.BENCHES))
            a = ap.parse_args(rest)
            print(write_suite(a.dir, a.size, a.benches))
            return 0
    except (ValueError, OSError, KeyError) as exc:
        print(f"pftool {cmd}: {exc}", file=sys.stderr)
        return 1
    print(f"pftool: bad command line {argv!r}", file=sys.stderr)
    return 2


if __name__ == "__main__":
    sys.exit(main())
