#!/usr/bin/env python3
"""PTX -> IR-subset feature text for the 15 benchmarks.

The paper extracts its 24 static features from the kernels' unoptimised IR
(PAPER.md; grammar `/root/reference/pkg/src/phaseforge/irfeat.py:120-129`).
Here the IR is recovered from the compiled baseline variant itself:

1. every ``csrc/k_*.cu`` is compiled to PTX with NVVM optimisation off
   (``nvcc -ptx -arch=compute_100a -Xcicc -O0``), which leaves the CFG,
   the loads/stores and the out-of-SSA phi copies of the -O0 module intact;
2. the entry points of each benchmark's baseline variant (template tag
   ``<(pf::BenchId)B, V0>``, V0 = the empty-order variant) and the device
   functions they call are selected;
3. each PTX function becomes one ``func`` of the IR subset:
   labels -> blocks (fall-through made explicit), ``@p bra``/``bra.uni`` ->
   ``condbr``/``br``, ``ret``/``exit`` -> ``ret``; phis are recovered from
   the phi copies (a register written in >= 2 predecessors of a join block
   and read there before any write); instructions are classified into the
   grammar's body kinds (``ld`` -> load, ``st`` -> store, ``setp`` -> cmp,
   float arithmetic -> fadd, integer arithmetic -> iadd, special-register
   reads / barriers / atomics / calls -> call, the 64-bit add forming a
   memory address -> addr (its shift / wide-multiply feeders are folded
   into it, as one getelementptr), casts / selects / predicates -> other;
   parameter loads and plain register moves are not instructions).

Output: paper_1810_10496_b200/ir/<BENCH>.ir (committed; ``registry`` reads it).
"""

from __future__ import annotations

import re
import subprocess
import sys
import tempfile
from collections import defaultdict
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
PKG = ROOT / "paper_1810_10496_b200"
CSRC = PKG / "csrc"
OUT = PKG / "ir"

_TAG = re.compile(r"<\(pf::BenchId\)(\d+), (?:\(int\))?(\d+)[,>]")
_FUNC = re.compile(r"^\s*(?:\.visible\s+|\.weak\s+)?\.(entry|func)\s+(?:\([^)]*\)\s*)?([\w$]+)\s*\(?", re.M)
_CALL = re.compile(r"\bcall(?:\.uni)?\s+(?:\([^)]*\)\s*,\s*)?([\w$]+)")
_REG = re.compile(r"%[\w]+")
_ADDR_OPND = re.compile(r"\[\s*(%\w+)")
_SPECIAL = ("%tid", "%ntid", "%ctaid", "%nctaid", "%laneid", "%warpid", "%clock", "%smid", "%nsmid",
            "%globaltimer", "%lanemask", "%cluster", "%dynamic_smem")
_FLOAT_OPS = {"add", "sub", "mul", "div", "fma", "mad", "sqrt", "rsqrt", "rcp", "abs", "neg", "min", "max", "ex2",
              "lg2", "sin", "cos", "tanh", "copysign"}
_INT_OPS = {"add", "sub", "mul", "mad", "div", "rem", "shl", "shr", "and", "or", "xor", "not", "neg", "min", "max",
            "abs", "popc", "clz", "brev", "bfe", "bfi", "prmt", "mul24", "mad24", "sad", "cnot", "bfind", "fns",
            "szext", "dp4a", "dp2a", "lop3", "shf"}
_CALL_OPS = {"bar", "barrier", "membar", "fence", "atom", "red", "shfl", "vote", "match", "activemask", "mbarrier",
             "cp", "tcgen05", "griddepcontrol", "elect", "redux", "nanosleep", "trap", "prefetch", "prefetchu",
             "cvta", "applypriority", "discard", "createpolicy", "setmaxnreg", "wmma", "mma", "ldmatrix", "stmatrix",
             "multimem", "tensormap", "clusterlaunchcontrol", "getctarank", "mapa", "isspacep", "call"}
_FLOAT_TYPES = (".f32", ".f64", ".f16", ".bf16", ".f16x2", ".bf16x2", ".ftz.f32", ".f32x2")


def compile_ptx(src: Path, out: Path) -> str:
    cmd = ["nvcc", "-ptx", "-arch=compute_100a", "-std=c++17", "--expt-relaxed-constexpr", "-diag-suppress", "20168",
           "-Xcicc", "-O0", f"-I{CSRC}", str(src), "-o", str(out)]
    subprocess.run(cmd, check=True, capture_output=True, text=True)
    return out.read_text()


def split_functions(ptx: str) -> dict[str, tuple[str, list[str]]]:
    """name -> (kind, body lines) for every function definition with a body."""
    funcs = {}
    for m in _FUNC.finditer(ptx):
        kind, name = m.group(1), m.group(2)
        brace = ptx.find("{", m.end())
        semi = ptx.find(";", m.end())
        if brace < 0 or 0 <= semi < brace:
            continue  # a prototype: ';' before any body
        depth, i = 0, brace
        while True:
            c = ptx[i]
            if c == "{":
                depth += 1
            elif c == "}":
                depth -= 1
                if depth == 0:
                    break
            i += 1
        funcs[name] = (kind, ptx[brace + 1:i].splitlines())
    return funcs


def demangle(names: list[str]) -> list[str]:
    out = subprocess.run(["cu++filt"], input="\n".join(names), capture_output=True, text=True, check=True).stdout
    return out.splitlines()


def _statements(lines: list[str]):
    """Yield ('label', name) / ('insn', text) from PTX body lines."""
    buf = ""
    for raw in lines:
        line = raw.split("//", 1)[0].strip()
        if not line or line in ("{", "}"):
            continue
        if line.startswith("."):
            continue  # .reg / .local / .shared / .pragma declarations
        if re.fullmatch(r"[\w$]+:", line):
            yield ("label", line[:-1])
            continue
        buf += " " + line
        while ";" in buf:
            stmt, buf = buf.split(";", 1)
            stmt = stmt.strip()
            if stmt and stmt not in ("{", "}"):
                yield ("insn", stmt)


def _parse_insn(text: str):
    pred = None
    if text.startswith("@"):
        pred, text = text.split(None, 1)
    parts = text.split(None, 1)
    opcode = parts[0]
    operands = parts[1] if len(parts) > 1 else ""
    return pred, opcode, operands


def _dest(operands: str) -> str | None:
    first = operands.split(",", 1)[0].strip()
    if first.startswith("{"):
        return None
    return first if first.startswith("%") else None


def _classify(opcode: str, operands: str, addr_adds: set, folded: set) -> list[str]:
    base = opcode.split(".", 1)[0]
    dest = _dest(operands)
    if base == "mov":
        src = operands.split(",", 1)[1].strip() if "," in operands else ""
        return ["call"] if src.startswith(_SPECIAL) else []
    if base in ("ld", "ldu"):
        return [] if ".param" in opcode else ["load"]
    if base == "st":
        return [] if ".param" in opcode else ["store"]
    if base == "setp" or base == "set":
        return ["cmp"]
    if base in _CALL_OPS:
        return ["call"]
    if base in ("cvt", "selp", "slct", "testp"):
        return ["other"]
    if opcode.endswith(".pred") or opcode.startswith(("not.pred", "and.pred", "or.pred", "xor.pred")):
        return ["other"]
    if dest is not None and dest in folded:
        return []
    if dest is not None and dest in addr_adds:
        return ["addr"]
    if base in _FLOAT_OPS and any(t in opcode for t in _FLOAT_TYPES):
        return ["fadd", "fadd"] if base in ("fma", "mad") else ["fadd"]
    if base in _INT_OPS:
        return ["iadd", "iadd"] if base in ("mad", "mad24") else ["iadd"]
    return ["other"]


def translate(name: str, lines: list[str]) -> str:
    stmts = list(_statements(lines))
    # PTX labels carry a module-wide function counter ($L__BB<fn>_<n>); rename
    # them in order of definition so the text depends on this function only
    rename = {}
    for kind, s in stmts:
        if kind == "label":
            rename[s] = f"bb{len(rename) + 1}"
    stmts = [(k, rename[s] if k == "label" else re.sub(r"\$?L__BB\w+", lambda m: rename.get(m.group(0), m.group(0)), s))
             for k, s in stmts]
    # address recognition: 64-bit adds whose result is a memory operand, and
    # the shift / wide-multiply / index-extension feeding only them
    mem_regs = {m.group(1) for kind, s in stmts if kind == "insn" for m in _ADDR_OPND.finditer(s)}
    defs = {}
    for kind, s in stmts:
        if kind == "insn":
            _, op, opnds = _parse_insn(s)
            d = _dest(opnds)
            if d:
                defs.setdefault(d, []).append((op, opnds))
    addr_adds = {d for d, lst in defs.items() if d in mem_regs and all(o.startswith("add.") and o.endswith(("s64", "u64"))
                                                                        for o, _ in lst)}
    folded = set()
    for d in addr_adds:
        for _, opnds in defs[d]:
            for src in _REG.findall(opnds.split(",", 1)[1]):
                for op, _ in defs.get(src, []):
                    if op.startswith(("shl.b64", "mul.wide")):
                        folded.add(src)

    # blocks
    blocks: list[dict] = []
    counter = [0]

    def new_block(label: str) -> dict:
        b = {"label": label, "body": [], "term": None, "reads": [], "writes": set()}
        blocks.append(b)
        return b

    def fresh() -> str:
        counter[0] += 1
        return f"ft{counter[0]}"

    cur = new_block("entry")
    pending_cond = None  # (target) of a predicated branch awaiting its else edge
    i = 0
    while i < len(stmts):
        kind, s = stmts[i]
        if kind == "label":
            label = s.replace("$", "")
            if cur["term"] is None:
                cur["term"] = ("condbr", pending_cond, label) if pending_cond else ("br", label)
                pending_cond = None
            cur = new_block(label)
            i += 1
            continue
        if cur["term"] is not None:  # unreachable straight-line code after a terminator
            cur = new_block(fresh())
        pred, op, opnds = _parse_insn(s)
        base = op.split(".", 1)[0]
        if pending_cond is not None and not (base == "bra" and pred is None):
            # a predicated branch followed by more code: fall through to a new block
            label = fresh()
            cur["term"] = ("condbr", pending_cond, label)
            pending_cond = None
            cur = new_block(label)
        if base == "bra":
            target = opnds.strip().replace("$", "")
            if pred is not None:
                pending_cond = target
            elif pending_cond is not None:
                cur["term"] = ("condbr", pending_cond, target)
                pending_cond = None
            else:
                cur["term"] = ("br", target)
            i += 1
            continue
        if base in ("ret", "exit"):
            cur["term"] = ("ret",)
            i += 1
            continue
        regs = _REG.findall(opnds)
        d = _dest(opnds)
        srcs = regs[1:] if d else regs
        for r in srcs:
            if r not in cur["writes"]:
                cur["reads"].append(r)
        if d:
            cur["writes"].add(d)
        cur["body"].extend(_classify(op, opnds, addr_adds, folded))
        i += 1
    if cur["term"] is None:
        cur["term"] = ("condbr", pending_cond, "exit_") if pending_cond else ("ret",)
        if pending_cond:
            new_block("exit_")["term"] = ("ret",)
    # drop empty unreachable fresh blocks is unnecessary: they carry a terminator

    preds = defaultdict(list)
    for b in blocks:
        for t in b["term"][1:]:
            preds[t].append(b["label"])
    by_label = {b["label"]: b for b in blocks}
    out = [f"func {name} {{"]
    for b in blocks:
        out.append(f"{b['label']}:")
        ps = preds.get(b["label"], [])
        if len(ps) >= 2:
            seen = set()
            for r in b["reads"]:
                if r in seen:
                    continue
                seen.add(r)
                if sum(1 for p in set(ps) if r in by_label[p]["writes"]) >= 2:
                    out.append(f"  phi {len(ps)}")
        for k in b["body"]:
            out.append(f"  {dict(int_arith='iadd', float_arith='fadd').get(k, k)}")
        term = b["term"]
        out.append("  " + " ".join(term))
    out.append("}")
    return "\n".join(out) + "\n"


def baseline_variants() -> dict[str, int]:
    from paper_1810_10496_b200 import passmodel, registry
    from paper_1810_10496_b200.backend.b200 import family

    return {b: family(b).select(passmodel.BASELINE_STATE) for b in registry.BENCHES}


def main() -> int:
    from paper_1810_10496_b200 import registry

    base = baseline_variants()
    want = {registry.bench_index(b): (b, v) for b, v in base.items()}
    per_bench: dict[str, list[tuple[str, str, str, dict]]] = defaultdict(list)
    with tempfile.TemporaryDirectory() as tmp:
        for src in sorted(CSRC.glob("k_*.cu")):
            ptx = compile_ptx(src, Path(tmp) / (src.stem + ".ptx"))
            funcs = split_functions(ptx)
            names = list(funcs)
            for name, dem in zip(names, demangle(names)):
                if funcs[name][0] != "entry":
                    continue
                m = _TAG.search(dem)
                if not m or int(m.group(1)) not in want:
                    continue
                bench, v0 = want[int(m.group(1))]
                if int(m.group(2)) != v0:
                    continue
                per_bench[bench].append((dem, name, src.name, funcs))
    OUT.mkdir(exist_ok=True)
    for bench in registry.BENCHES:
        entries = sorted(per_bench.get(bench, []), key=lambda t: t[0])
        if not entries:
            print(f"{bench}: no baseline kernels found", file=sys.stderr)
            return 1
        texts, done = [], set()
        header = [f"# {bench}: IR subset generated by tools/gen_ir.py from the -O0 PTX of the baseline variant"
                  f" (variant {base[bench]}) kernels"]
        for dem, name, srcname, funcs in entries:
            queue = [name]
            while queue:
                fn = queue.pop(0)
                if fn in done or fn not in funcs:
                    continue
                done.add(fn)
                body = funcs[fn][1]
                full = demangle([fn])[0].replace("<unnamed>", "anon").replace("(anonymous namespace)", "anon")
                sig = re.sub(r"\([^()]*\)$", "", full)  # drop the parameter list
                short = re.sub(r"<.*", "", sig).split("::")[-1].split()[-1]
                label = f"{re.sub(r'[^A-Za-z0-9_]', '_', short)}_{len(done)}"
                header.append(f"#   func {label}: {sig}  [{srcname}]")
                texts.append(translate(label, body))
                queue += [c for c in _CALL.findall("\n".join(body)) if c in funcs]
        (OUT / f"{bench}.ir").write_text("\n".join(header) + "\n" + "".join(texts))
        print(f"{bench}: {len(done)} function(s)")
    return 0


if __name__ == "__main__":
    sys.exit(main())
