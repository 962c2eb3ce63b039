#!/usr/bin/env python3
"""Extract per-variant SASS from libpfgpu.so into the artifact table.

Every variant kernel carries the template prefix ``<(pf::BenchId)B, V, ...>``,
so ``cuobjdump -sass`` + ``cu++filt`` attribute each function to its
(benchmark, variant).  A variant's artifact content is a small launch header
plus the SASS of its kernels with the (variant-specific) function names
normalised away; two variants whose machine code is identical therefore get
the same sha256 digest, which is what makes ``explore`` report REUSED records
(the "identical PTX -> reuse" rule of PAPER.md:163, applied to SASS).

Output: paper_1810_10496_b200/artifacts.json.gz
  {"version": 1, "benches": {BENCH: {"<V>": "<normalised SASS text>"}}}
"""

from __future__ import annotations

import gzip
import json
import re
import shutil
import subprocess
import sys
from collections import defaultdict
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
PKG = ROOT / "paper_1810_10496_b200"
LIB = PKG / "libpfgpu.so"
OUT = PKG / "artifacts.json.gz"

BENCHES = (
    "2DCONV", "3DCONV", "2MM", "3MM", "ATAX", "BICG", "CORR", "COVAR", "FDTD-2D",
    "GEMM", "GESUMMV", "GRAMSCHM", "MVT", "SYR2K", "SYRK",
)

_TAG = re.compile(r"<\(pf::BenchId\)(\d+), (?:\(int\))?(\d+)[,>]")
_ADDR = re.compile(r"^\s*/\*[0-9a-f]{4,}\*/\s*")


def _tool(name: str) -> str:
    for cand in (shutil.which(name), f"/usr/local/cuda/bin/{name}"):
        if cand and Path(cand).exists():
            return cand
    raise FileNotFoundError(name)


def extract(lib: Path = LIB) -> dict[str, dict[str, str]]:
    sass = subprocess.run([_tool("cuobjdump"), "-sass", str(lib)], capture_output=True, text=True, check=True).stdout
    chunks: list[tuple[str, list[str]]] = []
    for line in sass.splitlines():
        stripped = line.strip()
        if stripped.startswith("Function : "):
            chunks.append((stripped[len("Function : "):], []))
        elif chunks:
            chunks[-1][1].append(line)
    mangled = [name for name, _ in chunks]
    demangled = subprocess.run([_tool("cu++filt")], input="\n".join(mangled), capture_output=True, text=True,
                               check=True).stdout.splitlines()
    groups: dict[tuple[int, int], list[tuple[str, str]]] = defaultdict(list)
    for (name, body), dem in zip(chunks, demangled):
        m = _TAG.search(dem)
        if not m:
            continue
        bench, variant = int(m.group(1)), int(m.group(2))
        base = dem.split("<", 1)[0].split("::")[-1]
        lines = []
        for ln in body:
            ln = _ADDR.sub("", ln).rstrip()
            if not ln or ln.lstrip().startswith((".section", ".headerflags")):
                continue
            lines.append(ln.strip())
        # kernels of one variant in a stable order: base name, then the
        # remaining (non-variant) template arguments
        rest = _TAG.sub("<", dem)
        groups[(bench, variant)].append((base + rest, "\n".join(lines)))
    table: dict[str, dict[str, str]] = {}
    for (bench, variant), funcs in sorted(groups.items()):
        funcs.sort(key=lambda t: t[0])
        text = "".join(f"== kernel {i}\n{body}\n" for i, (_, body) in enumerate(funcs))
        table.setdefault(BENCHES[bench], {})[str(variant)] = text
    return table


def main() -> int:
    if not LIB.exists():
        print(f"missing {LIB}; run make first", file=sys.stderr)
        return 1
    table = extract()
    payload = json.dumps({"version": 1, "benches": table}, sort_keys=True).encode()
    OUT.write_bytes(gzip.compress(payload, compresslevel=6, mtime=0))
    n = sum(len(v) for v in table.values())
    print(f"wrote {OUT.name}: {len(table)} benchmarks, {n} variants, {len(payload)} bytes uncompressed")
    return 0


if __name__ == "__main__":
    sys.exit(main())
