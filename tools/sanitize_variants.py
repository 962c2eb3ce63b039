#!/usr/bin/env python3
"""Run every variant of one (or every) benchmark once at its validation size,
for compute-sanitizer (memcheck / racecheck / synccheck):

    compute-sanitizer --tool memcheck python tools/sanitize_variants.py GEMM

Prints one line per variant and a final count; the sanitizer's report goes to
its own log.  The outputs are not checked here (tests/test_gpu_parity.py does
that); the point is out-of-bounds accesses, shared-memory races and
barrier misuse in the kernels, including the inter-CTA flag protocols
(ordered split-K hand-over, GRAMSCHM panels, FDTD double buffers).
"""

from __future__ import annotations

import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

from paper_1810_10496_b200 import registry  # noqa: E402
from paper_1810_10496_b200.backend.b200 import B200Backend, family  # noqa: E402


def main(argv) -> int:
    benches = argv[1:] or list(registry.BENCHES)
    be = B200Backend(device=0, samples=1)
    ran = 0
    for bench in benches:
        dims = registry.SIZES[bench]["validation"]
        fam = family(bench)
        for v in range(len(fam.knobs)):
            if not be._supported(bench, v, dims):
                continue
            ws = be.workspace(bench, dims, True, -1)
            ws.run(v, samples=1, batch=1, restore=True, flush=False)
            ran += 1
            print(f"{bench} v{v} {fam.key(v)}", flush=True)
    be.close()
    print(f"ran {ran} variants of {len(benches)} benchmarks", flush=True)
    return 0


if __name__ == "__main__":
    sys.exit(main(sys.argv))
