"""GPU parity: every variant of every built benchmark vs the CPU oracle.

Each variant runs through the C-ABI (libpfgpu.so) on the stock validation
input and on two random inputs; its outputs must match the oracle
(oracle/liborc.so) within rtol = 1e-4 per element with an absolute floor of
1e-4 * max|ref| per output array (BASELINE.json north_star tolerance; the
floor handles near-zero outputs of mixed-sign stencils and centred data).
Input generation is checked bit-exactly against the oracle's generators.
"""

from __future__ import annotations

import numpy as np
import pytest

from oracle import oracle as orc
from paper_1810_10496_b200 import registry

pytestmark = pytest.mark.gpu

RTOL = 1e-4
ATOL_REL = 1e-4


def _close(got: np.ndarray, ref: np.ndarray) -> tuple[bool, float]:
    ref64 = ref.astype(np.float64)
    atol = ATOL_REL * float(np.max(np.abs(ref64))) if ref.size else 0.0
    diff = np.abs(got.astype(np.float64) - ref64)
    tol = np.maximum(atol, RTOL * np.abs(ref64))
    worst = float(np.max(diff / np.maximum(tol, 1e-300))) if ref.size else 0.0
    return bool(np.all(diff <= tol)), worst


def _built(name):
    from paper_1810_10496_b200.backend import b200

    try:
        b200.family(name)
        return True
    except Exception:
        return False


BUILT = [b for b in registry.BENCHES if _built(b)]


@pytest.mark.parametrize("bench", BUILT)
def test_inputs_bit_exact(bench, gpu_backend):
    dims = registry.SIZES[bench]["validation"]
    for stock, inst in ((True, -1), (False, 0), (False, 7)):
        ws = gpu_backend.workspace(bench, dims, stock, inst)
        ws.restore()  # earlier tests may have run variants on this cached workspace
        ref = orc.generate(bench, dims, stock, gpu_backend.seed, inst)
        for a, (name, role, _) in enumerate(ws.arrays):
            got = ws.download(a)
            assert np.array_equal(got, ref[a]), f"{bench} array {name} (stock={stock}, inst={inst}) differs"


@pytest.mark.parametrize("bench", BUILT)
def test_all_variants_match_oracle(bench, gpu_backend):
    from paper_1810_10496_b200.backend import b200

    fam = b200.family(bench)
    dims = registry.SIZES[bench]["validation"]
    failures = []
    for stock, inst in ((True, -1), (False, 1)):
        ref = orc.reference(bench, dims, stock, gpu_backend.seed, inst)
        for v in range(len(fam.knobs)):
            if not gpu_backend._supported(bench, v, dims):
                continue
            ws = gpu_backend.workspace(bench, dims, stock, inst)
            ws.run(v, samples=1, batch=1, restore=True, flush=False)
            outs = ws.outputs()
            for k, (g, r) in enumerate(zip(outs, ref)):
                ok, worst = _close(g, r)
                if not ok:
                    failures.append(f"v{v} [{fam.key(v)}] out{k} stock={stock}: worst/tol={worst:.3g}")
    assert not failures, "\n".join(failures[:40])


# Ragged sizes: non-multiples of the tile/vector widths (variants whose
# alignment constraints reject them are skipped through pf_variant_supported),
# odd FDTD step counts (double-buffer copy-back), M != N for GRAMSCHM.
EDGE = {
    "2DCONV": (67, 93), "3DCONV": (19, 23, 29), "2MM": (67, 45, 33, 51), "3MM": (37, 45, 29, 51, 33),
    "ATAX": (173, 201), "BICG": (173, 201), "CORR": (61, 77), "COVAR": (61, 77), "FDTD-2D": (37, 53, 7),
    "GEMM": (61, 67, 53), "GESUMMV": (301,), "GRAMSCHM": (73, 61), "MVT": (301,), "SYR2K": (77, 53),
    "SYRK": (77, 53),
}


@pytest.mark.parametrize("bench", BUILT)
def test_edge_sizes_match_oracle(bench, gpu_backend):
    from paper_1810_10496_b200.backend import b200

    fam = b200.family(bench)
    dims = EDGE[bench]
    ref = orc.reference(bench, dims, False, gpu_backend.seed, 3)
    failures, ran = [], 0
    for v in range(len(fam.knobs)):
        if not gpu_backend._supported(bench, v, dims):
            continue
        ws = gpu_backend.workspace(bench, dims, False, 3)
        ws.run(v, samples=1, batch=1, restore=True, flush=False)
        ran += 1
        for k, (g, r) in enumerate(zip(ws.outputs(), ref)):
            ok, worst = _close(g, r)
            if not ok:
                failures.append(f"v{v} [{fam.key(v)}] out{k}: worst/tol={worst:.3g}")
    assert ran > 0
    assert not failures, "\n".join(failures[:40])


# Tensor-core tile paths: sizes >= 256 select the CTA-pair (cta_group::2,
# 256x256) kernel, GEMM 512^3 adds split-K, ragged multiples of 4 exercise the
# TMA out-of-bounds fill and the partial-tile epilogue; CORR/COVAR's 1-based
# arrays take the packed-operand kernel.
TC_SIZES = {
    "GEMM": [(512, 512, 512), (260, 516, 132)],
    "2MM": [(384, 260, 300, 516)],
    "3MM": [(256, 260, 384, 300, 268)],
    "SYRK": [(520, 260)],
    "SYR2K": [(264, 300)],
    "CORR": [(300, 264)],
    "COVAR": [(300, 264)],
}


@pytest.mark.parametrize("bench", [b for b in TC_SIZES if b in BUILT])
def test_tensor_core_tiles_match_oracle(bench, gpu_backend):
    from paper_1810_10496_b200.backend import b200

    fam = b200.family(bench)
    keys = [v for v in range(len(fam.knobs)) if fam.key(v) == "stage=2"]
    assert keys
    failures = []
    for dims in TC_SIZES[bench]:
        ref = orc.reference(bench, dims, False, gpu_backend.seed, 5)
        for v in keys:
            assert gpu_backend._supported(bench, v, dims), (bench, dims)
            ws = gpu_backend.workspace(bench, dims, False, 5)
            ws.run(v, samples=1, batch=1, restore=True, flush=False)
            for k, (g, r) in enumerate(zip(ws.outputs(), ref)):
                ok, worst = _close(g, r)
                if not ok:
                    failures.append(f"{dims} v{v} out{k}: worst/tol={worst:.3g}")
    assert not failures, "\n".join(failures)


# Config-scale tensor-core paths the small sizes above never reach: CTA-pair
# tiles without split-K (operands pre-split into lo images, TMA epilogue with
# beta, chained lo images), pair tiles with a 2-way split (ordered in-kernel
# hand-over, TMA add-reductions), the K-concatenated SYR2K product, and CORR's
# upper-triangle split.
TC_LARGE_SIZES = {
    # (2048, 2048, 256, 2048) / 3MM: the later product consumes the lo image
    # that the earlier product's epilogue wrote
    "2MM": [(2048, 2048, 256, 1024), (2048, 2048, 256, 2048)],
    "3MM": [(2048, 2048, 256, 2048, 256)],
    "SYRK": [(2048, 512)],
    "SYR2K": [(2048, 256)],
    "CORR": [(2048, 256)],
}


@pytest.mark.parametrize("bench", [b for b in TC_LARGE_SIZES if b in BUILT])
def test_tensor_core_config_paths_match_oracle(bench, gpu_backend):
    from paper_1810_10496_b200.backend import b200

    fam = b200.family(bench)
    v = next(i for i in range(len(fam.knobs)) if fam.key(i) == "stage=2")
    failures = []
    for dims in TC_LARGE_SIZES[bench]:
        ref = orc.reference(bench, dims, False, gpu_backend.seed, 7)
        ws = gpu_backend.workspace(bench, dims, False, 7)
        ws.run(v, samples=1, batch=1, restore=True, flush=False)
        for k, (g, r) in enumerate(zip(ws.outputs(), ref)):
            ok, worst = _close(g, r)
            if not ok:
                failures.append(f"{dims} out{k}: worst/tol={worst:.3g}")
    assert not failures, "\n".join(failures)


# Stencil tiling edges: partial 128-wide k tiles, j tiles and i runs that end
# mid-tile, tiny volumes where a run spans several column tiles.
# FDTD-2D: the register-tiled temporal blocking (stage 2) needs ny % 4 == 0 and
# only spans several column tiles when ny > 112; enough steps that region-edge
# errors would reach the stored columns and rows (halo width).
STENCIL_SIZES = {"3DCONV": [(37, 45, 132), (9, 20, 8), (64, 33, 260)], "2DCONV": [(67, 516), (5, 8)],
                 "FDTD-2D": [(64, 256, 12), (128, 512, 30), (40, 1000, 13), (150, 236, 9)]}


@pytest.mark.parametrize("bench", [b for b in STENCIL_SIZES if b in BUILT])
def test_stencil_tiles_match_oracle(bench, gpu_backend):
    from paper_1810_10496_b200.backend import b200

    fam = b200.family(bench)
    failures, ran = [], 0
    for dims in STENCIL_SIZES[bench]:
        ref = orc.reference(bench, dims, False, gpu_backend.seed, 2)
        for v in range(len(fam.knobs)):
            if fam.knobs[v][0] == 0 or not gpu_backend._supported(bench, v, dims):
                continue
            ws = gpu_backend.workspace(bench, dims, False, 2)
            ws.run(v, samples=1, batch=1, restore=True, flush=False)
            ran += 1
            for k, (g, r) in enumerate(zip(ws.outputs(), ref)):
                ok, worst = _close(g, r)
                if not ok:
                    failures.append(f"{dims} v{v} [{fam.key(v)}] out{k}: worst/tol={worst:.3g}")
    assert ran > 0
    assert not failures, "\n".join(failures)
