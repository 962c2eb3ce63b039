"""The paper's two secondary studies on the B200 backend.

* Cross-application matrix (Fig. 3): every kernel's best order applied to
  every other kernel -- ``explorer.cross_apply`` (`/root/reference/pkg/src/
  phaseforge/explorer.py:386-410`), front door ``_cmd_cross_apply``
  (cli.py:245-257), written with ``export_matrix_csv`` (results.py).
* Permutation study (Fig. 5): random permutations of each kernel's best
  order, bucketed by time(best)/time(permutation) -- ``_cmd_permute``
  (cli.py:260-297) over ``random_permutations`` (catalog.py:172-192) and
  ``permutation_histogram`` (results.py:156-194).

Both follow the reference flows exactly, with one documented deviation shared
with ``campaign``: each target kernel is validated under its own tolerance
(rtol, atol = rtol * max|reference outputs|).  Permutation orders that map to
an already-measured artifact may reuse its measurement (``reuse=True``, the
"identical machine code, identical performance" premise of explorer.py:175-183),
which keeps a 1000-permutation study to minutes.
"""

from __future__ import annotations

import json
import time
from pathlib import Path
from random import Random

from . import explorer, results
from .campaign import kernel_config
from .catalog import PhaseOrder, random_permutations, render_phase_order
from .explorer import CellResult, CrossApplyMatrix, EvaluationRecord, RecordStatus, evaluate_candidate


def cross_apply_matrix(kernels, kb: explorer.KnowledgeBase, backend, config: explorer.ExplorationConfig,
                       per_kernel_tolerance: bool = True) -> CrossApplyMatrix:
    """Cell (owner, target) = best_time(target) / time(target under owner's best order)."""
    missing = [k.id for k in kernels if k.id not in kb.entries]
    if missing:
        raise ValueError(f"knowledge base has no entry for kernel {missing[0]!r}")
    cells: dict[tuple[str, str], CellResult] = {}
    for owner in kernels:
        order = kb.entries[owner.id].best_order
        for target in kernels:
            cfg = kernel_config(config, target, config.rtol) if per_kernel_tolerance else config
            got = evaluate_candidate(backend, target, order, cfg)
            if got.status is RecordStatus.VALID:
                cells[(owner.id, target.id)] = CellResult(kb.entries[target.id].best_time / got.wall_time, False)
            else:
                cells[(owner.id, target.id)] = CellResult(None, True)
    return CrossApplyMatrix(tuple(k.id for k in kernels), cells)


def permutation_study(kernels, kb: explorer.KnowledgeBase, backend, config: explorer.ExplorationConfig,
                      trials: int = 1000, seed: int = 1729, bucket_width: float = 0.1,
                      per_kernel_tolerance: bool = True):
    """{kernel id: (records, histogram)} for kernels with a non-empty best
    order; one shared RNG across kernels, as cli.py:267 draws it."""
    rng = Random(seed)
    out = {}
    for kernel in kernels:
        best = kb.entries[kernel.id].best_order
        if len(best) == 0:
            continue
        orders = [best] + [p for p in random_permutations(best, trials, rng) if p.passes != best.passes]
        cfg = kernel_config(config, kernel, config.rtol) if per_kernel_tolerance else config
        records = []
        for index, order in enumerate(orders):
            got = evaluate_candidate(backend, kernel, order, cfg)
            records.append(EvaluationRecord(kernel.id, order, got.digest, got.status, got.wall_time, index))
        out[kernel.id] = (records, results.permutation_histogram(records, bucket_width))
    return out


def write_permute_csv(study: dict, path: str | Path) -> None:
    """The ``permute.csv`` layout of cli.py:287-296."""
    with open(path, "w", newline="") as fh:
        fh.write("kernel_id,bucket_low,bucket_high,percent\n")
        for kid, (_, hist) in study.items():
            for b in hist.buckets:
                fh.write(f"{kid},{b.low:.6f},{b.high:.6f},{b.percent:.6f}\n")
            fh.write(f"{kid},FAIL,FAIL,{hist.failure_percent:.6f}\n")


def run_study(kernels, kb: explorer.KnowledgeBase, backend, config: explorer.ExplorationConfig,
              out_dir: str | Path, trials: int = 1000, seed: int = 1729, bucket_width: float = 0.1,
              reuse: bool = True, log=print) -> dict:
    out = Path(out_dir)
    out.mkdir(parents=True, exist_ok=True)
    kernels = [k for k in kernels if k.id in kb.entries]
    saved = getattr(backend, "measurement_cache", None)
    if reuse and hasattr(backend, "measurement_cache"):
        backend.measurement_cache = {}
    try:
        t0 = time.time()
        matrix = cross_apply_matrix(kernels, kb, backend, config)
        t_matrix = time.time() - t0
        results.export_matrix_csv(matrix, out / "matrix.csv")
        results.export_matrix_json(matrix, out / "matrix.json")
        log(f"cross-application matrix {len(kernels)}x{len(kernels)} in {t_matrix:.0f}s")
        t0 = time.time()
        perm = permutation_study(kernels, kb, backend, config, trials, seed, bucket_width)
        t_perm = time.time() - t0
        write_permute_csv(perm, out / "permute.csv")
        results.export_records_csv([r for recs, _ in perm.values() for r in recs], out / "permute_records.csv")
    finally:
        if hasattr(backend, "measurement_cache"):
            backend.measurement_cache = saved
    ids = matrix.kernel_ids
    off = [matrix.cells[(o, t)] for o in ids for t in ids if o != t]
    summary = {
        "kernels": list(ids),
        "diagonal": {k: matrix.cells[(k, k)].ratio for k in ids},
        "off_diagonal_fail_fraction": sum(c.failed for c in off) / max(1, len(off)),
        "off_diagonal_mean_ratio": (sum(min(1.0, c.ratio) for c in off if not c.failed)
                                    / max(1, sum(not c.failed for c in off))),
        "permutations": {
            kid: {"best_order": render_phase_order(kb.entries[kid].best_order), "evaluated": len(recs),
                  "distinct_digests": len({r.artifact_digest for r in recs if r.artifact_digest}),
                  "at_least_0.9_of_best_percent": sum(b.percent for b in hist.buckets if b.low >= 0.9 - 1e-9),
                  "failure_percent": hist.failure_percent}
            for kid, (recs, hist) in perm.items()},
        "seconds": {"matrix": t_matrix, "permutations": t_perm},
        "measurement_reuse_by_digest": reuse,
    }
    (out / "study.json").write_text(json.dumps(summary, indent=1, sort_keys=True) + "\n")
    for kid, p in summary["permutations"].items():
        log(f"{kid:9s} perms {p['evaluated']:5d} digests {p['distinct_digests']:3d} "
            f">=0.9x best {p['at_least_0.9_of_best_percent']:5.1f}%  fail {p['failure_percent']:5.1f}%")
    return summary


__all__ = ["cross_apply_matrix", "permutation_study", "run_study", "write_permute_csv"]
