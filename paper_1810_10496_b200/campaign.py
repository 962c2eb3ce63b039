"""The paper's end-to-end flow on the B200 backend.

Mirrors the reference front door ``cmd_explore`` (`/root/reference/pkg/src/
phaseforge/cli.py:168-218`) for each benchmark of the registry:

  features -> baseline measure_average (final_reps) -> timeout override
  (4x baseline, cli.py:194-195) -> explore -> finalize -> reduce_order ->
  measure_average(reduced) -> KbEntry (empty order if no improvement)

then ``build_speedup_report`` (the headline geomean, results.py:125-140) and
the leave-one-out feature-transfer evaluation (``_cmd_loo``, cli.py:300-322 ->
advisor.leave_one_out) whose kNN curve gives the 1-NN / 3-NN numbers of the
paper.

Deviation, documented: each kernel gets its own ExplorationConfig with
rtol = 1e-4 (the north-star fp32 tolerance) and atol = rtol * max|reference
outputs|, because the validation outputs span many orders of magnitude
across kernels.
"""

from __future__ import annotations

import json
import math
import time
from dataclasses import dataclass, replace
from pathlib import Path

from . import advisor, explorer, passmodel, registry, results
from .backend.types import TIMED_STATUSES, BackendError, InputKind
from .catalog import PassCatalog, PhaseOrder, render_phase_order
from .irfeat import extract_features, parse_ir


@dataclass
class CampaignResult:
    kb: explorer.KnowledgeBase
    store: results.ResultsStore
    report: results.SpeedupReport
    loo: dict | None
    per_kernel: dict
    seconds: float


def kernel_config(base: explorer.ExplorationConfig, kernel, rtol: float = 1e-4) -> explorer.ExplorationConfig:
    scale = max((abs(x) for x in kernel.reference_outputs), default=1.0)
    return replace(base, rtol=rtol, atol=rtol * scale)


def _serial_map(fn, items, costs=None):
    return [fn(x) for x in items]


# ---------------------------------------------------------------- rank-parallel engine steps
# Each helper returns exactly what its explorer.* counterpart returns when every
# evaluation is deterministic; the independent evaluations inside it are
# spread over ranks by ``pmap`` (``Dist.map``) and gathered to every rank.

def explore_parallel(kernel, catalog, config, backend, pmap) -> list[explorer.EvaluationRecord]:
    """explore (explorer.py:152-192): compiles are pure, so every rank compiles
    the whole stream; the fresh evaluations (first order of each digest) are
    sharded; records are assembled identically on every rank."""
    if not kernel.reference_outputs:
        raise ValueError(f"kernel {kernel.id!r} has no reference outputs for validation")
    orders = explorer.draw_orders(catalog, config)
    compiled = [backend.compile(kernel, o) for o in orders]
    fresh, seen = [], set()
    for i, c in enumerate(compiled):
        if c.is_ok and c.artifact.digest not in seen:
            seen.add(c.artifact.digest)
            fresh.append(i)
    outcomes = pmap(lambda i: explorer._fresh_evaluation(backend, kernel, orders[i], compiled[i], config), fresh)
    by_digest = {compiled[i].artifact.digest: o for i, o in zip(fresh, outcomes)}
    records, first = [], {}
    for index, (order, c) in enumerate(zip(orders, compiled)):
        if not c.is_ok:
            records.append(explorer.EvaluationRecord(kernel.id, order, None, explorer.RecordStatus.NO_IR, None, index))
            continue
        d = c.artifact.digest
        if d in first:
            records.append(explorer.EvaluationRecord(kernel.id, order, d, explorer.RecordStatus.REUSED,
                                                     first[d].wall_time, index))
            continue
        o = by_digest[d]
        first[d] = explorer.EvaluationRecord(kernel.id, order, d, o.status, o.wall_time, index)
        records.append(first[d])
    return explorer._sorted_records(records)


def measure_average_parallel(backend, kernel, order, reps, config, pmap) -> float | None:
    """measure_average (explorer.py:217-235) with the reps sharded."""
    compiled = backend.compile(kernel, order)
    if not compiled.is_ok:
        return None

    def one(_):
        with backend.measurement_lock:
            run = backend.execute(kernel, order, compiled.artifact, InputKind.MEASUREMENT)
        return run.wall_time if run.status in TIMED_STATUSES else None

    samples = pmap(one, list(range(reps)))
    if any(s is None for s in samples):
        return None
    return math.fsum(samples) / len(samples)


def finalize_parallel(kernel, records, config, backend, pmap) -> tuple[PhaseOrder, float]:
    """finalize (explorer.py:271-324): each top-k candidate's revalidation and
    final_reps average run on one rank; the winner is picked in candidate order."""
    candidates = explorer._top_candidates(records, config.top_k)
    if not candidates:
        raise explorer.NoValidCandidateError(f"no valid exploration results for kernel {kernel.id!r}")
    baseline = backend.compile(kernel, PhaseOrder())
    if not baseline.is_ok:
        raise BackendError(f"baseline compile failed for kernel {kernel.id!r}")

    def one(order):
        compiled = backend.compile(kernel, order)
        if not compiled.is_ok:
            return None
        if not explorer._passes_random_input_validation(backend, kernel, order, compiled.artifact,
                                                        baseline.artifact, config):
            return None
        return explorer.measure_average(backend, kernel, order, config.final_reps, config)

    best_time = best_order = None
    for order, mean in zip(candidates, pmap(one, candidates)):
        if mean is not None and (best_time is None or mean < best_time):
            best_time, best_order = mean, order
    if best_order is None:
        raise explorer.NoValidCandidateError(
            f"all top-{len(candidates)} candidates failed revalidation for kernel {kernel.id!r}")
    return best_order, best_time


def reduce_order_parallel(kernel, order, backend, epsilon, config, pmap, width: int) -> PhaseOrder:
    """reduce_order (explorer.py:327-365) with speculative deletion windows:
    the trials for positions pos .. pos+width-1 are evaluated at once (each
    assumes the earlier ones in the window are rejected, which is what the
    sequential scan would have seen up to the first acceptance); the first
    accepted one is applied and the rest discarded.  width=1 is the
    sequential algorithm."""
    if epsilon < 0:
        raise ValueError(f"epsilon must be non-negative, got {epsilon}")
    start = pmap(lambda o: explorer.evaluate_candidate(backend, kernel, o, config), [order])[0]
    if start.status is not explorer.RecordStatus.VALID:
        raise ValueError(f"order must validate on kernel {kernel.id!r} before reduction (got {start.status.value})")
    best = start.wall_time
    passes = list(order.passes)
    progress = True
    while progress:
        progress = False
        pos = 0
        while pos < len(passes):
            window = list(range(pos, min(pos + max(1, width), len(passes))))
            trials = [PhaseOrder(tuple(passes[:p] + passes[p + 1:])) for p in window]
            got = pmap(lambda t: explorer.evaluate_candidate(backend, kernel, t, config), trials)
            for p, trial, g in zip(window, trials, got):
                if g.status is explorer.RecordStatus.VALID and g.wall_time <= (1.0 + epsilon) * best:
                    passes = list(trial.passes)
                    best = min(best, g.wall_time)
                    progress = True
                    pos = p
                    break
            else:
                pos = window[-1] + 1
    return PhaseOrder(tuple(passes))


def run_campaign(kernels, backend, config: explorer.ExplorationConfig, catalog: PassCatalog | None = None,
                 epsilon: float = 0.01, timeout_factor: float = 4.0, loo_k: int = 3, loo_trials: int = 100,
                 loo_seed: int = 1729, log=print, out_dir: str | Path | None = None, dist=None) -> CampaignResult:
    """The cmd_explore flow per kernel, then the report and LOO.  With ``dist``
    (world > 1) every step's independent evaluations are sharded over the
    ranks; every rank ends with the same KB, records,
    report and LOO table, and only rank 0 writes ``out_dir``."""
    catalog = catalog or passmodel.default_catalog()
    parallel = dist is not None and dist.world > 1
    pmap = dist.map if parallel else _serial_map
    width = dist.world if parallel else 1
    t0 = time.time()
    kb = explorer.KnowledgeBase()
    store = results.ResultsStore()
    per = {}
    for i, kernel in enumerate(kernels):
        tk = time.time()
        cfg = replace(kernel_config(config, kernel), seed=config.seed + i)
        features = extract_features(parse_ir(kernel.ir_text))
        if parallel:
            baseline = measure_average_parallel(backend, kernel, PhaseOrder(), cfg.final_reps, cfg, pmap)
        else:
            baseline = explorer.measure_average(backend, kernel, PhaseOrder(), cfg.final_reps, cfg)
        if baseline is None:
            raise RuntimeError(f"baseline measurement failed for {kernel.id}")
        backend.set_timeout_override(kernel.id, timeout_factor * baseline)
        if parallel:
            records = explore_parallel(kernel, catalog, cfg, backend, pmap)
        else:
            records = explorer.explore(kernel, catalog, cfg, backend)
        store.extend(records)
        fresh = [r for r in records if r.status is not explorer.RecordStatus.REUSED]
        try:
            if parallel:
                best, best_time = finalize_parallel(kernel, records, cfg, backend, pmap)
            else:
                best, best_time = explorer.finalize(kernel, records, cfg, backend)
        except explorer.NoValidCandidateError as exc:
            log(f"{kernel.id}: {exc}")
            kb.add(kernel.id, explorer.KbEntry(PhaseOrder(), baseline, baseline, features))
            continue
        if parallel:
            reduced = reduce_order_parallel(kernel, best, backend, epsilon, cfg, pmap, width)
            reduced_avg = measure_average_parallel(backend, kernel, reduced, cfg.final_reps, cfg, pmap)
        else:
            reduced = explorer.reduce_order(kernel, best, backend, epsilon, cfg)
            reduced_avg = explorer.measure_average(backend, kernel, reduced, cfg.final_reps, cfg)
        if reduced_avg is not None and reduced_avg < baseline:
            entry = explorer.KbEntry(reduced, reduced_avg, baseline, features)
        else:
            entry = explorer.KbEntry(PhaseOrder(), baseline, baseline, features)
        kb.add(kernel.id, entry)
        per[kernel.id] = {
            "baseline_s": baseline, "best_s": entry.best_time, "speedup": baseline / entry.best_time,
            "finalized_order_len": len(best), "reduced_order": render_phase_order(entry.best_order),
            "records": len(records), "fresh_evaluations": len(fresh),
            "statuses": {s.value: sum(1 for r in records if r.status is s) for s in explorer.RecordStatus},
            "seconds": time.time() - tk,
        }
        if hasattr(backend, "variant_for"):
            from .backend.b200 import family

            variant = backend.variant_for(kernel, entry.best_order)[1]
            per[kernel.id]["variant"] = family(registry.bench_of(kernel)).key(variant)
        log(f"{kernel.id:9s} baseline {baseline * 1e3:10.3f} ms  best {entry.best_time * 1e3:9.3f} ms  "
            f"x{baseline / entry.best_time:8.2f}  [{per[kernel.id].get('variant', '')}]  "
            f"fresh {len(fresh)}/{len(records)}  '{render_phase_order(entry.best_order)}'  "
            f"({time.time() - tk:.0f}s)")
    report = results.build_speedup_report(kb)
    log(f"geomean speedup over baseline ({len(kb.entries)} kernels): {report.geomean:.3f}x")
    loo = None
    if loo_k and len(kb.entries) > 1:
        refset = advisor.ReferenceSet.from_knowledge_base(kb)
        by_id = {k.id: k for k in kernels}
        cache_was = getattr(backend, "measurement_cache", None)
        if hasattr(backend, "measurement_cache"):
            backend.measurement_cache = {} if cache_was is None else cache_was
        loo_cfg = replace(config, final_reps=1, final_random_inputs=1)
        loo = _loo_per_kernel(refset, [by_id[k] for k in kb.entries], backend, loo_k, loo_trials, loo_seed, loo_cfg,
                              pmap)
        if hasattr(backend, "measurement_cache"):
            backend.measurement_cache = cache_was
        log("leave-one-out geomean speedup: " + ", ".join(
            f"{m}: " + " ".join(f"{v:.3f}" for v in curve) for m, curve in loo.items()))
    res = CampaignResult(kb, store, report, loo, per, time.time() - t0)
    if out_dir is not None and (dist is None or dist.rank == 0):
        save(res, out_dir)
    return res


def _loo_per_kernel(refset, kernels, backend, k_max, trials, seed, config, pmap=_serial_map):
    """advisor.leave_one_out (advisor.py:273-308), each kernel evaluated under
    its own tolerance and on one rank; the log-curves are summed in kernel
    order on every rank."""
    tables = pmap(lambda kernel: advisor.leave_one_out(refset, [kernel], backend, k_max, trials=trials, seed=seed,
                                                       config=kernel_config(config, kernel)), kernels)
    logs = {m: [0.0] * k_max for m in advisor.LOO_METHODS}
    for table in tables:
        for m, curve in table.items():
            for i, v in enumerate(curve):
                logs[m][i] += math.log(v)
    return {m: [math.exp(s / len(kernels)) for s in logs[m]] for m in advisor.LOO_METHODS}


def save(res: CampaignResult, out_dir: str | Path) -> None:
    out = Path(out_dir)
    out.mkdir(parents=True, exist_ok=True)
    res.kb.save(out / "kb.json")
    results.export_records_csv(res.store.records, out / "records.csv")
    results.export_report_json(res.report, out / "report.json")
    results.export_report_csv(res.report, out / "report.csv")
    if res.loo is not None:
        results.export_loo_csv(res.loo, out / "loo.csv")
    summary = {"geomean_speedup": res.report.geomean, "loo": res.loo, "per_kernel": res.per_kernel,
               "seconds": res.seconds,
               "failure_summary": {k.value: v for k, v in results.failure_summary(res.store).items()}}
    (out / "summary.json").write_text(json.dumps(summary, indent=1, sort_keys=True) + "\n")


__all__ = ["CampaignResult", "kernel_config", "run_campaign", "save"]
