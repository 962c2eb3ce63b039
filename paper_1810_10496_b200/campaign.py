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
import time
from dataclasses import dataclass, replace
from pathlib import Path

from . import advisor, explorer, passmodel, registry, results
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


def run_campaign(kernels, backend, config: explorer.ExplorationConfig, catalog: PassCatalog | None = None,
                 epsilon: float = 0.01, timeout_factor: float = 4.0, loo_k: int = 3, loo_trials: int = 100,
                 loo_seed: int = 1729, log=print, out_dir: str | Path | None = None) -> CampaignResult:
    catalog = catalog or passmodel.default_catalog()
    t0 = time.time()
    kb = explorer.KnowledgeBase()
    store = results.ResultsStore()
    per = {}
    for i, kernel in enumerate(kernels):
        tk = time.time()
        cfg = replace(kernel_config(config, kernel), seed=config.seed + i)
        features = extract_features(parse_ir(kernel.ir_text))
        baseline = explorer.measure_average(backend, kernel, PhaseOrder(), cfg.final_reps, cfg)
        if baseline is None:
            raise RuntimeError(f"baseline measurement failed for {kernel.id}")
        backend.set_timeout_override(kernel.id, timeout_factor * baseline)
        records = explorer.explore(kernel, catalog, cfg, backend)
        store.extend(records)
        fresh = [r for r in records if r.status is not explorer.RecordStatus.REUSED]
        try:
            best, best_time = explorer.finalize(kernel, records, cfg, backend)
        except explorer.NoValidCandidateError as exc:
            log(f"{kernel.id}: {exc}")
            kb.add(kernel.id, explorer.KbEntry(PhaseOrder(), baseline, baseline, features))
            continue
        reduced = explorer.reduce_order(kernel, best, backend, epsilon, cfg)
        reduced_avg = explorer.measure_average(backend, kernel, reduced, cfg.final_reps, cfg)
        if reduced_avg is not None and reduced_avg < baseline:
            entry = explorer.KbEntry(reduced, reduced_avg, baseline, features)
        else:
            entry = explorer.KbEntry(PhaseOrder(), baseline, baseline, features)
        kb.add(kernel.id, entry)
        variant = backend.variant_for(kernel, entry.best_order)[1]
        from .backend.b200 import family

        per[kernel.id] = {
            "baseline_s": baseline, "best_s": entry.best_time, "speedup": baseline / entry.best_time,
            "finalized_order_len": len(best), "reduced_order": render_phase_order(entry.best_order),
            "variant": family(registry.bench_of(kernel)).key(variant),
            "records": len(records), "fresh_evaluations": len(fresh),
            "statuses": {s.value: sum(1 for r in records if r.status is s) for s in explorer.RecordStatus},
            "seconds": time.time() - tk,
        }
        log(f"{kernel.id:9s} baseline {baseline * 1e3:10.3f} ms  best {entry.best_time * 1e3:9.3f} ms  "
            f"x{baseline / entry.best_time:8.2f}  [{per[kernel.id]['variant']}]  "
            f"fresh {len(fresh)}/{len(records)}  '{render_phase_order(entry.best_order)}'  "
            f"({time.time() - tk:.0f}s)")
    report = results.build_speedup_report(kb)
    log(f"geomean speedup over baseline (15 kernels): {report.geomean:.3f}x")
    loo = None
    if loo_k and len(kb.entries) > 1:
        refset = advisor.ReferenceSet.from_knowledge_base(kb)
        by_id = {k.id: k for k in kernels}
        cache_was = getattr(backend, "measurement_cache", None)
        if hasattr(backend, "measurement_cache"):
            backend.measurement_cache = {} if cache_was is None else cache_was
        loo_cfg = replace(config, final_reps=1, final_random_inputs=1)
        # per-kernel tolerance: evaluate each kernel with its own config
        loo = _loo_per_kernel(refset, [by_id[k] for k in kb.entries], backend, loo_k, loo_trials, loo_seed, loo_cfg)
        if hasattr(backend, "measurement_cache"):
            backend.measurement_cache = cache_was
        log("leave-one-out geomean speedup: " + ", ".join(
            f"{m}: " + " ".join(f"{v:.3f}" for v in curve) for m, curve in loo.items()))
    res = CampaignResult(kb, store, report, loo, per, time.time() - t0)
    if out_dir is not None:
        save(res, out_dir)
    return res


def _loo_per_kernel(refset, kernels, backend, k_max, trials, seed, config):
    """advisor.leave_one_out, with each kernel evaluated under its own tolerance."""
    import math

    logs = {m: [0.0] * k_max for m in advisor.LOO_METHODS}
    for kernel in kernels:
        cfg = kernel_config(config, kernel)
        table = advisor.leave_one_out(refset, [kernel], backend, k_max, trials=trials, seed=seed, config=cfg)
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
