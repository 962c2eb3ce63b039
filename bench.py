#!/usr/bin/env python3
"""Benchmark: candidate evaluations/s of the exploration loop on the BLAS-2 set.

Workload (BASELINE.json configs[1]): ATAX, BICG, MVT and GESUMMV at
N = 16384, fp32.  One *step* is one exploration round of the product path
-- ``explore()`` (explorer.py, the reference's loop restated) on each of the
four kernels over a fresh 1000-order stream (max_len 256, the default pass
catalog), through ``B200Backend`` with its device work batched ahead
(``sweep.explore_suite``: compile lookup, digest dedup / REUSED records,
validation run + output compare, one CUDA-event-timed measurement run per
fresh candidate after an L2 flush).  ``value`` is fresh evaluations/s (the
paper's unit: one validation + one measurement of a new artifact), whole
job (sum over ranks / max step time over ranks); every step draws new
orders (seed changes per step and rank), so compiles and candidates are new
work each step.

Each rank drives one GPU (one process per GPU, torchrun) with its own
order streams: weak scaling, no data-path collective;
torch.distributed is used only for the barrier and the max-over-ranks
timing reduction.

Extra keys: ``e2e`` (the same explore() round with every input array --
validation and measurement, 5.4 GB per step -- uploaded from pinned host
memory inside the timed region, outputs read back), ``roofline`` (GESUMMV's
stage-2 kernel as timed inside the steps vs the measured HBM peak),
``cpu_baseline`` (the reference's own path on the host: its unmodified
explore() + ToolchainBackend with the oracle runner, a bounded sample; plus
the oracle kernels single-thread / all threads and the reference explore()
on its simulator), ``geomean_speedup``, ``clocks``, ``gpu_launches``.

``--impl reference`` runs the reference's path alone on the host (rank 0):
its unmodified explore() driving ToolchainBackend, whose runner process
computes each kernel with the CPU oracle on all host threads (oracle/
pf_cpu_runner; PolyBench/GPU is not part of the reference), over a bounded
sample of orders per kernel and step.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time
from dataclasses import replace
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "geomean speedup specialized vs baseline variant; HBM GB/s / % peak; evals/sec @1-8 GPU"
KERNELS = ("ATAX", "BICG", "MVT", "GESUMMV")


def _peaks() -> dict:
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return {"hbm_gbs": float(d["hbm_gbs"]), "source": "measured"}
    return {"hbm_gbs": 6650.0, "source": "fallback"}


def _dims(bench: str, n: int) -> tuple[int, ...]:
    return (n, n) if bench in ("ATAX", "BICG") else (n,)


def _workload(n: int) -> str:
    return f"BLAS-2 set ATAX/BICG/MVT/GESUMMV, N={n} fp32 (BASELINE configs[1]): explore() rounds"


# ---------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled every 200 ms."""

    FIELDS = ("clocks.sm", "clocks.max.sm", "clocks_event_reasons.active", "clocks_event_reasons.hw_slowdown",
              "clocks_event_reasons.hw_thermal_slowdown", "clocks_event_reasons.sw_thermal_slowdown",
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows: list[list[str]] = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", "--query-gpu=" + ",".join(self.FIELDS),
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self) -> dict:
        sm = [float(r[0]) for r in self.rows if r and r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if len(r) > 1 and r[1].replace(".", "").isdigit()]
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        reasons = set()
        for r in self.rows:
            for name, v in zip(names, r[3:7]):
                if v.lower() == "active":
                    reasons.add(name)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


# ---------------------------------------------------------------- distributed plumbing
from paper_1810_10496_b200.dist import Dist  # noqa: E402


class StepTimer:
    """Device-side timing of one step: CUDA events on torch's current stream,
    recorded after a full device synchronize on both sides (the step is a
    host + device pipeline: the events bracket all of it)."""

    def __init__(self):
        import torch

        self.torch = torch
        self.pairs = []

    def __enter__(self):
        t = self.torch
        t.cuda.synchronize()
        self.a, self.b = t.cuda.Event(enable_timing=True), t.cuda.Event(enable_timing=True)
        self.a.record()
        return self

    def __exit__(self, *exc):
        self.b.record()
        self.torch.cuda.synchronize()
        self.pairs.append(self.a.elapsed_time(self.b))

    @property
    def ms(self) -> float:
        return self.pairs[-1]


# ---------------------------------------------------------------- reference-side CPU legs
def _ref_setup(n: int):
    from oracle import ref_arm
    from paper_1810_10496_b200 import passmodel

    pf = ref_arm.reference_engine()
    if pf is None:
        return None
    work = ref_arm.workdir()
    be = ref_arm.toolchain_backend(pf, work)
    dims = {b: _dims(b, n) for b in KERNELS}
    cases = ref_arm.kernel_cases(pf, KERNELS, dims, work)
    names = [p.name for p in passmodel.default_catalog().passes]
    return ref_arm, pf, be, cases, names, dims


def cpu_baseline(n: int, orders: int) -> dict:
    """The reference's CPU path on a bounded sample (rank 0, N=1)."""
    setup = _ref_setup(n)
    from oracle import ref_arm

    dims = {b: _dims(b, n) for b in KERNELS}
    out = {"cpu_model": ref_arm.cpu_model(), "host_cores": ref_arm.cores()}
    out.update(ref_arm.oracle_rates(KERNELS, dims, min_seconds=2.0))
    if setup is None:
        mt = out["oracle_mt"]
        out.update({"value": mt["evals_per_s"], "unit": "evals/s", "cores": mt["cores"], "kind": "port",
                    "sample": f"{mt['evals']} oracle kernel evaluations at N={n} (reference package absent)"})
        return out
    ref_arm_mod, pf, be, cases, names, _ = setup
    fresh, recs, secs = ref_arm.explore_step(pf, be, cases, names, orders, 1729)
    out.update({"value": fresh / secs, "unit": "evals/s", "cores": ref_arm.cores(), "kind": "port",
                "sample": f"phaseforge.explore + ToolchainBackend (oracle runner, all threads), {orders} orders x "
                          f"{len(KERNELS)} kernels at N={n}: {fresh} fresh evaluations in {secs:.2f} s"})
    out["reference_simulator_explore"] = ref_arm.simulator_rate(pf, names)
    return out


def run_reference(args, dist: Dist) -> int:
    if dist.rank != 0:
        return 0
    setup = _ref_setup(args.n)
    if setup is None:
        print(json.dumps({"impl": "reference", "unavailable": "reference package not importable "
                          "(neither /root/reference/pkg/src nor baseline/_ref)"}), flush=True)
        return 0
    ref_arm, pf, be, cases, names, _ = setup
    for w in range(args.warmup):
        ref_arm.explore_step(pf, be, cases, names, args.ref_orders, 1729 + 104729 * (w + 1))
    fresh = recs = valid = 0
    secs = 0.0
    for s in range(args.steps):
        f, r, t = ref_arm.explore_step(pf, be, cases, names, args.ref_orders, 1729 + 104729 * (1000 + s))
        fresh, recs, secs, valid = fresh + f, recs + r, secs + t, valid + ref_arm.explore_step.valid
    value = fresh / secs
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "evals/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * secs / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic (PolyBench/GPU init formulas)",
        "config": {"workload": _workload(args.n), "n": args.n, "kernels": list(KERNELS),
                   "orders_per_kernel_per_step": args.ref_orders, "max_len": 256,
                   "path": "phaseforge.explore (unmodified) -> ToolchainBackend: 4 compile-stage processes per "
                           "candidate, 1 runner process per execute (oracle/pf_cpu_runner, CPU oracle kernels)"},
        "fresh_evaluations": fresh, "records": recs, "valid_fraction": valid / max(1, fresh),
        "cpu_baseline": {"value": value, "unit": "evals/s", "cores": ref_arm.cores(), "kind": "port",
                         "cpu_model": ref_arm.cpu_model(),
                         "sample": f"{args.steps} steps x {len(KERNELS)} kernels x {args.ref_orders} orders "
                                   f"(every order a distinct artifact) at N={args.n}"},
        "e2e": {"value": value, "unit": "evals/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------- GPU side
def _stock_host_inputs(be, cases, keep):
    """Pinned host copies of every generated input array (validation and
    measurement workspaces) -- the data the runner would load -- and the
    bytes per upload round."""
    from paper_1810_10496_b200 import _abi, registry
    from paper_1810_10496_b200.backend.b200 import _Staging
    import ctypes
    import numpy as np

    table, h2d = {}, 0
    for case in cases:
        for kind, desc in (("validation", case.validation_input), ("measurement", case.measurement_input)):
            bench, dims = registry.parse_descriptor(desc)
            ws = be.workspace(bench, dims, True, -1)
            ptrs = {}
            for a, (_, role, _) in enumerate(ws.arrays):
                if role == _abi.ROLE_OUT:
                    continue
                st = _Staging(_abi.lib(), 4 * ws.elems[a])
                keep.append(st)
                np.ctypeslib.as_array((ctypes.c_float * ws.elems[a]).from_address(st.ptr))[:] = ws.download(a)
                ptrs[a] = st.ptr
                h2d += 4 * ws.elems[a]
            table[(case.id, kind)] = ptrs
    return table, h2d


def run_gpu(args, dist: Dist) -> int:
    from paper_1810_10496_b200 import passmodel, registry
    from paper_1810_10496_b200.backend.b200 import B200Backend, alg_work, family
    from paper_1810_10496_b200.campaign import kernel_config
    from paper_1810_10496_b200.explorer import ExplorationConfig, RecordStatus
    from paper_1810_10496_b200.sweep import explore_suite

    peaks = _peaks()
    device = dist.local
    be = B200Backend(device=device, samples=1, flush_l2=True)
    n = args.n
    cases = registry.build_suite(be, size="config", benches=KERNELS) if n == 16384 else [
        registry.kernel_case(b, measurement_dims=_dims(b, n)) for b in KERNELS]
    if n != 16384:
        cases = [replace(c, reference_outputs=be.baseline_outputs(c)) for c in cases]
    catalog = passmodel.default_catalog()
    base = ExplorationConfig(num_sequences=args.num_sequences, max_len=256)

    def configs(step: int):
        return [replace(kernel_config(base, c), seed=1729 + 7919 * dist.rank + 104729 * step + k)
                for k, c in enumerate(cases)]

    stage2 = {b: next(v for v in range(len(family(b).knobs)) if family(b).knobs[v][0] == 2) for b in KERNELS}
    s2_digest = {b: be.artifact(b, v).digest for b, v in stage2.items()}

    def fresh_of(recs):
        return [r for r in recs if r.status not in (RecordStatus.REUSED, RecordStatus.NO_IR)]

    def one_step(step, timer, host_inputs=None):
        runs0, launches0 = be.device_runs, be.kernel_launches
        with timer:
            out = explore_suite(cases, catalog, configs(step), be, host_inputs)
        fresh = {k: fresh_of(v) for k, v in out.items()}
        return out, fresh, be.device_runs - runs0, be.kernel_launches - launches0

    timer = StepTimer()
    for w in range(max(3, args.warmup)):
        one_step(-1 - w, timer)
    # steady state: every variant of the four families has had its first-use
    # warm-up (as in a long campaign), so the timed steps hold no cold runs
    for c in cases:
        be.prewarm(c)

    dist.barrier()
    n_fresh = n_records = n_runs = n_launch = 0
    s2_ms = {b: [] for b in KERNELS}
    valid = 0
    best = {}  # kernel -> (fastest valid record time ms, order)
    batch0 = be.batch_ms
    with ClockSampler(device) as clocks:
        for s in range(args.steps):
            recs, fresh, runs, launches = one_step(s, timer)
            n_fresh += sum(len(v) for v in fresh.values())
            n_records += sum(len(v) for v in recs.values())
            valid += sum(1 for v in fresh.values() for r in v if r.status is RecordStatus.VALID)
            n_runs += runs
            n_launch += launches
            for b in KERNELS:
                s2_ms[b] += [1e3 * r.wall_time for r in fresh[b] if r.artifact_digest == s2_digest[b]
                             and r.wall_time]
                top = recs[b][0]  # explore's output is sorted: fastest valid record first
                if top.status is RecordStatus.VALID and (b not in best or 1e3 * top.wall_time < best[b][0]):
                    best[b] = (1e3 * top.wall_time, top.order)
    dist.barrier()
    step_ms = timer.pairs[-args.steps:]
    local_s = sum(step_ms) / 1e3
    max_s = dist.max(local_s)
    value = dist.sum(n_fresh) / max_s
    # every collective runs on every rank, before the rank-0-only JSON line
    all_records, all_runs, all_launches = dist.sum(n_records), dist.sum(n_runs), dist.sum(n_launch)
    batch_busy = (be.batch_ms - batch0) / 1e3 / local_s

    # ---- end to end: inputs uploaded from pinned host memory every step
    e2e = None
    if args.e2e_steps > 0:
        keep = []
        host_inputs, h2d = _stock_host_inputs(be, cases, keep)
        one_step(-100, StepTimer(), host_inputs)  # warm
        et = StepTimer()
        e_fresh, d2h = 0, 0
        dist.barrier()
        # the same order streams as the first timed steps -- the same candidates, plus the host traffic --
        # with the host-side memos (order draws, compiles) cleared so the host work is the same too
        from paper_1810_10496_b200 import explorer as _explorer

        _explorer._DRAWN.clear()
        be._compile_memo.clear()
        be._variant_memo.clear()
        for s in range(args.e2e_steps):
            recs, fresh, _, _ = one_step(s, et, host_inputs)
            e_fresh += sum(len(v) for v in fresh.values())
            d2h += sum(4 * len(c.reference_outputs) * len(fresh[c.id]) for c in cases)
        dist.barrier()
        e_max = dist.max(sum(et.pairs) / 1e3)
        e2e = {"value": dist.sum(e_fresh) / e_max, "unit": "evals/s", "h2d_bytes_per_step": h2d,
               "d2h_bytes_per_step": d2h // args.e2e_steps, "steps": args.e2e_steps,
               "path": "sweep.explore_suite -> explore() x4 with B200Backend.prefetch_many(host_inputs=pinned "
                       "copies of every input array); validation outputs read back per candidate"}
        be._drain()
        for st in keep:
            st.free()

    # ---- BASELINE configs[4] sample: explore() over all 15 kernels at their config sizes
    sweep = sweep_sample(be, args.sweep_orders, dist) if args.sweep_orders > 0 else None

    # ---- per-kernel report (outside the timed region)
    report = {}
    for c in cases:
        b = c.id
        _, dims = registry.parse_descriptor(c.measurement_input)
        t_base = be.time_variant(b, dims, 0, samples=3) * 1e3  # the empty order (nvcc-shaped baseline)
        t_best, order = best[b]
        bytes_, _ = alg_work(b, dims)
        report[b] = {"baseline_ms": t_base, "best_ms": t_best,
                     "best_variant": family(b).key(be.variant_for(c, order)[1]),
                     "speedup": t_base / t_best, "best_gbs": bytes_ / (t_best * 1e-3) / 1e9,
                     "stage2_ms_in_steps": statistics.mean(s2_ms[b]) if s2_ms[b] else None}
    geo = math.exp(sum(math.log(r["speedup"]) for r in report.values()) / len(report))

    roofline = None
    rb = "GESUMMV"
    if s2_ms[rb]:
        ms = statistics.mean(s2_ms[rb])
        bytes_, _ = alg_work(rb, _dims(rb, n))
        achieved = bytes_ / (ms * 1e-3) / 1e9
        roofline = {"bound": "hbm", "achieved": achieved, "peak": peaks["hbm_gbs"], "unit": "GB/s",
                    "frac": achieved / peaks["hbm_gbs"], "traffic": args.traffic or ncu_traffic(rb, stage2[rb]),
                    "kernel": f"{rb} {family(rb).key(stage2[rb])}", "alg_bytes_per_launch": bytes_,
                    "mean_launch_ms": ms, "launches_timed": len(s2_ms[rb]),
                    "peak_source": peaks["source"] + " (burst copy, MEASURED_PEAKS.json)"}

    cpu = None
    if dist.rank == 0 and dist.world == 1 and args.cpu_orders > 0:
        cpu = cpu_baseline(n, args.cpu_orders)

    if dist.rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "evals/s", "n_gpus": dist.world, "steps": args.steps,
            "warmup": max(3, args.warmup), "ms_per_step": 1e3 * max_s / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic (PolyBench/GPU init formulas generated on device)",
            "config": {"workload": _workload(n), "n": n, "kernels": list(KERNELS),
                       "orders_per_kernel": args.num_sequences, "max_len": 256,
                       "catalog": "20 Table-1 passes + 4 staging passes (passmodel.DEFAULT_CATALOG_PASSES)",
                       "measurement": "B200Backend(samples=1): one CUDA-event-timed run per fresh candidate, "
                                      "L2 flushed before it; every variant's first-use warm-up done before "
                                      "the timed steps (B200Backend.prewarm)",
                       "l2": "inputs larger than L2 (A is 1-2 GiB per kernel) and L2 flushed (2x L2 memset + "
                             "read) before every timed run",
                       "parallelism": f"candidate streams x{dist.world} (one process per GPU, independent)"},
            "fresh_evaluations_per_step": n_fresh / args.steps,
            "candidate_records_per_s": all_records / max_s,
            "device_runs_per_s": all_runs / max_s,
            "valid_fraction": valid / max(1, n_fresh),
            "device_busy_fraction": batch_busy,
            "geomean_speedup": geo,
            "per_kernel": report,
            "roofline": roofline,
            "e2e": e2e,
            "sweep": sweep,
            "cpu_baseline": cpu,
            "gpu_launches": int(all_launches),
            "clocks": clocks.summary(),
        }
        print(json.dumps(line), flush=True)
    be.close()
    return 0


# per-kernel seconds of the B200 full sweep (profiles/r02_campaign_staging): LPT weights for sharding the
# configs[4] sample's kernels over ranks (all timed runs of a kernel stay on one device)
SWEEP_COSTS = {"2DCONV": 1, "3DCONV": 3, "2MM": 12, "3MM": 15, "ATAX": 6, "BICG": 6, "CORR": 138, "COVAR": 142,
               "FDTD-2D": 12, "GEMM": 1, "GESUMMV": 4, "GRAMSCHM": 846, "MVT": 6, "SYR2K": 28, "SYRK": 21}


def sweep_sample(be, orders: int, dist: Dist) -> dict:
    """A bounded sample of BASELINE configs[4] (the full 15-kernel sweep):
    ``explore()`` on every kernel at its config size over an ``orders``-long
    stream through the same product path (compile, digest dedup, validation
    + compare, one measurement per fresh artifact), kernels sharded over the
    ranks by LPT with device affinity.  The whole sweep with finalize /
    reduce_order / LOO (1000 orders, ~21 min on one B200) is
    tools/run_campaign.py (profiles/r02_campaign_*)."""
    from paper_1810_10496_b200 import passmodel, registry
    from paper_1810_10496_b200.campaign import kernel_config, kernel_owners
    from paper_1810_10496_b200.explorer import ExplorationConfig, RecordStatus
    from paper_1810_10496_b200.sweep import explore_suite

    kernels = [registry.kernel_case(b, "config") for b in registry.BENCHES]
    owners = kernel_owners(kernels, dist.world, SWEEP_COSTS)
    mine = registry.build_suite(be, size="config",
                                benches=[k.id for k, o in zip(kernels, owners) if o == dist.rank])
    base = ExplorationConfig(num_sequences=orders, max_len=256)
    cfgs = [replace(kernel_config(base, c), seed=4242 + i) for i, c in enumerate(mine)]
    timer = StepTimer()
    dist.barrier()
    with timer:
        out = explore_suite(mine, passmodel.default_catalog(), cfgs, be)
    dist.barrier()
    fresh = sum(1 for v in out.values() for r in v if r.status not in (RecordStatus.REUSED, RecordStatus.NO_IR))
    records = sum(len(v) for v in out.values())
    seconds = dist.max(timer.ms / 1e3)
    total_fresh = dist.sum(fresh)
    return {"workload": f"BASELINE configs[4] sample: explore() on all 15 kernels at config sizes, {orders} orders "
                        "each (default catalog, max_len 256)",
            "value": total_fresh / seconds, "unit": "evals/s", "fresh_evaluations": total_fresh,
            "records": dist.sum(records), "seconds": seconds, "scaling": "strong (kernels sharded over ranks)",
            "timing": "CUDA events around the whole explore() sample after a device synchronize, max over ranks"}


def ncu_traffic(bench: str, variant: int):
    """DRAM bytes per launch of the roofline kernel from the committed ncu
    --set full capture (profiles/r01_traffic.json), or None."""
    from paper_1810_10496_b200.backend.b200 import family

    path = ROOT / "profiles" / "r01_traffic.json"
    try:
        entry = json.loads(path.read_text()).get(f"{bench} {family(bench).key(variant)}")
    except (OSError, ValueError):
        return None
    return entry["traffic"] if entry else None


def main() -> int:
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=("b200", "reference"), default="b200")
    ap.add_argument("--n", type=int, default=16384)
    ap.add_argument("--num-sequences", type=int, default=1000)
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--cpu-orders", type=int, default=2, help="orders per kernel in the cpu_baseline sample")
    ap.add_argument("--ref-orders", type=int, default=2, help="orders per kernel per step of --impl reference")
    ap.add_argument("--sweep-orders", type=int, default=30,
                    help="orders per kernel of the configs[4] sample (explore() on all 15 kernels); 0: skip")
    ap.add_argument("--traffic", type=float, default=None,
                    help="dram bytes per launch of the roofline kernel from an ncu --set full capture")
    args = ap.parse_args()
    args.warmup = max(3, args.warmup)
    dist = Dist()
    try:
        if args.impl == "reference":
            return run_reference(args, dist)
        return run_gpu(args, dist)
    finally:
        dist.close()


if __name__ == "__main__":
    sys.exit(main())
