#!/usr/bin/env python3
"""Benchmark: candidate-evaluation throughput on the memory-bound BLAS-2 set.

Workload (BASELINE.json configs[1]): ATAX, BICG, MVT and GESUMMV at
N = 16384, fp32.  One *step* is one exploration round of the hot path: every
fresh candidate that ``explore`` would evaluate on a 1000-order seeded stream
(the distinct artifacts, plus the baseline) gets one device-timed
measurement run through the C-ABI (``pf_eval_batch``).  ``value`` is the
whole-job evaluations/s (sum over ranks / max step time over ranks).

Each rank drives one GPU (one process per GPU, torchrun) with its own
candidate stream (seed 1729 + 7919*rank): weak scaling, no data-path
collective; torch.distributed is used only for the barrier and
the max-over-ranks timing reduction.

Extra keys: ``roofline`` (dominant specialized kernel, HBM bytes vs the
measured peak), ``e2e`` (same metric with the inputs uploaded from pinned
host memory and outputs read back inside the timed region),
``cpu_baseline`` (the C oracle on the host cores, bounded sample),
``geomean_speedup`` (best candidate vs baseline variant per kernel),
``clocks`` (nvidia-smi sampled during the timed region), ``gpu_launches``.

``--impl reference`` times the reference-side CPU implementation of the same
workload (the oracle port: PolyBench/GPU is not in /root/reference, and the
reference package itself is pure Python with no kernel code) on all host
threads and prints its own line.
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


# ---------------------------------------------------------------- CPU side
def cpu_eval_rate(n: int, evals_target: int, threads: int = 0) -> dict:
    """The C oracle on the host: evaluations/s over the 4 kernels at size n."""
    from oracle import oracle as orc

    used = orc.set_threads(threads)
    arrays = {b: orc.generate(b, _dims(b, n)) for b in KERNELS}
    done, secs = 0, 0.0
    while done < evals_target:
        for b in KERNELS:
            work = [a.copy() if i in (1, 2) and b == "MVT" else a for i, a in enumerate(arrays[b])]
            t0 = time.perf_counter()
            orc.run(b, _dims(b, n), work)
            secs += time.perf_counter() - t0
            done += 1
    return {"value": done / secs, "unit": "evals/s", "cores": used, "kind": "port", "seconds": secs, "evals": done,
            "sample": f"{done} oracle evaluations ({'/'.join(KERNELS)} round-robin) at N={n}, fp64 accumulation, "
                      f"{used} pthreads"}


def run_reference(args, dist: Dist) -> int:
    if dist.rank != 0:
        return 0
    from oracle import oracle as orc

    threads = orc.set_threads(0)
    n = args.n
    arrays = {b: orc.generate(b, _dims(b, n)) for b in KERNELS}

    def step() -> tuple[int, float]:
        t = 0.0
        for b in KERNELS:
            work = [a.copy() if b == "MVT" and i in (1, 2) else a for i, a in enumerate(arrays[b])]
            t0 = time.perf_counter()
            orc.run(b, _dims(b, n), work)
            t += time.perf_counter() - t0
        return len(KERNELS), t

    for _ in range(args.warmup):
        step()
    evals, secs = 0, 0.0
    for _ in range(args.steps):
        e, t = step()
        evals += e
        secs += t
    value = evals / secs
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "evals/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * secs / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic (PolyBench/GPU init formulas)",
        "config": {"workload": "BLAS-2 set ATAX/BICG/MVT/GESUMMV, N=%d fp32 (BASELINE configs[1])" % n,
                   "n": n, "kernels": list(KERNELS)},
        "cpu_baseline": {"value": value, "unit": "evals/s", "cores": threads, "kind": "port",
                         "sample": f"{args.steps} steps x {len(KERNELS)} oracle evaluations at N={n}"},
        "e2e": {"value": value, "unit": "evals/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------- GPU side
def run_gpu(args, dist: Dist) -> int:
    import numpy as np

    from paper_1810_10496_b200 import _abi
    from paper_1810_10496_b200.backend.b200 import B200Backend, alg_work, family
    from paper_1810_10496_b200.sweep import candidate_set, evaluate_round, launches_of

    peaks = _peaks()
    device = dist.local
    be = B200Backend(device=device, samples=1)
    n = args.n
    seed = 1729 + 7919 * dist.rank
    items = []           # (ws, variant) in evaluation order
    per_kernel = {}
    for k, b in enumerate(KERNELS):
        ws = be.workspace(b, _dims(b, n), True, -1)
        cands = candidate_set(be, b, num_sequences=args.num_sequences, max_len=256, seed=seed + k)
        per_kernel[b] = {"ws": ws, "cands": cands}
        items += [(ws, c.variant) for c in cands]

    for _ in range(max(3, args.warmup)):
        evaluate_round(items, flush_l2=True)

    dist.barrier()
    t_steps = []
    ms_acc = [0.0] * len(items)
    with ClockSampler(device) as clocks:
        for _ in range(args.steps):
            ms_each, ms_total = evaluate_round(items, flush_l2=True)
            t_steps.append(ms_total)
            for i, m in enumerate(ms_each):
                ms_acc[i] += m
    dist.barrier()
    local_s = sum(t_steps) / 1e3
    max_s = dist.max(local_s)
    total_evals = dist.sum(len(items) * args.steps)
    value = total_evals / max_s

    # ---- per-kernel analysis (device event times of this rank)
    mean_ms = [m / args.steps for m in ms_acc]
    report = {}
    best_stage2 = None
    for b in KERNELS:
        ws = per_kernel[b]["ws"]
        idx = [i for i, (w, _) in enumerate(items) if w is ws]
        fam = family(b)
        base_i = idx[0]
        best_i = min(idx, key=lambda i: mean_ms[i])
        bytes_, _ = alg_work(b, ws.dims)
        report[b] = {
            "candidates": len(idx),
            "baseline_ms": mean_ms[base_i],
            "best_ms": mean_ms[best_i],
            "best_variant": fam.key(items[best_i][1]),
            "speedup": mean_ms[base_i] / mean_ms[best_i],
            "best_gbs": bytes_ / (mean_ms[best_i] * 1e-3) / 1e9,
            "time_share": sum(mean_ms[i] for i in idx) / sum(mean_ms),
        }
        for i in idx:
            if fam.knobs[items[i][1]][0] == 2:
                tot = mean_ms[i]
                if best_stage2 is None or tot > best_stage2[1]:
                    best_stage2 = (b, tot, i)
    geo = math.exp(sum(math.log(r["speedup"]) for r in report.values()) / len(report))

    roofline = None
    if best_stage2:
        b, ms, i = best_stage2
        ws = items[i][0]
        bytes_, _ = alg_work(b, ws.dims)
        achieved = bytes_ / (ms * 1e-3) / 1e9
        roofline = {"bound": "hbm", "achieved": achieved, "peak": peaks["hbm_gbs"], "unit": "GB/s",
                    "frac": achieved / peaks["hbm_gbs"], "traffic": args.traffic or ncu_traffic(b, items[i][1]),
                    "kernel": f"{b} {family(b).key(items[i][1])}",
                    "alg_bytes_per_launch": bytes_, "mean_launch_ms": ms,
                    "peak_source": peaks["source"] + " (burst copy, MEASURED_PEAKS.json)"}

    # ---- end to end: inputs from pinned host memory, outputs read back
    e2e = None
    if args.e2e_steps > 0:
        lib = _abi.lib()
        host_in, host_out, pinned = {}, {}, []
        h2d = d2h = 0
        for b in KERNELS:
            ws = per_kernel[b]["ws"]
            hin, hout = {}, {}
            for a, (_, role, is_out) in enumerate(ws.arrays):
                nbytes = ws.elems[a] * 4
                if role != _abi.ROLE_OUT:
                    p = ctypes_alloc(lib, nbytes, pinned)
                    src = ws.download(a)
                    ctypes_copy(p, src)
                    hin[a] = p
                    h2d += nbytes
                if is_out:
                    hout[a] = ctypes_alloc(lib, nbytes, pinned)
                    d2h += nbytes * len(per_kernel[b]["cands"])
            host_in[ws], host_out[ws] = hin, hout
        evaluate_round(items, flush_l2=True, host_in=host_in, host_out=host_out)  # warm
        dist.barrier()
        e2e_ms = []
        for _ in range(args.e2e_steps):
            _, tot = evaluate_round(items, flush_l2=True, host_in=host_in, host_out=host_out)
            e2e_ms.append(tot)
        dist.barrier()
        e2e_max = dist.max(sum(e2e_ms) / 1e3)
        e2e_val = dist.sum(len(items) * args.e2e_steps) / e2e_max
        e2e = {"value": e2e_val, "unit": "evals/s", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
               "steps": args.e2e_steps, "path": "pf_eval_batch with pinned host_in/host_out (C-ABI)"}
        for p in pinned:
            lib.pf_host_free(p)

    cpu = None
    if dist.rank == 0 and dist.world == 1 and args.cpu_evals > 0:
        cpu = cpu_eval_rate(n, args.cpu_evals)

    launches = launches_of(items) * args.steps
    if dist.rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "evals/s", "n_gpus": dist.world, "steps": args.steps,
            "warmup": max(3, args.warmup), "ms_per_step": 1e3 * max_s / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic (PolyBench/GPU init formulas generated on device)",
            "config": {"workload": f"BLAS-2 set ATAX/BICG/MVT/GESUMMV, N={n} fp32 (BASELINE configs[1])",
                       "n": n, "kernels": list(KERNELS), "orders_per_kernel": args.num_sequences,
                       "evals_per_step_per_gpu": len(items),
                       "l2": "inputs larger than L2 (A is 1-2 GiB per kernel) and L2 flushed (2x L2 memset) "
                             "before every candidate",
                       "parallelism": f"candidate sharding x{dist.world} (independent streams)"},
            "geomean_speedup": geo,
            "per_kernel": report,
            "roofline": roofline,
            "e2e": e2e,
            "cpu_baseline": cpu,
            "gpu_launches": launches,
            "clocks": clocks.summary(),
        }
        print(json.dumps(line), flush=True)
    be.close()
    return 0


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


def ctypes_alloc(lib, nbytes: int, keep: list):
    import ctypes

    p = ctypes.c_void_p()
    from paper_1810_10496_b200 import _abi

    _abi.check(lib.pf_host_alloc(nbytes, ctypes.byref(p)))
    keep.append(p)
    return p.value


def ctypes_copy(ptr: int, src) -> None:
    import ctypes

    ctypes.memmove(ptr, src.ctypes.data, src.nbytes)


def main() -> int:
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=("b200", "reference"), default="b200")
    ap.add_argument("--n", type=int, default=16384)
    ap.add_argument("--num-sequences", type=int, default=1000)
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--cpu-evals", type=int, default=8)
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
