"""The reference's own CPU path for the bench's workload (baseline infrastructure).

Only bench.py's ``cpu_baseline`` leg and ``--impl reference`` (and tests)
use this module; the product never does.

The reference evaluates candidates through its unmodified engine
(``phaseforge.explore``, /root/reference/pkg/src/phaseforge/explorer.py:
152-214) and ``ToolchainBackend`` (backend/toolchain.py:122-307): four
compile-stage processes per candidate and one runner process per execute.
PolyBench/GPU (the kernel arithmetic) is not part of the reference, so the
runner computes the kernels with this repository's CPU oracle
(oracle/pf_cpu_runner, all host threads).  The compile stages are identity
tools that keep the phase order in the artifact (every distinct order is a
distinct artifact: there is no optimizer to make two orders' code equal).

The reference package is imported read-only from /root/reference/pkg/src
(build container) or from its pip install in baseline/_ref (GPU box).
"""

from __future__ import annotations

import math
import os
import sys
import tempfile
import time
from pathlib import Path

HERE = Path(__file__).resolve().parent
ROOT = HERE.parent
RUNNER = HERE / "pf_cpu_runner"
SOURCES = (Path("/root/reference/pkg/src"), ROOT / "baseline" / "_ref")


def reference_engine():
    """The unmodified ``phaseforge`` package, or None when it is absent."""
    for src in SOURCES:
        if (src / "phaseforge" / "__init__.py").exists():
            sys.dont_write_bytecode = True
            if str(src) not in sys.path:
                sys.path.append(str(src))
            import phaseforge  # noqa: WPS433

            return phaseforge
    return None


def build_runner() -> Path:
    if not RUNNER.exists():
        import subprocess

        subprocess.run(["make", "-s", "-C", str(HERE), "pf_cpu_runner"], check=True)
    return RUNNER


def toolchain_backend(pf, work: Path):
    """The reference ToolchainBackend over identity compile stages and the
    oracle runner (runner template ``{artifact} {data} {kind}``)."""
    build_runner()
    spec = pf.ToolchainSpec(
        frontend_cmd="cp {input} {output}",
        optimizer_cmd="sh -c 'cp \"$0\" \"$1\" && echo \"$@\" >> \"$1\"' {input} {output} {passes}",
        linker_cmd="cp {input} {output}",
        codegen_cmd="cp {input} {output}",
        runner_cmd=f"{RUNNER} {{artifact}} {{data}} {{kind}}",
        work_dir=work / "toolchain",
        exec_timeout=600.0,
    )
    return pf.ToolchainBackend(spec)


def kernel_cases(pf, benches, measurement_dims, work: Path):
    """Reference KernelCases: source = a file naming the benchmark, inputs =
    the B200 registry's descriptors, reference_outputs = the oracle's stock
    validation-input outputs."""
    from oracle import oracle as orc
    from paper_1810_10496_b200 import registry

    cases = []
    for b in benches:
        src = work / f"{b}.src"
        src.write_text(f"polybench-gpu:{b}\n")
        vdims = registry.SIZES[b]["validation"]
        ref = [float(x) for arr in orc.reference(b, vdims, True, 1729, -1) for x in arr.tolist()]
        cases.append(pf.KernelCase(b, str(src), registry.describe(b, vdims),
                                   registry.describe(b, measurement_dims[b]), tuple(ref), ""))
    return cases


def explore_step(pf, backend, cases, catalog_names, orders: int, seed: int) -> tuple[int, int, float]:
    """One exploration round of the reference engine over ``cases``:
    (fresh evaluations, records, seconds); ``explore_step.valid`` counts the
    VALID fresh records of the last call."""
    catalog = pf.PassCatalog.of(*catalog_names)
    fresh = records = valid = 0
    t0 = time.perf_counter()
    for k, case in enumerate(cases):
        scale = max((abs(x) for x in case.reference_outputs), default=1.0)
        cfg = pf.ExplorationConfig(num_sequences=orders, max_len=256, seed=seed + k, rtol=1e-4, atol=1e-4 * scale)
        recs = pf.explore(case, catalog, cfg, backend)
        records += len(recs)
        fresh += sum(1 for r in recs if r.status.value not in ("reused", "no_ir"))
        valid += sum(1 for r in recs if r.status.value == "valid")
    explore_step.valid = valid
    return fresh, records, time.perf_counter() - t0


def simulator_rate(pf, catalog_names, num_sequences: int = 1000) -> dict:
    """The reference explore() on its SimulatorBackend (engine only, no kernel
    work): evaluations/s on one core."""
    model = pf.backend.simulator.SimKernelModel(baseline_time=1e-3)
    case = pf.KernelCase("SIM", model, "v", "m", (1.0, 2.0), "")
    cfg = pf.ExplorationConfig(num_sequences=num_sequences, max_len=256, seed=1729)
    catalog = pf.PassCatalog.of(*catalog_names)
    t0 = time.perf_counter()
    recs = pf.explore(case, catalog, cfg, pf.backend.simulator.SimulatorBackend())
    dt = time.perf_counter() - t0
    fresh = sum(1 for r in recs if r.status.value not in ("reused", "no_ir"))
    return {"candidates_per_s": len(recs) / dt, "fresh_evals_per_s": fresh / dt, "candidates": len(recs),
            "cores": 1, "sample": f"phaseforge.explore on SimulatorBackend, {num_sequences} orders, max_len 256"}


def oracle_rates(benches, dims_of, threads_list=(1, 0), min_seconds: float = 2.0) -> dict:
    """Kernel-only oracle evaluations/s on the host (single thread and all
    threads), round-robin over ``benches`` at their measurement dims."""
    from oracle import oracle as orc

    out = {}
    arrays = {b: orc.generate(b, dims_of[b]) for b in benches}
    for threads in threads_list:
        used = orc.set_threads(threads)
        done, secs = 0, 0.0
        while secs < min_seconds or done < len(benches):
            for b in benches:
                work = [a.copy() if b == "MVT" and i in (1, 2) else a for i, a in enumerate(arrays[b])]
                t0 = time.perf_counter()
                orc.run(b, dims_of[b], work)
                secs += time.perf_counter() - t0
                done += 1
        out["oracle_1t" if used == 1 else "oracle_mt"] = {"evals_per_s": done / secs, "cores": used,
                                                          "evals": done, "seconds": secs}
    orc.set_threads(0)
    return out


def cores() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


def cpu_model() -> str:
    try:
        for line in Path("/proc/cpuinfo").read_text().splitlines():
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def workdir() -> Path:
    return Path(tempfile.mkdtemp(prefix="pf-ref-arm-"))


def geomean(xs) -> float:
    xs = [x for x in xs if x > 0]
    return math.exp(sum(math.log(x) for x in xs) / len(xs)) if xs else float("nan")


__all__ = ["cores", "cpu_model", "explore_step", "kernel_cases", "oracle_rates", "reference_engine",
           "simulator_rate", "toolchain_backend", "workdir"]
