#!/usr/bin/env python3
"""Generate tests/golden/engine.json from the unmodified reference package.

Imports ``phaseforge`` read-only from /root/reference/pkg/src (this container
only) and records:

* order streams of ``random_phase_order`` for several seeds/catalogs/lengths
  (catalog.py:138-145) and ``random_permutations`` outputs (catalog.py:172-192);
* feature vectors (irfeat.py:243-303) of the 15 registry IR texts, of the
  reference tests' fixed IR texts, and of seeded random modules;
* cosine distances (irfeat.py:306-318) and kNN suggestions (advisor.py:66-90);
* full explore -> finalize -> reduce_order runs (explorer.py:152-365) of the
  reference demo suite on the reference SimulatorBackend, together with every
  (compile | execute) answer the backend gave -- a replay table that lets the
  restated engine be driven by exactly the same backend behaviour without the
  reference installed;
* leave_one_out (advisor.py:273-353) and geometric_mean / speedup reports.

The script is committed so the fixture can be regenerated; the fixture is
what tests/test_engine_golden.py consumes.
"""

from __future__ import annotations

import json
import sys
from pathlib import Path
from random import Random

ROOT = Path(__file__).resolve().parent.parent
REF = Path("/root/reference/pkg/src")
sys.dont_write_bytecode = True
sys.path.insert(0, str(ROOT))
sys.path.append(str(REF))

import phaseforge as pf  # noqa: E402
from phaseforge.backend import simulator as sim  # noqa: E402
from phaseforge.backend.types import Backend  # noqa: E402

from paper_1810_10496_b200 import passmodel, registry  # noqa: E402

OUT = ROOT / "tests" / "golden" / "engine.json"
DEMO = Path("/root/reference/pkg/demo")


def render(o) -> str:
    return pf.render_phase_order(o)


class Recorder(Backend):
    """Proxy that records every answer of the wrapped reference backend."""

    def __init__(self, inner):
        super().__init__()
        self.inner = inner
        self.table: dict[str, dict] = {}

    def compile(self, kernel, order):
        out = self.inner.compile(kernel, order)
        key = f"C|{kernel.id}|{render(order)}"
        self.table[key] = {"status": out.status.value, "digest": out.artifact.digest if out.artifact else None,
                           "log": out.log}
        return out

    def execute(self, kernel, order, artifact, input_kind, random_input_index=None):
        out = self.inner.execute(kernel, order, artifact, input_kind, random_input_index)
        key = f"E|{kernel.id}|{render(order)}|{input_kind.value}|{random_input_index}"
        self.table[key] = {"status": out.status.value, "wall_time": out.wall_time,
                           "outputs": list(out.outputs) if out.outputs is not None else None, "log": out.log}
        return out


def random_ir(rng: Random) -> str:
    """Seeded random (valid) IR-subset module."""
    lines = []
    for f in range(rng.randint(1, 3)):
        nblocks = rng.randint(1, 6)
        labels = [f"b{i}" for i in range(nblocks)]
        lines.append(f"func f{f} {{")
        for i, lab in enumerate(labels):
            lines.append(f"{lab}:")
            for _ in range(rng.randint(0, 2)):
                lines.append(f"  phi {rng.randint(1, 4)}")
            for _ in range(rng.randint(0, 6)):
                lines.append("  " + rng.choice(["load", "store", "iadd", "fadd", "cmp", "call", "addr", "other"]))
            kind = rng.choice(["br", "condbr", "switch", "ret"])
            if kind == "br":
                lines.append(f"  br {rng.choice(labels)}")
            elif kind == "condbr":
                lines.append(f"  condbr {rng.choice(labels)} {rng.choice(labels)}")
            elif kind == "switch":
                lines.append("  switch " + " ".join(rng.choice(labels) for _ in range(rng.randint(1, 4))))
            else:
                lines.append("  ret")
        lines.append("}")
    return "\n".join(lines) + "\n"


def main() -> int:
    g: dict = {"generator": "tools/make_golden.py", "reference": "/root/reference/pkg/src/phaseforge"}

    # ---- order streams
    table1 = pf.PassCatalog.of(*passmodel.TABLE1_PASSES)
    full = passmodel.default_catalog()
    demo_cat = pf.PassCatalog.load(DEMO / "catalog.txt")
    ref_full = pf.PassCatalog.of(*[p.name for p in full.passes])
    streams = {}
    for name, cat in (("table1", table1), ("default", ref_full), ("demo", demo_cat)):
        for seed in (1729, 1, 424242):
            for max_len in (256, 16, 1):
                rng = Random(seed)
                streams[f"{name}|{seed}|{max_len}"] = [render(pf.random_phase_order(cat, max_len, rng)) for _ in range(200)]
    g["streams"] = streams
    g["demo_catalog"] = [p.name for p in demo_cat.passes]
    perms = {}
    for text, count, seed in (("-a -b -c", 10, 1), ("-licm -gvn -licm -sroa", 5, 7), ("-x -y -z -w -v -u", 50, 3)):
        perms[f"{text}|{count}|{seed}"] = [render(p) for p in pf.random_permutations(pf.parse_phase_order(text), count,
                                                                                        Random(seed))]
    g["permutations"] = perms

    # ---- features / distances / kNN
    feats = {f"registry:{b}": list(pf.extract_features(pf.parse_ir(t)).values) for b, t in registry.IR_TEXTS.items()}
    rng = Random(99)
    randoms = {}
    for i in range(60):
        text = random_ir(rng)
        try:
            fv = list(pf.extract_features(pf.parse_ir(text)).values)
        except ValueError as exc:
            fv = f"error: {exc}"
        randoms[str(i)] = {"text": text, "features": fv}
    g["features"] = feats
    g["random_ir"] = randoms
    names = sorted(registry.IR_TEXTS)
    vecs = {b: pf.FeatureVector(tuple(feats[f"registry:{b}"])) for b in names}
    g["cosine"] = {f"{a}|{b}": pf.cosine_distance(vecs[a], vecs[b]) for a in names for b in names}
    orders = {b: pf.parse_phase_order(f"-licm -gvn{' -sroa' * (i % 3)} -dse{' -instcombine' * (i % 2)}")
              for i, b in enumerate(names)}
    refset = pf.ReferenceSet(tuple(pf.ReferenceEntry(b, vecs[b], orders[b]) for b in names))
    knn = {}
    for q in names:
        sub = refset.without(q)
        for k in (1, 3, 5, 14):
            knn[f"{q}|{k}"] = [[kid, render(o)] for kid, o in pf.suggest_knn(vecs[q], sub, k)]
    g["knn_orders"] = {b: render(o) for b, o in orders.items()}
    g["knn"] = knn

    # ---- engine runs on the demo suite (simulator) with a replay table
    suite = json.loads((DEMO / "suite.json").read_text())
    kernels = []
    for raw in suite["kernels"]:
        kernels.append(pf.KernelCase(id=raw["id"], source=sim.SimKernelModel.from_json_dict(raw["model"]),
                                     validation_input=raw["validation_input"],
                                     measurement_input=raw["measurement_input"],
                                     reference_outputs=tuple(raw["reference_outputs"]), ir_text=raw["ir"]))
    g["demo_kernels"] = [{"id": k.id, "validation_input": k.validation_input, "measurement_input": k.measurement_input,
                          "reference_outputs": list(k.reference_outputs), "ir": k.ir_text} for k in kernels]
    runs = []
    rec = Recorder(sim.SimulatorBackend())
    for cfg in ({"num_sequences": 300, "max_len": 16, "seed": 1729, "top_k": 5, "final_reps": 7,
                 "final_random_inputs": 6},
                {"num_sequences": 120, "max_len": 64, "seed": 7, "top_k": 3, "final_reps": 3,
                 "final_random_inputs": 4, "rtol": 0.05}):
        config = pf.ExplorationConfig(**cfg)
        for kernel in kernels:
            records = pf.explore(kernel, demo_cat, config, rec)
            try:
                best, best_time = pf.finalize(kernel, records, config, rec)
                reduced = pf.reduce_order(kernel, best, rec, 0.01, config)
                fin = {"best": render(best), "best_time": best_time, "reduced": render(reduced)}
            except pf.NoValidCandidateError as exc:
                fin = {"error": str(exc)}
            runs.append({
                "config": cfg, "kernel": kernel.id,
                "records": [[r.kernel_id, render(r.order), r.artifact_digest, r.status.value, r.wall_time,
                             r.eval_index] for r in records],
                "finalize": fin,
            })
    g["runs"] = runs

    # ---- leave-one-out over a KB built from the runs
    kb = pf.KnowledgeBase()
    for kernel in kernels:
        best = next(r for r in runs if r["kernel"] == kernel.id and "best" in r["finalize"])
        fv = pf.extract_features(pf.parse_ir(kernel.ir_text))
        t = best["finalize"]["best_time"]
        kb.add(kernel.id, pf.KbEntry(pf.parse_phase_order(best["finalize"]["reduced"]), t, max(t, 1.0), fv))
    loo_ref = pf.ReferenceSet.from_knowledge_base(kb)
    g["kb"] = kb.to_json_dict()
    g["kb_order"] = list(kb.entries)
    g["loo"] = pf.leave_one_out(loo_ref, kernels, rec, k_max=2, trials=50, seed=3,
                                config=pf.ExplorationConfig(final_reps=2, final_random_inputs=2))
    g["replay"] = rec.table

    # ---- results
    camp = [1.0, 1.05, 1.63, 1.82, 1.47, 1.48, 5.36, 5.7, 1.0, 1.73, 1.02, 1.52, 1.44, 2.05, 1.14]
    g["geomean"] = {"values": camp, "geomean": pf.geometric_mean(camp)}
    rep = pf.build_speedup_report(kb)
    g["speedup_report"] = {"geomean": rep.geomean,
                           "per_kernel": {k: [v.baseline_time, v.best_time, v.speedup] for k, v in rep.per_kernel.items()}}
    cmp_cases = []
    crng = Random(5)
    for _ in range(300):
        n = crng.randint(0, 4)
        ref = [crng.choice([0.0, 1.0, -2.5, 1e-7, 3.0]) for _ in range(n)]
        cand = [r + crng.choice([0.0, 1e-7, 0.01, -0.02, 1.0]) for r in ref]
        if crng.random() < 0.1:
            cand = cand[:-1]
        rtol, atol = crng.choice([0.0, 0.01, 0.1]), crng.choice([0.0, 1e-6, 0.05])
        cmp_cases.append([ref, cand, rtol, atol, pf.compare_outputs(ref, cand, rtol, atol)])
    g["compare_outputs"] = cmp_cases

    OUT.parent.mkdir(parents=True, exist_ok=True)
    OUT.write_text(json.dumps(g, sort_keys=True, separators=(",", ":")) + "\n")
    print(f"wrote {OUT} ({OUT.stat().st_size} bytes, {len(rec.table)} replay entries)")
    return 0


if __name__ == "__main__":
    sys.exit(main())
