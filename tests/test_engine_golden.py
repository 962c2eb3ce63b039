"""Exact parity of the restated engine with golden outputs of the reference.

tests/golden/engine.json is produced by tools/make_golden.py from the
unmodified reference package (order streams, permutations, features, cosine
distances, kNN rankings, explore/finalize/reduce runs on the reference
simulator with every backend answer recorded, leave-one-out, reports).  The
engine runs here are driven by a replay backend answering from that table,
so record streams must match bit for bit.  Runs without /root/reference.
"""

from __future__ import annotations

import json
from pathlib import Path
from random import Random

import pytest

from paper_1810_10496_b200 import advisor, catalog, explorer, irfeat, passmodel, registry, results
from paper_1810_10496_b200.backend.types import (
    Artifact, Backend, CompileOutcome, CompileStatus, ExecutionOutcome, ExecutionStatus, KernelCase,
)

G = json.loads((Path(__file__).parent / "golden" / "engine.json").read_text())


class ReplayBackend(Backend):
    """Answers compile/execute from the recorded reference-simulator table."""

    def __init__(self, table):
        super().__init__()
        self.table = table
        self.misses = []

    def compile(self, kernel, order):
        key = f"C|{kernel.id}|{catalog.render_phase_order(order)}"
        rec = self.table.get(key)
        if rec is None:
            self.misses.append(key)
            raise KeyError(key)
        st = CompileStatus(rec["status"])
        art = Artifact(b"", rec["digest"]) if rec["digest"] else None
        return CompileOutcome(st, art, rec["log"])

    def execute(self, kernel, order, artifact, input_kind, random_input_index=None):
        key = f"E|{kernel.id}|{catalog.render_phase_order(order)}|{input_kind.value}|{random_input_index}"
        rec = self.table.get(key)
        if rec is None:
            self.misses.append(key)
            raise KeyError(key)
        outs = tuple(rec["outputs"]) if rec["outputs"] is not None else None
        return ExecutionOutcome(ExecutionStatus(rec["status"]), rec["wall_time"], outs, rec["log"])


def _catalog(name):
    if name == "table1":
        return catalog.PassCatalog.of(*passmodel.TABLE1_PASSES)
    if name == "default":
        return passmodel.default_catalog()
    return catalog.PassCatalog.of(*G["demo_catalog"])


def test_order_streams_bit_identical():
    for key, expected in G["streams"].items():
        name, seed, max_len = key.split("|")
        rng = Random(int(seed))
        cat = _catalog(name)
        got = [catalog.render_phase_order(catalog.random_phase_order(cat, int(max_len), rng)) for _ in expected]
        assert got == expected, key


def test_permutations_identical():
    for key, expected in G["permutations"].items():
        text, count, seed = key.split("|")
        got = catalog.random_permutations(catalog.parse_phase_order(text), int(count), Random(int(seed)))
        assert [catalog.render_phase_order(p) for p in got] == expected


def test_features_identical():
    for b, text in registry.IR_TEXTS.items():
        assert list(irfeat.extract_features(irfeat.parse_ir(text)).values) == G["features"][f"registry:{b}"]
    for key, item in G["random_ir"].items():
        try:
            got = list(irfeat.extract_features(irfeat.parse_ir(item["text"])).values)
        except ValueError as exc:
            got = f"error: {exc}"
        assert got == item["features"], key


def test_cosine_and_knn_identical():
    names = sorted(registry.IR_TEXTS)
    vecs = {b: irfeat.FeatureVector(tuple(G["features"][f"registry:{b}"])) for b in names}
    for key, d in G["cosine"].items():
        a, b = key.split("|")
        assert irfeat.cosine_distance(vecs[a], vecs[b]) == d
    orders = {b: catalog.parse_phase_order(t) for b, t in G["knn_orders"].items()}
    refset = advisor.ReferenceSet(tuple(advisor.ReferenceEntry(b, vecs[b], orders[b]) for b in names))
    for key, expected in G["knn"].items():
        q, k = key.split("|")
        got = advisor.suggest_knn(vecs[q], refset.without(q), int(k))
        assert [[kid, catalog.render_phase_order(o)] for kid, o in got] == expected, key


def _kernels():
    return [KernelCase(k["id"], "replay", k["validation_input"], k["measurement_input"],
                       tuple(k["reference_outputs"]), k["ir"]) for k in G["demo_kernels"]]


def test_explore_finalize_reduce_replay_identical():
    be = ReplayBackend(G["replay"])
    kernels = {k.id: k for k in _kernels()}
    cat = _catalog("demo")
    for run in G["runs"]:
        cfg = explorer.ExplorationConfig(**run["config"])
        kernel = kernels[run["kernel"]]
        records = explorer.explore(kernel, cat, cfg, be)
        got = [[r.kernel_id, catalog.render_phase_order(r.order), r.artifact_digest, r.status.value, r.wall_time,
                r.eval_index] for r in records]
        assert got == run["records"], (run["kernel"], run["config"])
        if "best" in run["finalize"]:
            best, t = explorer.finalize(kernel, records, cfg, be)
            assert catalog.render_phase_order(best) == run["finalize"]["best"]
            assert t == run["finalize"]["best_time"]
            red = explorer.reduce_order(kernel, best, be, 0.01, cfg)
            assert catalog.render_phase_order(red) == run["finalize"]["reduced"]
        else:
            with pytest.raises(explorer.NoValidCandidateError):
                explorer.finalize(kernel, records, cfg, be)
    assert not be.misses


def test_leave_one_out_and_reports_identical():
    be = ReplayBackend(G["replay"])
    loaded = explorer.KnowledgeBase.from_json_dict(G["kb"])
    kb = explorer.KnowledgeBase({k: loaded.entries[k] for k in G["kb_order"]})  # insertion order feeds rng.sample
    refset = advisor.ReferenceSet.from_knowledge_base(kb)
    table = advisor.leave_one_out(refset, _kernels(), be, k_max=2, trials=50, seed=3,
                                  config=explorer.ExplorationConfig(final_reps=2, final_random_inputs=2))
    assert table == G["loo"]
    rep = results.build_speedup_report(kb)
    assert rep.geomean == G["speedup_report"]["geomean"]
    assert {k: [v.baseline_time, v.best_time, v.speedup] for k, v in rep.per_kernel.items()} == \
        G["speedup_report"]["per_kernel"]
    assert results.geometric_mean(G["geomean"]["values"]) == G["geomean"]["geomean"]


def test_compare_outputs_identical():
    for ref, cand, rtol, atol, expected in G["compare_outputs"]:
        assert explorer.compare_outputs(ref, cand, rtol, atol) is expected
