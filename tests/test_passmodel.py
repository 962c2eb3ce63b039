"""The pass-semantics interpreter (passmodel.py) and variant selection."""

from __future__ import annotations

from random import Random

import pytest

from paper_1810_10496_b200 import passmodel
from paper_1810_10496_b200.catalog import PhaseOrder, parse_phase_order, random_permutations, random_phase_order

TABLE1 = {
    "2MM": "-cfl-anders-aa -dse -loop-reduce -licm -instcombine",
    "3MM": "-loop-reduce -gvn-hoist -reg2mem -cfl-anders-aa -sroa -licm",
    "ATAX": "-bb-vectorize -loop-reduce -licm -cfl-anders-aa",
    "BICG": "-gvn -loop-reduce -cfl-anders-aa -licm -loop-reduce",
    "CORR": "-cfl-anders-aa -loop-reduce -gvn -sink -loop-extract-single -loop-unswitch -loop-unswitch -ipsccp "
            "-reg2mem -licm -nvptx-lower-alloca",
    "COVAR": "-cfl-anders-aa -loop-unswitch -reassociate -jump-threading -loop-reduce -gvn -loop-unswitch "
             "-reassociate -sink -loop-unswitch -loop-reduce -jump-threading -reg2mem -licm -nvptx-lower-alloca",
    "GEMM": "-cfl-anders-aa -print-memdeps -loop-reduce -licm",
    "GESUMMV": "-instcombine -reg2mem -mem2reg",
    "GRAMSCHM": "-sink -reg2mem -licm -cfl-anders-aa -sroa",
    "MVT": "-gvn -loop-reduce -cfl-anders-aa -licm",
    "SYR2K": "-loop-reduce -loop-unroll -instcombine -loop-reduce -licm -cfl-anders-aa",
    "SYRK": "-licm -cfl-anders-aa -reg2mem -licm -sroa",
}


def test_empty_order_is_baseline():
    assert passmodel.interpret(PhaseOrder()) == passmodel.BASELINE_STATE


@pytest.mark.parametrize("bench,text", sorted(TABLE1.items()))
def test_table1_orders_promote_except_gesummv(bench, text):
    st = passmodel.interpret(parse_phase_order(text))
    if bench == "GESUMMV":
        assert st.store == passmodel.STORE_RMW  # no licm in its order
    else:
        assert st.store in (passmodel.STORE_REG, passmodel.STORE_DEPOT)
    if bench in ("CORR", "COVAR"):
        assert st.store == passmodel.STORE_DEPOT  # reg2mem without mem2reg: __local_depot
    assert st.stage == 0


def test_order_sensitivity_permutations_change_variants():
    # Fig. 5: a large share of permutations of a best order lose its effect
    order = parse_phase_order("-cfl-anders-aa -licm -loop-unroll -slp-vectorizer -reg2mem -sroa -loop-interchange"
                              " -loop-data-prefetch")
    base = passmodel.interpret(order)
    perms = random_permutations(order, 200, Random(1))
    states = {passmodel.interpret(p) for p in perms}
    assert len(states) > 4
    assert sum(passmodel.interpret(p) != base for p in perms) > len(perms) // 3


def test_positional_rules():
    i = lambda t: passmodel.interpret(parse_phase_order(t))
    assert i("-licm -cfl-anders-aa").store == passmodel.STORE_REG        # AA is position independent
    assert i("-cfl-anders-aa -licm -reg2mem").store == passmodel.STORE_DEPOT
    assert i("-cfl-anders-aa -licm -reg2mem -mem2reg").store == passmodel.STORE_REG
    assert i("-cfl-anders-aa -reg2mem -sroa -licm").store == passmodel.STORE_REG
    assert i("-gvn").unroll == 2 and i("-loop-unroll -loop-unroll").unroll == 8
    assert i("-loop-unroll " * 5).unroll == 16
    assert i("-slp-vectorizer -loop-unroll").vec == 0 and i("-loop-unroll -slp-vectorizer").vec == 1
    assert i("-cfl-anders-aa -licm -loop-interchange").stage == 1
    assert i("-cfl-anders-aa -licm -loop-data-prefetch -loop-interchange").stage == 1
    assert i("-cfl-anders-aa -licm -loop-interchange -loop-data-prefetch").stage == 2
    assert i("-licm -loop-interchange -loop-data-prefetch").stage == 0  # no alias analysis
    assert i("-loop-reduce").lsr == 1


def test_family_selection_complete_and_unique():
    # a synthetic family shaped like make_variants<2, 4, 2, 1>
    knobs = [(0, 0, 0, 0, 0)]
    knobs += [(0, s, u, l, v) for s in range(3) for u in (2, 4, 8, 16) for l in range(2) for v in range(2)]
    knobs += [(1, 1, u, 0, v) for u in (2, 4, 8, 16) for v in range(2)]
    knobs += [(2, 1, 1, 0, 0)]
    fam = passmodel.VariantFamily("X", knobs)
    rng = Random(5)
    cat = passmodel.default_catalog()
    hit = set()
    for _ in range(3000):
        st = passmodel.interpret(random_phase_order(cat, rng.choice([4, 16, 64, 256]), rng))
        v = fam.select(st)
        k = knobs[v]
        assert k[0] == st.stage
        for idx in fam.relevant(k[0]):
            assert k[idx] == st.as_tuple()[idx]
        hit.add(v)
    assert fam.select(passmodel.BASELINE_STATE) == 0
    assert len(hit) > 40


def test_default_catalog_has_table1_and_staging_passes():
    names = [p.name for p in passmodel.default_catalog()]
    assert len(names) == len(set(names)) == 24
    assert set(passmodel.TABLE1_PASSES) <= set(names)
