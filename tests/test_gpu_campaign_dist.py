"""The sharded campaign on a GPU: world size 2 (gloo control plane), both
ranks on cuda:0.  Kernels are owned by ranks (device affinity: every timed
run of a kernel in its owner's process), results are gathered, and both
ranks end with the same KB / records / report / LOO table -- the same kernel
set and flow as the single-process campaign."""

from __future__ import annotations

import os
import socket

import pytest
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

BENCHES = ["GEMM", "ATAX", "2DCONV"]


def _cfg():
    from paper_1810_10496_b200 import explorer

    return explorer.ExplorationConfig(num_sequences=40, max_len=16, top_k=3, final_reps=3, final_random_inputs=2)


def _summary(res):
    return (res.kb.to_json_dict(), [(r.kernel_id, r.order.text, r.artifact_digest, r.status.value, r.wall_time,
                                     r.eval_index) for r in res.store.records], res.report.geomean, res.loo,
            {k: v.get("variant") for k, v in res.per_kernel.items()})


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world),
                      LOCAL_RANK="0")
    from paper_1810_10496_b200 import campaign, registry
    from paper_1810_10496_b200.backend.b200 import B200Backend
    from paper_1810_10496_b200.dist import Dist

    d = Dist(backend="gloo")
    try:
        be = B200Backend(device=0, samples=3)
        kernels = registry.build_suite(be, size="polybench", benches=BENCHES)
        ran = []
        res = campaign.run_campaign(kernels, be, _cfg(), loo_k=2, loo_trials=5, log=lambda m: ran.append(m[:9].strip()),
                                    dist=d, kernel_costs={"GEMM": 3.0, "ATAX": 2.0, "2DCONV": 1.0})
        q.put((rank, _summary(res), ran))
        be.close()
    finally:
        d.close()


@pytest.mark.timeout(900)
def test_sharded_campaign_on_gpu():
    from paper_1810_10496_b200 import campaign, registry
    from paper_1810_10496_b200.backend.b200 import B200Backend

    be = B200Backend(device=0, samples=3)
    kernels = registry.build_suite(be, size="polybench", benches=BENCHES)
    serial = _summary(campaign.run_campaign(kernels, be, _cfg(), loo_k=2, loo_trials=5, log=lambda *a: None))
    be.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = {}
    for _ in procs:
        rank, summ, ran = q.get(timeout=850)
        got[rank] = (summ, ran)
    for p in procs:
        p.join(timeout=60)
    assert got[0][0] == got[1][0]  # every rank holds the same gathered result
    owners = campaign.kernel_owners(kernels, 2, {"GEMM": 3.0, "ATAX": 2.0, "2DCONV": 1.0})
    for rank in (0, 1):  # each rank ran exactly the flows of the kernels it owns
        mine = [k.id for k, o in zip(kernels, owners) if o == rank]
        assert [m for m in got[rank][1] if m in BENCHES] == mine
    kb, records, geo, loo, variants = got[0][0]
    assert set(kb["entries"]) == set(serial[0]["entries"]) == set(BENCHES)
    assert {r[0] for r in records} == set(BENCHES) and len(records) == len(serial[1])
    assert geo > 1.0 and set(loo) == set(serial[3])
    assert variants["GEMM"] == serial[4]["GEMM"]  # the tcgen05 variant wins on either layout
