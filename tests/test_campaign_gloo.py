"""The rank-parallel campaign on world_size 2 (gloo,
CPU): kernels are sharded over the ranks with device affinity (every timed
run of a kernel on its owner's device: explore, finalize, reduce_order and
its LOO curves); with a deterministic backend the result is exactly the
single-process one -- the same KB, records, report and LOO curves on both
ranks."""

from __future__ import annotations

import hashlib
import os
import socket

import pytest
import torch.multiprocessing as mp

from paper_1810_10496_b200 import campaign, explorer, registry
from paper_1810_10496_b200.backend.types import (
    Artifact,
    Backend,
    CompileOutcome,
    ExecutionOutcome,
    ExecutionStatus,
    InputKind,
    KernelCase,
)

BENCHES = ["GEMM", "ATAX", "2DCONV", "SYRK"]
REF = (1.0, 2.0, 3.0, 4.0)


def _h(text: str) -> int:
    return int.from_bytes(hashlib.sha256(text.encode()).digest()[:8], "big")


class HashBackend(Backend):
    """Deterministic in (kernel, artifact): times, failures and outputs are
    hashes, so the result cannot depend on which rank ran what, or when."""

    def __init__(self):
        super().__init__()
        self.timeouts = {}

    def set_timeout_override(self, kernel_id, timeout):
        self.timeouts[kernel_id] = timeout

    def compile(self, kernel, order):
        names = [p.name for p in order.passes]
        if len(names) > 2 and _h("noir" + "-".join(names)) % 23 == 0:
            return CompileOutcome.optimizer_failure("bad order")
        # commutative-ish artifact: pass set + how many loop-unrolls (max 3), so digests collide
        key = f"{kernel.id}|{sorted(set(names))}|{min(3, names.count('loop-unroll'))}"
        return CompileOutcome.success(Artifact.from_content(key.encode()))

    def execute(self, kernel, order, artifact, input_kind, random_input_index=None):
        h = _h(artifact.digest)
        empty = len(order) == 0
        if input_kind is InputKind.MEASUREMENT:
            t = 1.0 if empty else 0.3 + (h % 1000) / 1000.0
            if not empty and h % 29 == 0:
                return ExecutionOutcome(ExecutionStatus.CRASH, log="boom")
            return ExecutionOutcome(ExecutionStatus.VALID, wall_time=t, outputs=None)
        outs = REF
        if not empty and h % 17 == 0:
            outs = tuple(x * 1.5 for x in REF)  # wrong answers
        if random_input_index is not None and not empty and (h + random_input_index) % 31 == 0:
            outs = tuple(x + 1.0 for x in REF)  # fails revalidation only
        return ExecutionOutcome(ExecutionStatus.VALID, wall_time=1e-3, outputs=outs)


def _kernels():
    return [KernelCase(b, registry.source_of(b), "v", "m", REF, registry.kernel_case(b).ir_text) for b in BENCHES]


CFG = explorer.ExplorationConfig(num_sequences=120, max_len=10, top_k=4, final_reps=5, final_random_inputs=4)


def _summary(res):
    return (res.kb.to_json_dict(), [(r.kernel_id, r.order.text, r.artifact_digest, r.status.value, r.wall_time,
                                     r.eval_index) for r in res.store.records],
            res.report.geomean, res.loo)


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world),
                      LOCAL_RANK=str(rank))
    from paper_1810_10496_b200.dist import Dist

    d = Dist(backend="gloo")
    try:
        res = campaign.run_campaign(_kernels(), HashBackend(), CFG, loo_k=3, loo_trials=20, log=lambda *a: None,
                                    dist=d)
        q.put((rank, _summary(res)))
    finally:
        d.close()


def test_kernel_owners_lpt_and_affinity():
    ks = _kernels()
    assert campaign.kernel_owners(ks, 1) == [0, 0, 0, 0]
    owners = campaign.kernel_owners(ks, 2, {"GEMM": 10.0, "ATAX": 1.0, "2DCONV": 1.0, "SYRK": 8.0})
    assert owners[0] != owners[3]  # the two expensive kernels go to different ranks
    assert sorted(set(owners)) == [0, 1]


@pytest.mark.timeout(300)
def test_campaign_world_size_two_equals_serial():
    serial = _summary(campaign.run_campaign(_kernels(), HashBackend(), CFG, loo_k=3, loo_trials=20,
                                            log=lambda *a: None))
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = dict(q.get(timeout=280) for _ in procs)
    for p in procs:
        p.join(timeout=30)
    assert got[0] == serial
    assert got[1] == serial
