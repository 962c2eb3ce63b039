"""Multi-process (world_size 2, gloo, CPU) coverage of the N>1 path:
LPT sharding of a candidate round, max-over-ranks timing, evaluation counts
and record gathering -- the same plumbing bench.py uses over NCCL."""

from __future__ import annotations

import os
import socket

import pytest
import torch.multiprocessing as mp

from paper_1810_10496_b200.sweep import shard


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world),
                      LOCAL_RANK=str(rank))
    from paper_1810_10496_b200.dist import Dist
    from paper_1810_10496_b200.sweep import shard as shard_fn

    d = Dist(backend="gloo")
    work = [f"cand{i}" for i in range(37)]
    costs = [float((i * 7919) % 23 + 1) for i in range(37)]
    mine = shard_fn(work, costs, d.world, d.rank)
    local_time = sum(costs[work.index(w)] for w in mine)
    d.barrier()
    t_max = d.max(local_time)
    n_total = d.sum(len(mine))
    gathered = d.gather(mine)
    d.close()
    q.put((rank, mine, local_time, t_max, n_total, gathered))


def test_shard_partitions_and_balances_single_process():
    work = list(range(50))
    costs = [float(1 + (i % 5) * 3) for i in work]
    parts = [shard(work, costs, 4, r) for r in range(4)]
    flat = sorted(x for p in parts for x in p)
    assert flat == work
    loads = [sum(costs[x] for x in p) for p in parts]
    assert max(loads) - min(loads) <= max(costs)


@pytest.mark.timeout(120)
def test_world_size_two_gloo():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = [q.get(timeout=100) for _ in procs]
    for p in procs:
        p.join(timeout=30)
        assert p.exitcode == 0
    got.sort()
    (r0, m0, t0, tmax0, n0, g0), (r1, m1, t1, tmax1, n1, g1) = got
    assert set(m0).isdisjoint(m1) and len(m0) + len(m1) == 37
    assert tmax0 == tmax1 == max(t0, t1)
    assert n0 == n1 == 37
    assert g0 == g1 == [m0, m1]
