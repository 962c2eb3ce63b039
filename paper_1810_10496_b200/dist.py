"""One-process-per-GPU plumbing for candidate sharding.

``Dist.map`` is the one scheduling primitive: independent evaluations are
sharded over ranks and their (small) results gathered to every rank, so all
ranks hold identical engine state afterwards.

Candidate evaluations are independent, so no collective touches the data
path: torch.distributed is used only for barriers, the max-over-ranks timing
reduction, sums of evaluation counts and gathering small result records.
NCCL when CUDA is available (the bench under torchrun), gloo otherwise (the
CPU tests).
"""

from __future__ import annotations

import os


class Dist:
    def __init__(self, backend: str | None = None):
        self.world = int(os.environ.get("WORLD_SIZE", "1"))
        self.rank = int(os.environ.get("RANK", "0"))
        self.local = int(os.environ.get("LOCAL_RANK", "0"))
        # test hooks: PF_DIST_ONE_DEVICE=1 puts every rank on device 0 and
        # PF_DIST_BACKEND=gloo forces the gloo control plane (NCCL refuses two
        # ranks on one GPU) -- the multi-rank paths then run on a one-GPU box
        if os.environ.get("PF_DIST_ONE_DEVICE") == "1":
            self.local = 0
        backend = backend or os.environ.get("PF_DIST_BACKEND") or None
        self.pg = None
        self.device = None
        if self.world > 1:
            import torch
            import torch.distributed as dist

            if backend is None:
                backend = "nccl" if torch.cuda.is_available() else "gloo"
            if backend == "nccl":
                torch.cuda.set_device(self.local)
                self.device = torch.device("cuda", self.local)
                dist.init_process_group("nccl", device_id=self.device)
            else:
                self.device = torch.device("cpu")
                dist.init_process_group("gloo")
            self.pg = dist

    def barrier(self) -> None:
        if self.pg:
            self.pg.barrier()

    def _reduce(self, x: float, op) -> float:
        import torch

        t = torch.tensor([float(x)], dtype=torch.float64, device=self.device)
        self.pg.all_reduce(t, op=op)
        return float(t.item())

    def max(self, x: float) -> float:
        return x if not self.pg else self._reduce(x, self.pg.ReduceOp.MAX)

    def sum(self, x: float) -> float:
        return x if not self.pg else self._reduce(x, self.pg.ReduceOp.SUM)

    def gather(self, obj) -> list:
        """All ranks' objects (small records only), in rank order."""
        if not self.pg:
            return [obj]
        out = [None] * self.world
        self.pg.all_gather_object(out, obj)
        return out

    def map(self, fn, items: list, costs: list[float] | None = None) -> list:
        """``[fn(x) for x in items]`` with the items sharded over ranks (LPT on
        ``costs``) and the results gathered to every rank, in item order.  An
        exception on any rank is re-raised on every rank (after the gather, so
        no rank is left waiting in it)."""
        if not self.pg:
            return [fn(x) for x in items]
        mine = shard(list(range(len(items))), costs or [1.0] * len(items), self.world, self.rank)
        local = {}
        for i in mine:
            try:
                local[i] = (True, fn(items[i]))
            except Exception as exc:  # noqa: BLE001 -- re-raised below on every rank
                local[i] = (False, exc)
        merged: dict = {}
        for part in self.gather(local):
            merged.update(part)
        out = []
        for i in range(len(items)):
            ok, value = merged[i]
            if not ok:
                raise value
            out.append(value)
        return out

    def map_owned(self, fn, items: list, owners: list[int]) -> list:
        """``[fn(x) for x in items]`` with item i evaluated on rank
        ``owners[i]`` (device affinity), gathered to every rank in item
        order; exceptions are re-raised on every rank as in ``map``."""
        if not self.pg:
            return [fn(x) for x in items]
        local = {}
        for i, x in enumerate(items):
            if owners[i] != self.rank:
                continue
            try:
                local[i] = (True, fn(x))
            except Exception as exc:  # noqa: BLE001 -- re-raised below on every rank
                local[i] = (False, exc)
        merged: dict = {}
        for part in self.gather(local):
            merged.update(part)
        out = []
        for i in range(len(items)):
            ok, value = merged[i]
            if not ok:
                raise value
            out.append(value)
        return out

    def close(self) -> None:
        if self.pg:
            self.pg.destroy_process_group()
            self.pg = None


def assign(costs: list[float], world: int) -> list[int]:
    """Owner rank of each item: longest-processing-time-first (ties by index)."""
    order = sorted(range(len(costs)), key=lambda i: (-costs[i], i))
    loads = [0.0] * world
    owner = [0] * len(costs)
    for i in order:
        r = min(range(world), key=lambda k: loads[k])
        owner[i] = r
        loads[r] += costs[i]
    return owner


def shard(work: list, costs: list[float], world: int, rank: int) -> list:
    """Longest-processing-time-first assignment; returns this rank's items in
    their original order."""
    order = sorted(range(len(work)), key=lambda i: -costs[i])
    loads = [0.0] * world
    owner = [0] * len(work)
    for i in order:
        r = min(range(world), key=lambda k: loads[k])
        owner[i] = r
        loads[r] += costs[i]
    return [w for i, w in enumerate(work) if owner[i] == rank]
