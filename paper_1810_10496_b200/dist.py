"""One-process-per-GPU plumbing for candidate sharding.

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

    def close(self) -> None:
        if self.pg:
            self.pg.destroy_process_group()
            self.pg = None
