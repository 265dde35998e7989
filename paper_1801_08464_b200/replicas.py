"""Replica plumbing for multi-GPU runs (the solve does not shard).

One process per GPU; each rank solves its own independent system (seeded by
rank), the only communication is timing: a barrier around the timed region
and the max of the per-rank device times (torch.distributed, NCCL on GPUs,
gloo on CPU for the tests).  No data-path collective exists, by design.
"""
from __future__ import annotations

import os


def env():
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")),
            int(os.environ.get("LOCAL_RANK", "0")))


class Replicas:
    def __init__(self, backend: str | None = None):
        self.rank, self.world, self.local = env()
        self.dist = None
        self.device = None
        if self.world > 1:
            import torch
            import torch.distributed as dist
            if backend is None:
                backend = "nccl" if torch.cuda.is_available() else "gloo"
            if backend == "nccl":
                torch.cuda.set_device(self.local)
                self.device = f"cuda:{self.local}"
            else:
                self.device = "cpu"
            if not dist.is_initialized():
                dist.init_process_group(backend)
            self.dist = dist

    def barrier(self):
        if self.dist:
            self.dist.barrier()

    def max(self, value: float) -> float:
        if not self.dist:
            return float(value)
        import torch
        t = torch.tensor([float(value)], dtype=torch.float64, device=self.device)
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX)
        return float(t.item())

    def sum(self, value: float) -> float:
        if not self.dist:
            return float(value)
        import torch
        t = torch.tensor([float(value)], dtype=torch.float64, device=self.device)
        self.dist.all_reduce(t, op=self.dist.ReduceOp.SUM)
        return float(t.item())

    def seed(self, base: int = 0) -> int:
        """Independent system per replica (config-5 sequence style: seed + rank)."""
        return base + self.rank

    def close(self):
        if self.dist and self.dist.is_initialized():
            self.dist.barrier()
            self.dist.destroy_process_group()
