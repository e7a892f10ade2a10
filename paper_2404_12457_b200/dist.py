"""Multi-GPU plumbing for the hot path (one process per GPU).

* requests are routed data-parallel: request ``id mod world`` goes to rank
  ``id mod world``; each rank owns an independent knowledge-tree + pool
  replica, so its decisions equal a ragsim run on its routed sub-trace;
* the corpus is split in contiguous row shards; a retrieval step gathers the
  ranks' queries, scans the local shard for all of them, gathers the
  per-shard staged top-k lists and merges them (score desc, id asc) — stage s
  is the top-k over the union of every shard's first (s+1)/S rows.

``Dist`` wraps torch.distributed (NCCL on the GPU box, gloo in CPU tests);
all_gather writes one [world, ...] buffer (all_gather_into_tensor, NCCL and gloo).
"""

from __future__ import annotations

import os

import torch


def shard_bounds(n_rows: int, rank: int, world: int) -> tuple[int, int]:
    return (n_rows * rank) // world, (n_rows * (rank + 1)) // world


def route(requests, rank: int, world: int):
    return [r for r in requests if r.id % world == rank]


class Dist:
    def __init__(self) -> None:
        self.world = int(os.environ.get("WORLD_SIZE", "1"))
        self.rank = int(os.environ.get("RANK", "0"))
        self.local = int(os.environ.get("LOCAL_RANK", "0"))
        self.pg = None
        self.device = "cpu"
        self.backend = None

    def init(self, backend: str = "nccl") -> "Dist":
        self.backend = backend
        self.device = "cuda" if backend == "nccl" else "cpu"
        if self.world > 1:
            import torch.distributed as dist

            os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
            dist.init_process_group(backend=backend, rank=self.rank, world_size=self.world)
            self.pg = dist
        return self

    def barrier(self) -> None:
        if self.pg is not None:
            self.pg.barrier()

    def max(self, x: float) -> float:
        if self.pg is None:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=self.device)
        self.pg.all_reduce(t, op=self.pg.ReduceOp.MAX)
        return float(t.item())

    def sum(self, x: float) -> float:
        if self.pg is None:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=self.device)
        self.pg.all_reduce(t)
        return float(t.item())

    def all_gather(self, t: torch.Tensor) -> torch.Tensor:
        """[world, *t.shape] (rank order)."""
        if self.pg is None:
            return t.unsqueeze(0)
        if self.backend == "gloo" and t.is_cuda:  # gloo: list form for device tensors
            parts = [torch.empty_like(t) for _ in range(self.world)]
            self.pg.all_gather(parts, t.contiguous())
            return torch.stack(parts)
        out = torch.empty(self.world * t.numel(), dtype=t.dtype, device=t.device)
        self.pg.all_gather_into_tensor(out, t.contiguous().reshape(-1))  # one buffer, no stack
        return out.view((self.world,) + tuple(t.shape))

    def all_gather_object(self, obj) -> list:
        """Picklable object of every rank, rank order (setup-time exchanges)."""
        if self.pg is None:
            return [obj]
        out = [None] * self.world
        self.pg.all_gather_object(out, obj)
        return out

    def close(self) -> None:
        if self.pg is not None:
            self.pg.destroy_process_group()
            self.pg = None
