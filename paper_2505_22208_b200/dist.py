"""Data-parallel plumbing of the train step (one process per GPU).

The reference simulates G workers in one process: worker g takes
MiniBatch.samples[g*B .. g*B+B) of every scheduled mini-batch
(S/trainer.cpp:262-268, pack_batch S/scheduler.cpp:43-58), computes its own
masked loss and gradient, and the G gradients are averaged (S/trainer.cpp:319).
Here worker g is rank g: it packs exactly that slice, and liblamm_b200's
lamm_train_step closes the step with one NCCL allreduce. torch.distributed
(gloo) is only used for the rendezvous: exchanging the 128-byte NCCL unique id,
barriers and the max/sum of host scalars for timing.
"""
from __future__ import annotations

import os

import numpy as np

from .api import select


def minibatch_ids(sched: dict, step: int, world: int, batch_per_rank: int) -> np.ndarray:
    """Sample ids of mini-batch `step`, worker-major (the reference's order)."""
    per = world * batch_per_rank
    return sched["sample"][step * per:(step + 1) * per]


def shard_ids(sched: dict, step: int, rank: int, world: int, batch_per_rank: int) -> np.ndarray:
    """Rank `rank`'s B samples of mini-batch `step` (MiniBatch.samples[rank*B, rank*B+B))."""
    ids = minibatch_ids(sched, step, world, batch_per_rank)
    assert np.all(sched["worker"][step * world * batch_per_rank:(step + 1) * world * batch_per_rank]
                  [rank * batch_per_rank:(rank + 1) * batch_per_rank] == rank)
    return ids[rank * batch_per_rank:(rank + 1) * batch_per_rank]


def shard(pool: dict, sched: dict, step: int, rank: int, world: int, batch_per_rank: int) -> dict:
    return select(pool, shard_ids(sched, step, rank, world, batch_per_rank))


class Dist:
    """Rendezvous from the torchrun environment (RANK, WORLD_SIZE, LOCAL_RANK, MASTER_*)."""

    def __init__(self, backend: str = "gloo"):
        self.world = int(os.environ.get("WORLD_SIZE", "1"))
        self.rank = int(os.environ.get("RANK", "0"))
        self.local_rank = int(os.environ.get("LOCAL_RANK", "0"))
        self.td = None
        if self.world > 1:
            import torch.distributed as td
            os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
            if not td.is_initialized():
                td.init_process_group(backend, rank=self.rank, world_size=self.world)
            self.td = td

    def barrier(self):
        if self.td:
            self.td.barrier()

    def allreduce(self, x: float, op: str = "sum") -> float:
        if not self.td:
            return x
        import torch
        t = torch.tensor([x], dtype=torch.float64)
        self.td.all_reduce(t, op=self.td.ReduceOp.MAX if op == "max" else self.td.ReduceOp.SUM)
        return float(t.item())

    def allreduce_array(self, a: np.ndarray, op: str = "sum") -> np.ndarray:
        if not self.td:
            return a
        import torch
        t = torch.from_numpy(np.ascontiguousarray(a, np.float64).copy())
        self.td.all_reduce(t, op=self.td.ReduceOp.MAX if op == "max" else self.td.ReduceOp.SUM)
        return t.numpy()

    def bcast_bytes(self, b: bytes | None) -> bytes:
        if not self.td:
            return b
        obj = [b]
        self.td.broadcast_object_list(obj, src=0)
        return obj[0]

    def close(self):
        if self.td and self.td.is_initialized():
            self.td.destroy_process_group()
