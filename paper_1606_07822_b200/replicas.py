"""Multi-GPU data parallelism for the training pass.

The corpus shards naturally (the reference already gives each worker its own byte
range, corpus.hpp:192-223): one process per GPU holds a full syn0+syn1 replica,
trains its own shard of the id stream with the device kernels, and every
``sync_words`` words per replica the replicas average their models with one
all-reduce (NCCL over NVLink/NVSwitch at N > 1; gloo on CPU in the tests). The
learning rate follows the global schedule estimated as N x local progress.

The local step and the model buffer are injected so that the same orchestration
drives a GPU ``api.Session`` (bench.py) and a CPU stand-in (tests/test_replicas.py).
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Callable


@dataclass
class Chunk:
    begin: int
    end: int


def plan_chunks(n_tokens: int, sync_words: int) -> list[Chunk]:
    """Consecutive ranges of the local shard between two averaging points."""
    if n_tokens <= 0:
        return []
    step = max(1, int(sync_words))
    return [Chunk(a, min(n_tokens, a + step)) for a in range(0, n_tokens, step)]


def shard_bounds(total: int, world: int, rank: int) -> tuple[int, int]:
    """Near-equal contiguous split of a global id stream (corpus.hpp:192-223 on ids)."""
    a = total * rank // world
    b = total * (rank + 1) // world
    return a, b


class ReplicaTrainer:
    """Runs passes of `local_step` over a replica's shard and averages the model.

    local_step(epoch, begin, end, progress_base, progress_mult) trains ids[begin:end)
    of this replica's shard and returns per-call stats (anything).
    model: a tensor aliasing the replica's whole model buffer (syn0 and syn1).
    """

    def __init__(self, local_step: Callable, model, world: int = 1, rank: int = 0, sync_words: int = 1_000_000,
                 group=None):
        self.local_step = local_step
        self.model = model
        self.world = world
        self.rank = rank
        self.sync_words = sync_words
        self.group = group
        self.syncs = 0

    def average(self) -> None:
        if self.world <= 1:
            return
        import torch.distributed as dist

        if dist.get_backend(self.group) == "nccl":
            dist.all_reduce(self.model, op=dist.ReduceOp.AVG, group=self.group)
        else:  # gloo has no AVG
            dist.all_reduce(self.model, op=dist.ReduceOp.SUM, group=self.group)
            self.model.div_(self.world)
        self.syncs += 1

    def run_pass(self, epoch: int, n_tokens: int, tokens_before: int = 0) -> list:
        """One pass over the local shard; `tokens_before` = local tokens of earlier passes."""
        out = []
        for ch in plan_chunks(n_tokens, self.sync_words if self.world > 1 else n_tokens):
            out.append(self.local_step(epoch, ch.begin, ch.end, (tokens_before + ch.begin) * self.world, self.world))
            self.average()
        return out
