"""Multi-GPU data parallelism for the training pass.

The corpus shards naturally (the reference already gives each worker its own byte
range, corpus.hpp:192-223): one process per GPU holds a full syn0+syn1 replica and
trains its own shard of the id stream with the device kernels. The reference's workers
all add into ONE model (trainer.hpp:72-74, 249-253), so replicas keep additive
semantics: every ``sync_words`` words per replica each replica's delta since the last
sync (model - snapshot) is all-reduced with SUM (NCCL over NVLink/NVSwitch at N > 1;
gloo on CPU in the tests) and applied to the snapshot row by row with the sync scale
(cg_session_sync_apply / cg_sync_row_scale: rows few replicas touched are summed, a row
every replica updated from the same snapshot gets at most 128 stale updates' worth and at
least the replicas' average). The learning rate follows the global schedule estimated as
N x local progress. ``mode="average"`` keeps round 1's whole-model averaging (local SGD
with model averaging) for comparison.

The local step and the replica's sync operations are injected so that the same
orchestration drives a GPU ``api.Session`` (bench.py) and a CPU stand-in
(tests/test_replicas.py).
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Callable


@dataclass
class Chunk:
    begin: int
    end: int


def plan_chunks(n_tokens: int, sync_words: int) -> list[Chunk]:
    """Consecutive ranges of the local shard between two sync points."""
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
    """Runs passes of `local_step` over a replica's shard and syncs the replicas.

    local_step(epoch, begin, end, progress_base, progress_mult) trains ids[begin:end)
    of this replica's shard and returns per-call stats (anything).
    replica: an object with sync_begin(), sync_delta_tensor() -> tensor (delta = model -
    snapshot, all-reduced in place) and sync_apply(n_replicas, words_per_replica) -- an
    ``api.Session`` on the GPU. For mode="average", `model` is a tensor aliasing the
    replica's whole model buffer instead.
    """

    def __init__(self, local_step: Callable, model=None, world: int = 1, rank: int = 0,
                 sync_words: int = 1_000_000, group=None, replica=None, mode: str = "delta"):
        if mode not in ("delta", "average"):
            raise ValueError("mode must be 'delta' or 'average'")
        if world > 1 and mode == "delta" and replica is None:
            raise ValueError("delta sync needs the replica's sync operations")
        if world > 1 and mode == "average" and model is None:
            raise ValueError("averaging needs the model tensor")
        self.local_step = local_step
        self.model = model
        self.replica = replica
        self.world = world
        self.rank = rank
        self.sync_words = sync_words
        self.group = group
        self.mode = mode
        self.syncs = 0
        self.sync_bytes = 0
        self.sync_seconds = 0.0  # host wall time inside sync points (their device work is blocking)
        self._begun = False

    def _all_reduce_sum(self, t) -> None:
        import torch.distributed as dist

        dist.all_reduce(t, op=dist.ReduceOp.SUM, group=self.group)

    def average(self) -> None:
        import torch.distributed as dist

        if dist.get_backend(self.group) == "nccl":
            dist.all_reduce(self.model, op=dist.ReduceOp.AVG, group=self.group)
        else:  # gloo has no AVG
            self._all_reduce_sum(self.model)
            self.model.div_(self.world)
        self.sync_bytes += self.model.numel() * self.model.element_size()

    def sync(self, words: int) -> None:
        """One sync point after `words` tokens per replica since the last one."""
        if self.world <= 1:
            return
        import time

        t0 = time.perf_counter()
        if self.mode == "average":
            self.average()
        else:
            d = self.replica.sync_delta_tensor()
            self._all_reduce_sum(d)
            self.replica.sync_apply(self.world, words)
            self.sync_bytes += d.numel() * d.element_size()
        self.syncs += 1
        self.sync_seconds += time.perf_counter() - t0

    def run_pass(self, epoch: int, n_tokens: int, tokens_before: int = 0) -> list:
        """One pass over the local shard; `tokens_before` = local tokens of earlier passes."""
        if self.world > 1 and self.mode == "delta" and not self._begun:
            self.replica.sync_begin()
            self._begun = True
        out = []
        for ch in plan_chunks(n_tokens, self.sync_words if self.world > 1 else n_tokens):
            out.append(self.local_step(epoch, ch.begin, ch.end, (tokens_before + ch.begin) * self.world, self.world))
            self.sync(self.sync_words)
        return out
