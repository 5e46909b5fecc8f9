"""Batch-sharded multi-GPU driver.

Images are independent, so the path shards without any collective inside the
forward pass: rank r runs its own engine replica over its slice of the batch,
and the only exchange is one all-gather of the [batch, classes] fp32 logits at
the end of a step (NCCL over NVLink on the GPUs; gloo in the CPU tests).
"""

from __future__ import annotations

from dataclasses import dataclass

import torch
import torch.distributed as dist


@dataclass(frozen=True)
class Shard:
    rank: int
    world: int
    start: int
    stop: int

    @property
    def size(self) -> int:
        return self.stop - self.start


def shard_batch(global_batch: int, rank: int, world: int) -> Shard:
    """Contiguous, near-equal shards (the first `global_batch % world` ranks get
    one extra image), so the gathered logits come back in input order."""
    if not (0 <= rank < world) or global_batch < world:
        raise ValueError(f"cannot shard {global_batch} images over {world} ranks (rank {rank})")
    base, extra = divmod(global_batch, world)
    start = rank * base + min(rank, extra)
    return Shard(rank, world, start, start + base + (1 if rank < extra else 0))


class ReplicaDriver:
    """One engine replica per process; `step` runs it and gathers the logits."""

    def __init__(self, run_local, group=None, equal_shards: bool = False):
        self.run_local = run_local  # callable: () -> local logits tensor [b_local, classes]
        self.group = group
        self.equal_shards = equal_shards  # skip the size exchange (weak scaling: same batch per rank)
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        self._out = None

    def gather(self, local: torch.Tensor) -> torch.Tensor:
        if self.world == 1:
            return local
        local = local.contiguous()
        if self.equal_shards:
            n = [local.shape[0]] * self.world
            if self._out is None or self._out.shape != (sum(n), *local.shape[1:]):
                self._out = torch.empty((sum(n), *local.shape[1:]), dtype=local.dtype, device=local.device)
            dist.all_gather_into_tensor(self._out, local, group=self.group)
            return self._out
        sizes = [torch.zeros(1, dtype=torch.int64, device=local.device) for _ in range(self.world)]
        dist.all_gather(sizes, torch.tensor([local.shape[0]], device=local.device), group=self.group)
        n = [int(s.item()) for s in sizes]
        if len(set(n)) == 1:  # equal shards: one flat collective
            if self._out is None or self._out.shape != (sum(n), *local.shape[1:]):
                self._out = torch.empty((sum(n), *local.shape[1:]), dtype=local.dtype, device=local.device)
            dist.all_gather_into_tensor(self._out, local, group=self.group)
            return self._out
        # ragged shards: pad to the largest shard (collectives need equal sizes), then trim
        big = max(n)
        padded = torch.zeros((big, *local.shape[1:]), dtype=local.dtype, device=local.device)
        padded[: local.shape[0]] = local
        parts = [torch.empty_like(padded) for _ in n]
        dist.all_gather(parts, padded, group=self.group)
        return torch.cat([part[:k] for part, k in zip(parts, n)])

    def step(self) -> torch.Tensor:
        return self.gather(self.run_local())
