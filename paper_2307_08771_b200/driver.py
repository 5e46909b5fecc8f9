"""Batch-sharded multi-GPU driver.

Images are independent, so the path shards without any collective inside the
forward pass.  A global batch of G images is split into contiguous shards of
G/g images (strong scaling, north_star: "batch 256 -> 256/g images per
replica"); rank r runs its own engine replica over its shard, and the only
exchange is one all-gather of the [G, classes] fp32 logits per step (NCCL over
NVLink on the GPUs; gloo in the CPU tests).

On CUDA the gather of step i runs on a side stream while step i+1's forward
replays: the logits are copied into one of two send buffers on the compute
stream, the comm stream waits for that copy and issues the all-gather; a send
buffer is reused only after the gather that read it has finished.
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
    """One engine replica per process over its shard of a global batch.

    `submit(local)` hands over this step's local logits (already enqueued on the
    current stream) and starts their gather; `result()` returns the last step's
    gathered [G, classes] logits in input order; `drain()` makes the current
    stream wait for every gather in flight.  `step()` = run_local + submit +
    result, the synchronous form."""

    def __init__(self, run_local=None, global_batch: int | None = None, group=None, overlap: bool = True):
        self.run_local = run_local
        self.group = group
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.global_batch = global_batch
        self.overlap = overlap
        self.shards = ([shard_batch(global_batch, r, self.world) for r in range(self.world)]
                       if global_batch is not None else None)
        self._send = self._out = None
        self._done = [None, None]
        self._k = 0
        self._last = None
        self._comm = None
        self._sizes = None

    @property
    def shard(self) -> Shard:
        return self.shards[self.rank]

    def _buffers(self, local: torch.Tensor):
        if self._send is not None and self._send[0].shape[1:] == local.shape[1:]:
            return
        if self.shards is None:  # sizes unknown: exchange them once
            t = torch.tensor([local.shape[0]], dtype=torch.int64,
                             device=local.device if local.is_cuda else "cpu")
            parts = [torch.zeros_like(t) for _ in range(self.world)]
            dist.all_gather(parts, t, group=self.group)
            self._sizes = [int(p.item()) for p in parts]
        else:
            self._sizes = [s.size for s in self.shards]
        pad = max(self._sizes)
        shp = (pad, *local.shape[1:])
        self._send = [torch.zeros(shp, dtype=local.dtype, device=local.device) for _ in range(2)]
        self._out = [torch.zeros((self.world * pad, *local.shape[1:]), dtype=local.dtype, device=local.device)
                     for _ in range(2)]
        if local.is_cuda and self.overlap:
            self._comm = torch.cuda.Stream(device=local.device)

    def submit(self, local: torch.Tensor) -> None:
        if self.world == 1:
            self._last = local
            return
        self._buffers(local)
        k = self._k
        self._k ^= 1
        send, out = self._send[k], self._out[k]
        if self._comm is not None:
            cur = torch.cuda.current_stream(local.device)
            if self._done[k] is not None:
                cur.wait_event(self._done[k])  # the gather that read send[k] two steps ago
            send[: local.shape[0]].copy_(local, non_blocking=True)
            ready = torch.cuda.Event()
            ready.record(cur)
            with torch.cuda.stream(self._comm):
                self._comm.wait_event(ready)
                work = dist.all_gather_into_tensor(out, send, group=self.group, async_op=True)
                work.wait()  # the comm stream (not the host) waits for NCCL
                done = torch.cuda.Event()
                done.record(self._comm)
            self._done[k] = done
        else:
            send[: local.shape[0]].copy_(local)
            parts = list(out.chunk(self.world))
            dist.all_gather(parts, send, group=self.group)
        self._last = k

    def drain(self) -> None:
        if self._comm is not None:
            torch.cuda.current_stream(self._comm.device).wait_stream(self._comm)

    def result(self) -> torch.Tensor:
        if self.world == 1:
            return self._last
        self.drain()
        out = self._out[self._last]
        pad = out.shape[0] // self.world
        if all(n == pad for n in self._sizes):
            return out
        return torch.cat([out[r * pad: r * pad + n] for r, n in enumerate(self._sizes)])

    def gather(self, local: torch.Tensor) -> torch.Tensor:
        self.submit(local)
        return self.result()

    def step(self) -> torch.Tensor:
        return self.gather(self.run_local())
