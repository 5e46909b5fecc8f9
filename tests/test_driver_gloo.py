"""Multi-process (world_size 2, gloo, CPU) coverage of the batch-sharded driver.

The GPU runs use NCCL with the same code path; here each rank produces
rank-tagged 'logits' for its shard and the gathered result must be the
global batch in input order.
"""

import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2307_08771_b200.driver import ReplicaDriver, shard_batch


def test_shard_batch_covers_in_order():
    for world in (1, 2, 3, 4, 8):
        for n in (8, 9, 256, 257):
            shards = [shard_batch(n, r, world) for r in range(world)]
            assert shards[0].start == 0 and shards[-1].stop == n
            assert all(a.stop == b.start for a, b in zip(shards, shards[1:]))
            assert max(s.size for s in shards) - min(s.size for s in shards) <= 1
    with pytest.raises(ValueError):
        shard_batch(1, 0, 2)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, n, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        sh = shard_batch(n, rank, world)
        ids = torch.arange(sh.start, sh.stop, dtype=torch.float32)

        def run_local():  # stands in for Engine.forward on this rank's shard
            return torch.stack([ids, ids * 10 + rank], dim=1)

        out = ReplicaDriver(run_local).step()
        q.put((rank, out.tolist()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("n", [8, 9])
def test_two_rank_logits_gather(n):
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = dict(q.get(timeout=60) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank in range(world):
        got = torch.tensor(results[rank])
        assert got.shape == (n, 2)
        assert torch.equal(got[:, 0], torch.arange(n, dtype=torch.float32))  # input order
        owner = torch.tensor([shard_batch(n, 0, world).stop <= i for i in range(n)], dtype=torch.float32)
        assert torch.equal(got[:, 1], got[:, 0] * 10 + owner)
