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


class _StubEngine:
    """Stands in for a captured Engine on CPU: the 'logits' of an image are a few of its
    own pixels, so the gathered result shows whether the shards came back in order."""

    def __init__(self, b):
        self.batch = b
        self.input_buf = torch.zeros(b, 3, 224, 224)
        self.n_launches = 7
        self._out = torch.zeros(b, 5)

    def replay(self, slot=0):
        self._out = self.input_buf[:, 0, 0, :5].clone()

    def output_tensor(self):
        return self._out


def _bench_worker(rank, world, port, q):
    import sys
    from types import SimpleNamespace

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world),
                      LOCAL_RANK=str(rank))
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    import bench

    args = SimpleNamespace(gpus=world, steps=3, warmup=3, batch=256, config="resnet50_s50", strategy="reorder",
                           gather="fused", no_extras=True, no_cpu_baseline=True)
    try:
        line, gathered = bench.run_ours(args, make=lambda b, dev: _StubEngine(b), device="cpu")
        q.put((rank, line, gathered.tolist()))
    finally:
        dist.destroy_process_group()


def test_bench_rank_logic_two_gloo_ranks():
    """bench.py's own rank logic (strong scaling: the global batch of 256 split 128 + 128,
    logits gathered in input order, ms max over ranks) with a stubbed engine."""
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_bench_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = {r: (line, g) for r, line, g in (q.get(timeout=180) for _ in range(world))}
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    x_all = torch.randn(256, 3, 224, 224, generator=torch.Generator().manual_seed(0))
    want = x_all[:, 0, 0, :5]
    for rank, (line, g) in results.items():
        assert line["n_gpus"] == 2 and line["scaling"] == "strong"
        assert line["config"]["global_batch"] == 256 and line["config"]["per_gpu_batch"] == 128
        assert torch.equal(torch.tensor(g), want)
    assert results[0][0]["ms_per_step"] == results[1][0]["ms_per_step"]  # max over ranks


def test_bench_refuses_mismatched_world(monkeypatch):
    import sys
    from types import SimpleNamespace

    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import bench

    monkeypatch.setenv("WORLD_SIZE", "1")
    with pytest.raises(SystemExit):
        bench.rank_env(SimpleNamespace(gpus=8))
