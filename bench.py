#!/usr/bin/env python
"""Benchmark: UPSCALE-exported ResNet-50 @ 50% on B200 (BASELINE.json configs[2]).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

One step = one forward pass of the exported pruned ResNet-50 over a GLOBAL batch
of 256 synthetic 224x224 images, sharded 256/N per GPU (strong scaling,
SURVEY.md 8e / north_star), followed by the one exchange of the path: an NCCL
all-gather of the [256, 1000] fp32 logits, overlapped with the next step's
forward.  `--gpus N > 1` without a torchrun environment relaunches itself under
`torch.distributed.run` with N ranks.  Rank 0 prints ONE JSON line: `value` is
device-timed (CUDA events, max over ranks) with inputs resident in HBM; `e2e`
goes through the public API (`api.Runner.run_many`) with pinned host input,
H2D + D2H inside the timed region.  `--impl reference` times the reference's
CPU path (the oracle port of interp.run over the same exported graph) on the
host cores, rank 0 only.
"""

from __future__ import annotations

import argparse
import json
import os
import socket
import statistics
import subprocess
import sys
import tempfile
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "pruned ResNet-50 images/sec + b1 latency, % roofline, 1/2/4/8 B200 vs CPU ref"
UNIT = "images/s"
PEAKS_FALLBACK = {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}


def peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        d["source"] = "measured (MEASURED_PEAKS.json)"
        return d
    d = dict(PEAKS_FALLBACK)
    d["source"] = "fallback (B200_PROFILING.md)"
    return d


# --------------------------------------------------------------------------- clocks
class ClockSampler:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.idx = gpu_index
        self.proc = None
        self.path = None

    def start(self):
        try:
            fd, self.path = tempfile.mkstemp(suffix=".csv")
            os.close(fd)
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.idx), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "50"], stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except (OSError, FileNotFoundError):
            self.proc = None

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        sm, smax, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in Path(self.path).read_text().splitlines():
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[1]))
                smax = float(parts[2])
            except ValueError:
                continue
            for n, v in zip(names, parts[4:8]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        os.unlink(self.path)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": smax, "reasons": sorted(reasons),
                "samples": len(sm)}


# --------------------------------------------------------------------------- CPU reference path
def _cpu_model(cfg_name: str, strategy: str):
    from oracle.apply_plan_ref import apply_plans_spatial
    from paper_2307_08771_b200 import export as E, plans as P
    from paper_2307_08771_b200.configs import CONFIGS, build_spatial_model

    cfg = CONFIGS[cfg_name]
    sm = build_spatial_model(cfg)
    plans = P.load_plans(cfg.asset_dir / f"plans_{strategy}.json")
    eg = E.export_graph(sm.graph, plans)
    w, v = apply_plans_spatial(plans, sm.graph, sm.weights, sm.vectors)
    return sm, eg, {k: t.float() for k, t in w.items()}, v


def _time_cpu(eg, sm, w, v, n, warm=2, runs=5, budget_s=8.0):
    import torch

    from oracle.spatial_ref import run_spatial

    x = torch.randn(n, 3, 224, 224, generator=torch.Generator().manual_seed(0))
    with torch.no_grad():
        for _ in range(warm):
            run_spatial(eg, sm.specs, w, v, x, dtype=torch.float32)
        times = []
        t_start = time.perf_counter()
        while len(times) < runs:
            t0 = time.perf_counter()
            run_spatial(eg, sm.specs, w, v, x, dtype=torch.float32)
            times.append(time.perf_counter() - t0)
            if time.perf_counter() - t_start > budget_s and len(times) >= 3:
                break
    return statistics.median(times), len(times)


def cpu_baseline(cfg_name: str) -> dict:
    """the reference's CPU path on this box's host cores -- the oracle port
    of interp.run (torch fp32, all threads) over both exports at N = 1 and N = 32
    (2 warm-ups, median of >= 3-5 runs), plus the reference's own export time
    (`reslice.plan_model` + `apply_plan`, single-threaded Python)."""
    import torch

    torch.set_num_threads(os.cpu_count() or 1)
    out = {"unit": UNIT, "cores": torch.get_num_threads(), "kind": "port", "legs": {}}
    for strategy in ("reorder", "baseline"):
        sm, eg, w, v = _cpu_model(cfg_name, strategy)
        for n in (1, 32):
            t, runs = _time_cpu(eg, sm, w, v, n)
            out["legs"][f"{strategy}_n{n}"] = {"images_per_s": round(n / t, 2), "median_s": round(t, 4), "runs": runs}
    out["value"] = out["legs"]["reorder_n32"]["images_per_s"]
    out["sample"] = (f"oracle/spatial_ref.py (fp32 torch CPU, {out['cores']} threads) over the reorder and baseline "
                     f"exports of {cfg_name} at N=1 and N=32, 2 warm-ups, median of 3-5 runs; value = reorder N=32")
    try:
        out["reference_export_seconds"] = reference_export_seconds(cfg_name)
    except Exception as exc:  # the reference package is optional on the box
        out["reference_export_seconds"] = {"unavailable": f"{type(exc).__name__}: {exc}"[:200]}
    return out


def reference_export_seconds(cfg_name: str) -> dict:
    """The reference export (pipeline.py:99-146) on the CPU: plan_model + apply_plan over
    the 2-D proxies, pure Python, for both strategies."""
    import numpy as np

    from paper_2307_08771_b200 import ir
    from paper_2307_08771_b200.configs import CONFIGS, build_spatial_model
    from paper_2307_08771_b200.ref import reslice

    cfg = CONFIGS[cfg_name]
    sm = build_spatial_model(cfg)
    masks = ir.load_masks(cfg.asset_dir / "masks.json")
    store = reslice.WeightStore({k: np.asarray(a) for k, a in sm.proxy_weights().items()})
    res = {}
    for strategy in ("baseline", "reorder"):
        t0 = time.perf_counter()
        plans, _ = reslice.plan_model(sm.graph, masks, "input", strategy, "baseline")
        t1 = time.perf_counter()
        g, st = sm.graph, store
        for p in plans:
            g, st = reslice.apply_plan(p, g, st)
        t2 = time.perf_counter()
        res[strategy] = {"plan_model_s": round(t1 - t0, 3), "apply_plan_s": round(t2 - t1, 3)}
    return res


def run_reference(args):
    """--impl reference: the reference's CPU path on the host cores, rank 0 only."""
    if int(os.environ.get("RANK", "0")) != 0:
        return
    import torch

    torch.set_num_threads(os.cpu_count() or 1)
    from oracle.spatial_ref import run_spatial

    sm, eg, w, v = _cpu_model(args.config, args.strategy)
    n = args.ref_images
    x = torch.randn(n, 3, 224, 224, generator=torch.Generator().manual_seed(0))
    with torch.no_grad():
        for _ in range(args.warmup):
            run_spatial(eg, sm.specs, w, v, x, dtype=torch.float32)
        t0 = time.perf_counter()
        for _ in range(args.steps):
            run_spatial(eg, sm.specs, w, v, x, dtype=torch.float32)
        dt = (time.perf_counter() - t0) / args.steps
    val = n / dt
    sample = (f"{n} images per step (a bounded sample of the {args.batch}-image global batch), "
              f"oracle/spatial_ref.py fp32 torch CPU over the {args.strategy} export")
    line = {"impl": "reference", "metric": METRIC, "value": val, "unit": UNIT, "n_gpus": 1,
            "launched_with_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt * 1e3,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic",
            "config": {"workload": f"{args.config} ({args.strategy} export), CPU sample of {n} images per step",
                       "global_batch": args.batch, "sample_batch": n, "image": [3, 224, 224]},
            "cpu_baseline": {"value": val, "unit": UNIT, "cores": torch.get_num_threads(), "kind": "port",
                             "sample": sample},
            "e2e": {"value": val, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# --------------------------------------------------------------------------- GPU path
def self_launch(args) -> int:
    """`--gpus N` outside torchrun: relaunch under torch.distributed.run, one rank per GPU."""
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", f"--master-port={port}", str(Path(__file__).resolve()), *sys.argv[1:]]
    return subprocess.call(cmd)


def rank_env(args) -> tuple[int, int, int]:
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")
    return rank, world, local


def default_engine_factory(args):
    """Builds the exported model's engine for a shard of `b` images (CUDA-graph captured,
    autotuned)."""
    from paper_2307_08771_b200 import engine as EN, export as E, plans as P
    from paper_2307_08771_b200.configs import CONFIGS, build_spatial_model

    cfg = CONFIGS[args.config]
    sm = build_spatial_model(cfg)

    def make(b, dev, strategy=None, gather=None):
        strategy = strategy or args.strategy
        plans = P.load_plans(cfg.asset_dir / f"plans_{strategy}.json")
        eg = E.export_graph(sm.graph, plans)
        maps = E.compose_maps(sm.graph, plans)
        eng = EN.from_plans(sm, eg, maps, batch=b, device=dev, gather_mode=gather or args.gather)
        eng.capture()
        eng.model = (sm, eg, maps, plans)
        return eng

    return make


class _Clock:
    """CUDA events on the launch stream (device time), or perf_counter on CPU."""

    def __init__(self, cuda: bool):
        import torch

        self.cuda = cuda
        if cuda:
            self.a = torch.cuda.Event(enable_timing=True)
            self.b = torch.cuda.Event(enable_timing=True)

    def start(self):
        import torch

        if self.cuda:
            torch.cuda.synchronize()
            self.a.record(torch.cuda.current_stream())
        else:
            self.t0 = time.perf_counter()

    def stop(self) -> float:
        import torch

        if self.cuda:
            self.b.record(torch.cuda.current_stream())
            torch.cuda.synchronize()
            return self.a.elapsed_time(self.b)
        return (time.perf_counter() - self.t0) * 1e3


def _max_over_ranks(ms: float, world: int, dev) -> float:
    import torch
    import torch.distributed as dist

    if world == 1:
        return ms
    t = torch.tensor([ms], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def time_sharded(eng, driver, steps: int, warmup: int, world: int, dev, cuda: bool) -> float:
    """Replay the shard's forward + hand its logits to the (overlapped) gather, K times;
    returns ms per step, max over ranks."""
    import torch.distributed as dist

    def step():
        eng.replay(0)
        driver.submit(eng.output_tensor())

    for _ in range(warmup):
        step()
    driver.drain()
    if world > 1:
        dist.barrier()
    clk = _Clock(cuda)
    clk.start()
    if cuda:  # NVTX range: `ncu --nvtx --nvtx-include "timed/"` profiles exactly these launches
        import torch

        torch.cuda.nvtx.range_push("timed")
    for _ in range(steps):
        step()
    if cuda:
        torch.cuda.nvtx.range_pop()
    driver.drain()
    ms = clk.stop() / steps
    if world > 1:
        dist.barrier()
    return _max_over_ranks(ms, world, dev)


def kernel_table(eng, batch: int, pk: dict, reps: int = 3) -> tuple[list[dict], float]:
    """Per-launch-group device time (CUDA events around each op's launches, eager, after
    warm-up) next to its algorithmic bytes/flops."""
    import torch

    stream = torch.cuda.current_stream()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in eng.ops]
    per_op = [0.0] * len(eng.ops)
    for op in eng.ops:
        op.launch()
    for _ in range(reps):
        for op, (a, b) in zip(eng.ops, evs):
            a.record(stream)
            op.launch()
            b.record(stream)
        torch.cuda.synchronize()
        for i, (a, b) in enumerate(evs):
            per_op[i] += a.elapsed_time(b) / reps
    hbm = pk["hbm_gbs"] * 1e9
    tc = pk["bf16_tflops_sustained"] * 1e12
    stats = {s.name: s for s in eng.conv_stats}
    rows = []
    for op, ms in zip(eng.ops, per_op):
        key = op.info.get("conv", op.output)
        st = stats.get(key) or stats.get(f"{op.output}(copy)")
        byts = (st.bytes + st.gather_bytes) * batch if st else 0.0
        fl = st.flops * batch if st else 0.0
        roof = max(fl / tc, byts / hbm) * 1e3
        rows.append({"op": key, "kernel": eng.kernel_label(op), "us": round(ms * 1e3, 2),
                     "alg_mb": round(byts / 1e6, 2), "gflop": round(fl / 1e9, 2),
                     "gbs": round(byts / (ms / 1e3) / 1e9, 1) if ms > 0 else None,
                     "roofline_us": round(roof * 1e3, 2), "frac": round(roof / ms, 3) if ms > 0 else None,
                     "bound": "tensor" if fl / tc > byts / hbm else "hbm"})
    return rows, sum(per_op)


def roofline_block(rows: list[dict], step_ms: float, pk: dict, b: int) -> dict:
    """`roofline` for the dominant kernel (conv_tc_kernel: most launches and most of the
    step): algorithmic bytes of its launches / their summed event time."""
    dom = [r for r in rows if r["kernel"].startswith("conv_tc")]
    dom_ms = sum(r["us"] for r in dom) / 1e3
    dom_bytes = sum(r["alg_mb"] for r in dom) * 1e6
    total_ms = sum(r["us"] for r in rows) / 1e3
    troof_ms = sum(r["roofline_us"] for r in rows) / 1e3
    achieved = dom_bytes / (dom_ms / 1e3) / 1e9 if dom_ms > 0 else 0.0
    traffic = None
    tfile = ROOT / "profiles" / "traffic.json"
    if tfile.exists():
        try:
            t = json.loads(tfile.read_text())
            if t.get("per_gpu_batch") == b:
                traffic = t.get("conv_tc_kernel", {}).get("dram_bytes_per_launch")
        except (ValueError, OSError):
            traffic = None
    return {"bound": "hbm", "achieved": round(achieved, 1), "peak": pk["hbm_gbs"], "unit": "GB/s",
            "frac": round(achieved / pk["hbm_gbs"], 4), "traffic": traffic,
            "kernel": f"conv_tc_kernel (generic tcgen05 implicit-GEMM conv), {len(dom)} launches per step",
            "algorithmic_bytes_per_launch": round(dom_bytes / max(len(dom), 1)),
            "avg_launch_us": round(dom_ms * 1e3 / max(len(dom), 1), 2),
            "dominant_share_of_step": round(dom_ms / total_ms, 4) if total_ms else None,
            "traffic_source": "profiles/traffic.json (ncu --set full, dram__bytes_read+write per launch)"
            if traffic else None,
            "step_roofline_ms": round(troof_ms, 4),
            "step_roofline_frac": round(troof_ms / step_ms, 4),
            "eager_sum_ms": round(total_ms, 4),
            "peak_source": pk["source"], "tensor_peak_tflops": pk["bf16_tflops_sustained"]}


def b1_latency(make, dev, steps: int, gather: str, strategy: str | None = None) -> dict:
    import torch

    eng1 = make(1, dev, strategy=strategy, gather=gather)
    x = torch.randn(1, 3, 224, 224, generator=torch.Generator().manual_seed(0)).to(dev)
    eng1.input_buf.copy_(x)
    for _ in range(10):
        eng1.replay(0)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    lat = []
    for _ in range(max(30, steps)):
        a.record()
        eng1.replay(0)
        b.record()
        b.synchronize()
        lat.append(a.elapsed_time(b))
    pk = peaks()
    hbm, tc = pk["hbm_gbs"] * 1e9, pk["bf16_tflops_sustained"] * 1e12
    roof = sum(max(s.flops / tc, (s.bytes + s.gather_bytes) / hbm) for s in eng1.conv_stats) * 1e3
    return {"ms": round(statistics.median(lat), 4), "roofline_ms": round(roof, 5), "launches": eng1.n_launches}


def run_ours(args, make=None, device=None):
    import torch
    import torch.distributed as dist

    from paper_2307_08771_b200.driver import ReplicaDriver, shard_batch

    rank, world, local = rank_env(args)
    cuda = device is None
    if cuda:
        torch.cuda.set_device(local)
        dev = torch.device("cuda", local)
    else:
        dev = torch.device(device)
    if world > 1 and not dist.is_initialized():
        if cuda:
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group("gloo")
    G = args.batch
    shard = shard_batch(G, rank, world)
    b = shard.size
    make = make or default_engine_factory(args)
    t0 = time.perf_counter()
    eng = make(b, dev)
    export_s = time.perf_counter() - t0
    x_all = torch.randn(G, 3, 224, 224, generator=torch.Generator().manual_seed(0))
    x = x_all[shard.start:shard.stop].contiguous()
    eng.input_buf.copy_(x.to(dev))
    driver = ReplicaDriver(global_batch=G)

    clocks = ClockSampler(local) if cuda else None
    if clocks:
        for _ in range(args.warmup):  # spin the clocks up before sampling starts
            eng.replay(0)
        clocks.start()
        time.sleep(0.2)
    ms = time_sharded(eng, driver, args.steps, args.warmup, world, dev, cuda)
    clk = clocks.stop() if clocks else None
    gathered = driver.result()
    value = G / (ms / 1e3)
    assert gathered.shape[0] == G

    line = {
        "metric": METRIC, "value": round(value, 2), "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(ms, 4), "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
        "config": {"workload": f"{args.config}: UPSCALE ({args.strategy}) export of random-init torchvision "
                               f"ResNet-50, 50% unconstrained L2 per-layer input pruning; 224x224 images",
                   "global_batch": G, "per_gpu_batch": b, "parallelism": f"batch-sharded replicas x{world}",
                   "gather_mode": args.gather,
                   "l2": "inputs larger than L2: per GPU step >= 0.9 GB of activation traffic (126 MB L2)"},
        "clocks": clk, "gpu_launches": eng.n_launches * args.steps, "launches_per_step": eng.n_launches,
        "export_seconds": round(export_s, 3),
        "logits_gather": "NCCL all_gather_into_tensor of [G, 1000] fp32 on a side stream, overlapped with the "
                         "next step" if world > 1 else None,
    }

    if cuda:
        pk = peaks()
        rows, _ = kernel_table(eng, b, pk)
        line["roofline"] = roofline_block(rows, ms, pk, b)
        line["kernels"] = sorted(rows, key=lambda r: -r["us"])[:16]
        line["e2e"] = e2e_leg(args, eng, x, G, world, dev)
        if not args.no_extras:
            line.update(extras(args, make, dev, G, b, world, driver, ms))
    if rank == 0 and world == 1 and cuda and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(args.config)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
    return line, gathered


def e2e_leg(args, eng, x, G, world, dev) -> dict:
    """Through the public API: api.Runner.run_many on this rank's shard of pinned host
    images (H2D of the kept input channels, graph forward, D2H of the logits, every step)."""
    import torch

    from paper_2307_08771_b200 import api, export as E, plans as P

    sm, eg, maps, plans = eng.model
    ex = api.Exported(E.ExportResult(eg, None, tuple(plans), P.copy_report(plans), ()), sm, maps)
    runner = api.Runner(ex, gather_mode=args.gather, device=dev)
    runner._engines[eng.batch] = eng
    host_x = x.pin_memory()
    for _ in runner.run_many([host_x] * 3):
        pass
    torch.cuda.synchronize()
    k2 = max(10, args.steps // 2)
    clk = _Clock(True)
    clk.start()
    outs = 0
    for out_np in runner.run_many(host_x for _ in range(k2)):
        outs += 1
    e2e_ms = _max_over_ranks(clk.stop() / k2, world, dev)
    assert outs == k2
    return {"value": round(G / (e2e_ms / 1e3), 2), "unit": UNIT, "h2d_bytes_per_step": runner.h2d_bytes * world,
            "d2h_bytes_per_step": int(out_np.nbytes) * world, "ms_per_step": round(e2e_ms, 4), "steps": k2,
            "path": "api.Runner.run_many per rank: pinned host NCHW fp32 shard -> H2D of the channels the INPUT "
                    "GATHER keeps (copy stream, overlapped with the previous forward) -> CUDA-graph forward -> "
                    "D2H logits -> host numpy, every step"}


def extras(args, make, dev, G, b, world, driver, ms) -> dict:
    """b1 latency (UPSCALE and baseline export) on rank 0, and the baseline-export
    (copy-then-conv) GPU arm at the same sharding."""
    import torch
    import torch.distributed as dist

    from paper_2307_08771_b200.driver import ReplicaDriver

    out = {}
    rank = dist.get_rank() if world > 1 else 0
    if rank == 0:
        up = b1_latency(make, dev, args.steps, args.gather)
        out["b1_latency_ms"] = up["ms"]
        out["b1_roofline_ms"] = up["roofline_ms"]
        out["b1_launches"] = up["launches"]
        if args.strategy == "reorder":
            out["b1_baseline_export_ms"] = b1_latency(make, dev, args.steps, "copy", strategy="baseline")["ms"]
    if rank == 0 and args.strategy == "reorder" and args.config == "resnet50_s50" and world == 1:
        out["configs"] = config_legs(args.steps)
    if args.strategy == "reorder":
        res = {}
        for label, gather in (("copy", "copy"), ("fused", "fused")):
            beng = make(b, dev, strategy="baseline", gather=gather)
            beng.input_buf.copy_(torch.randn(b, 3, 224, 224, generator=torch.Generator().manual_seed(1)).to(dev))
            bms = time_sharded(beng, ReplicaDriver(global_batch=G), args.steps, 3, world, dev, True)
            res[label] = {"value": round(G / (bms / 1e3), 2), "ms_per_step": round(bms, 4),
                          "launches_per_step": beng.n_launches, "upscale_speedup": round(bms / ms, 4)}
            del beng
        out["baseline_export_gpu"] = {
            **res["copy"], "unit": UNIT,
            "what": "reference baseline export (plan_baseline: identity layout, a GATHER before every partially "
                    "pruned reader) run copy-then-conv: every GATHER materialised by the vectorised channel-gather "
                    "kernel, then the same conv kernels",
            "fused_reads": res["fused"]}
    return out


def config_legs(steps: int) -> dict:
    """BASELINE.json configs 2 and 4 beside the headline: the MobileNetV3-Small batch-1
    latency sweep and DenseNet-121 @ 50 % at batch 128, each as UPSCALE (reorder) vs the
    baseline export run copy-then-conv (tools/sweep.py has the full sweep incl. config 5)."""
    import importlib.util

    spec = importlib.util.spec_from_file_location("sweep", ROOT / "tools" / "sweep.py")
    sw = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(sw)
    from paper_2307_08771_b200.configs import CONFIGS, MOBILENET_SWEEP, build_spatial_model

    out = {"mobilenet_v3_small_b1": [], "densenet121_s50_b128": None}
    for s_ in MOBILENET_SWEEP:
        name = f"mobilenet_v3_small_s{round(s_ * 100):02d}"
        cfg = CONFIGS[name]
        sm = build_spatial_model(cfg)
        up = sw.time_engine(sm, cfg, "reorder", "fused", 1, max(steps, 50))
        base = sw.time_engine(sm, cfg, "baseline", "copy", 1, max(steps, 50))
        out["mobilenet_v3_small_b1"].append({"sparsity": s_, "upscale_ms": up["ms"], "baseline_copy_ms": base["ms"],
                                             "upscale_speedup": round(base["ms"] / up["ms"], 4),
                                             "launches": [up["launches"], base["launches"]]})
    cfg = CONFIGS["densenet121_s50"]
    sm = build_spatial_model(cfg)
    up = sw.time_engine(sm, cfg, "reorder", "fused", cfg.batch, steps)
    base = sw.time_engine(sm, cfg, "baseline", "copy", cfg.batch, steps)
    out["densenet121_s50_b128"] = {"upscale": up, "baseline_copy": base,
                                   "upscale_speedup": round(base["ms"] / up["ms"], 4)}
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="resnet50_s50")
    ap.add_argument("--strategy", default="reorder")
    ap.add_argument("--gather", default="fused", choices=["fused", "copy"])
    ap.add_argument("--batch", type=int, default=256, help="GLOBAL batch per step (sharded over the GPUs)")
    ap.add_argument("--ref-images", type=int, default=32, help="--impl reference: images per step")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-extras", action="store_true", help="skip the b1 latency / baseline-export legs")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        sys.exit(self_launch(args))
    if args.impl == "reference":
        return run_reference(args)
    run_ours(args)
    import torch.distributed as dist

    if dist.is_initialized():
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
