#!/usr/bin/env python
"""Benchmark: UPSCALE-exported ResNet-50 @ 50% on B200 (BASELINE.json configs[2]).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

One step = one forward pass of the exported pruned ResNet-50 over a batch of
256 synthetic 224x224 images per GPU (weak scaling: replicas are independent;
the only exchange is an NCCL all-gather of the logits at the end of the step).
Rank 0 prints ONE JSON line.  `value` is device-timed with inputs resident in
HBM; `e2e` goes through the public API with pinned host input, H2D + D2H in
the timed region.  `--impl reference` times the reference's CPU path (the
oracle port of interp.run over the same exported graph) on the host cores.
"""

from __future__ import annotations

import argparse
import json
import os
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
                 "-lms", "100"], stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
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
def cpu_reference_sample(cfg_name: str, strategy: str, n_images: int, budget_s: float, seed: int = 0):
    """The reference's CPU path: the oracle port of interp.run (spatial ops, torch
    fp32, all host threads) over the SAME exported graph.  Returns images/s."""
    import torch

    from oracle.apply_plan_ref import apply_plans_spatial
    from oracle.spatial_ref import run_spatial
    from paper_2307_08771_b200 import export as E, plans as P
    from paper_2307_08771_b200.configs import CONFIGS, build_spatial_model

    torch.set_num_threads(os.cpu_count() or 1)
    cfg = CONFIGS[cfg_name]
    sm = build_spatial_model(cfg)
    plans = P.load_plans(cfg.asset_dir / f"plans_{strategy}.json")
    eg = E.export_graph(sm.graph, plans)
    w, v = apply_plans_spatial(plans, sm.graph, sm.weights, sm.vectors)
    w = {k: t.float() for k, t in w.items()}
    x = torch.randn(n_images, 3, 224, 224, generator=torch.Generator().manual_seed(seed))
    with torch.no_grad():
        run_spatial(eg, sm.specs, w, v, x[:1], dtype=torch.float32)  # warm-up
        times = []
        t_start = time.perf_counter()
        while True:
            t0 = time.perf_counter()
            run_spatial(eg, sm.specs, w, v, x, dtype=torch.float32)
            times.append(time.perf_counter() - t0)
            if time.perf_counter() - t_start > budget_s or len(times) >= 5:
                break
    t = statistics.median(times)
    return {"value": n_images / t, "unit": UNIT, "cores": torch.get_num_threads(), "kind": "port",
            "sample": f"{n_images} images x {len(times)} runs of oracle/spatial_ref.py (fp32 torch CPU) over "
                      f"the {strategy} export of {cfg_name}; median {t:.2f} s"}


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import torch

    torch.set_num_threads(os.cpu_count() or 1)
    from oracle.apply_plan_ref import apply_plans_spatial
    from oracle.spatial_ref import run_spatial
    from paper_2307_08771_b200 import export as E, plans as P
    from paper_2307_08771_b200.configs import CONFIGS, build_spatial_model

    cfg = CONFIGS[args.config]
    sm = build_spatial_model(cfg)
    plans = P.load_plans(cfg.asset_dir / f"plans_{args.strategy}.json")
    eg = E.export_graph(sm.graph, plans)
    w, v = apply_plans_spatial(plans, sm.graph, sm.weights, sm.vectors)
    w = {k: t.float() for k, t in w.items()}
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
    line = {"impl": "reference", "metric": METRIC, "value": val, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt * 1e3, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": f"{args.config} ({args.strategy} export), CPU sample of {n} images per step",
                       "global_batch": n, "image": [3, 224, 224]},
            "cpu_baseline": {"value": val, "unit": UNIT, "cores": torch.get_num_threads(), "kind": "port",
                             "sample": f"{n} images per step, oracle/spatial_ref.py fp32 torch CPU"},
            "e2e": {"value": val, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# --------------------------------------------------------------------------- GPU path
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="resnet50_s50")
    ap.add_argument("--strategy", default="reorder")
    ap.add_argument("--gather", default="fused", choices=["fused", "copy"])
    ap.add_argument("--batch", type=int, default=256, help="images per GPU per step")
    ap.add_argument("--ref-images", type=int, default=4, help="--impl reference: images per step")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-extras", action="store_true", help="skip b1 latency / baseline-export / e2e legs")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    if args.impl == "reference":
        return run_reference(args)

    import torch
    import torch.distributed as dist

    from paper_2307_08771_b200 import _lib, api, engine as EN, export as E, plans as P
    from paper_2307_08771_b200.configs import CONFIGS, build_spatial_model
    from paper_2307_08771_b200.driver import ReplicaDriver

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)

    cfg = CONFIGS[args.config]
    B = args.batch
    sm = build_spatial_model(cfg)
    plans = P.load_plans(cfg.asset_dir / f"plans_{args.strategy}.json")
    eg = E.export_graph(sm.graph, plans)
    maps = E.compose_maps(sm.graph, plans)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    eng = EN.from_plans(sm, eg, maps, batch=B, device=dev, gather_mode=args.gather)
    torch.cuda.synchronize()
    export_s = time.perf_counter() - t0
    eng.capture()
    x = torch.randn(B, 3, 224, 224, generator=torch.Generator().manual_seed(rank)).to(dev)
    eng.input_buf.copy_(x)
    logits = eng.output_tensor()
    driver = ReplicaDriver(lambda: eng.output_tensor(), equal_shards=True)
    stream = torch.cuda.current_stream()

    def step():
        eng._graph_exec.replay()
        if world > 1:
            driver.gather(driver.run_local())  # the one exchange: NCCL all-gather of the logits

    def barrier():
        if world > 1:
            dist.barrier()

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    clocks = ClockSampler(local)
    clocks.start()
    time.sleep(0.3)
    barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        step()
    e1.record(stream)
    torch.cuda.synchronize()
    barrier()
    ms = e0.elapsed_time(e1) / args.steps
    clk = clocks.stop()
    if world > 1:
        t = torch.tensor([ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    value = world * B / (ms / 1e3)
    launches_per_step = eng.n_launches

    # ---- per-kernel roofline of the dominant kernel family (conv), eager + events
    pk = peaks()
    conv_ops = [op for op in eng.ops if op.kind == "conv"]
    stats = {s.name: s for s in eng.conv_stats}
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in eng.ops]
    per_op = [0.0] * len(eng.ops)
    reps = 3
    for _ in range(reps):
        for op, (a, b) in zip(eng.ops, evs):
            a.record(stream)
            op.launch()
            b.record(stream)
        torch.cuda.synchronize()
        for i, (a, b) in enumerate(evs):
            per_op[i] += a.elapsed_time(b) / reps
    conv_ms = sum(t for op, t in zip(eng.ops, per_op) if op.kind == "conv")
    eager_ms = sum(per_op)
    conv_bytes = sum(stats[op.info["conv"]].bytes * B for op in conv_ops)
    conv_flops = sum(stats[op.info["conv"]].flops * B for op in conv_ops)
    hbm = pk["hbm_gbs"] * 1e9
    tc = pk["bf16_tflops_sustained"] * 1e12
    troof = sum(max(stats[op.info["conv"]].flops * B / tc, stats[op.info["conv"]].bytes * B / hbm)
                for op in conv_ops)
    achieved = conv_bytes / (conv_ms / 1e3) / 1e9
    traffic = None
    tfile = ROOT / "profiles" / "conv_traffic.json"
    if tfile.exists():
        try:
            traffic = json.loads(tfile.read_text()).get("dram_bytes_per_step_conv")
        except (ValueError, OSError):
            traffic = None
    roofline = {"bound": "hbm", "achieved": round(achieved, 1), "peak": pk["hbm_gbs"], "unit": "GB/s",
                "frac": round(achieved / pk["hbm_gbs"], 4), "traffic": traffic,
                "kernel": "conv kernels of one step (conv_tc, conv_halo3, stem_s2d_pack_rows + stem_pool, channel_gather_2d)",
                "algorithmic_bytes_per_step": conv_bytes, "algorithmic_flops_per_step": conv_flops,
                "conv_ms_per_step_eager": round(conv_ms, 4), "conv_share_of_step": round(conv_ms / eager_ms, 4),
                "mixed_roofline_ms": round(troof * 1e3, 4),
                "mixed_roofline_frac": round(troof * 1e3 / conv_ms, 4),
                "step_roofline_frac": round(troof * 1e3 / ms, 4),
                "peak_source": pk["source"], "tensor_peak_tflops": pk["bf16_tflops_sustained"]}

    extras = {}
    e2e = None
    if not args.no_extras and rank == 0:
        # ---- e2e through the public API: api.Runner.run(host batch) -> host logits.
        # Timed region: pinned host fp32 -> H2D, CUDA-graph forward, D2H of the logits.
        ex = api.Exported(E.ExportResult(eg, None, tuple(plans), P.copy_report(plans), ()), sm, maps)
        runner = api.Runner(ex, gather_mode=args.gather, device=dev)
        runner._engines[B] = eng
        host_x = x.cpu().pin_memory()
        for _ in runner.run_many([host_x] * 3):
            pass
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        k2 = max(10, args.steps // 2)
        a.record(stream)
        outs = 0
        for out_np in runner.run_many(host_x for _ in range(k2)):
            outs += 1
        b.record(stream)
        torch.cuda.synchronize()
        assert outs == k2
        e2e_ms = a.elapsed_time(b) / k2
        e2e = {"value": round(B / (e2e_ms / 1e3), 2), "unit": UNIT, "h2d_bytes_per_step": runner.h2d_bytes,
               "d2h_bytes_per_step": int(out_np.nbytes), "ms_per_step": round(e2e_ms, 4),
               "steps": k2,
               "path": "api.Runner.run_many: pinned host NCHW fp32 -> H2D of the channels the INPUT GATHER "
                       "keeps (copy stream, overlapped with the previous batch's forward) -> CUDA-graph "
                       "forward -> D2H logits -> host numpy, every step"}
        # ---- batch-1 latency
        eng1 = EN.from_plans(sm, eg, maps, batch=1, device=dev, gather_mode=args.gather)
        eng1.capture()
        eng1.input_buf.copy_(x[:1])
        for _ in range(10):
            eng1._graph_exec.replay()
        torch.cuda.synchronize()
        lat = []
        for _ in range(max(20, args.steps)):
            a.record(stream)
            eng1._graph_exec.replay()
            b.record(stream)
            b.synchronize()
            lat.append(a.elapsed_time(b))
        b1_roof = sum(max(s.flops / tc, s.bytes / hbm) for s in eng1.conv_stats) * 1e3
        extras["b1_latency_ms"] = round(statistics.median(lat), 4)
        extras["b1_roofline_ms"] = round(b1_roof, 5)
        del eng1
        # ---- baseline-export GPU variant (copy-then-conv), same batch
        if args.strategy == "reorder":
            bplans = P.load_plans(cfg.asset_dir / "plans_baseline.json")
            beg = E.export_graph(sm.graph, bplans)
            bmaps = E.compose_maps(sm.graph, bplans)
            beng = EN.from_plans(sm, beg, bmaps, batch=B, device=dev, gather_mode="copy")
            beng.capture()
            beng.input_buf.copy_(x)
            for _ in range(3):
                beng._graph_exec.replay()
            torch.cuda.synchronize()
            a.record(stream)
            for _ in range(args.steps):
                beng._graph_exec.replay()
            b.record(stream)
            torch.cuda.synchronize()
            bms = a.elapsed_time(b) / args.steps
            extras["baseline_export_gpu"] = {"value": B / (bms / 1e3), "unit": UNIT, "ms_per_step": round(bms, 4),
                                             "launches_per_step": beng.n_launches,
                                             "upscale_speedup": round(bms / ms, 4)}
            del beng

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_reference_sample(args.config, args.strategy, n_images=4, budget_s=20.0)

    if rank == 0:
        line = {
            "metric": METRIC, "value": round(value, 2), "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(ms, 4), "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
            "config": {"workload": f"{args.config}: UPSCALE ({args.strategy}) export of random-init torchvision "
                                   f"ResNet-50, 50% unconstrained L2 per-layer input pruning; 224x224 images",
                       "global_batch": world * B, "per_gpu_batch": B, "parallelism": f"replicas x{world}",
                       "gather_mode": args.gather,
                       "l2": "inputs larger than L2 (154 MB fp32 batch + ~GB of activations per step)"},
            "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e, "clocks": clk,
            "gpu_launches": launches_per_step * args.steps, "launches_per_step": launches_per_step,
            "export_seconds": round(export_s, 3), **extras,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
