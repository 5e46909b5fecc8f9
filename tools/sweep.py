#!/usr/bin/env python
"""Config sweep on one B200 (BASELINE.json configs 2, 4, 5): UPSCALE (reorder) export vs
the baseline (copy-then-conv) export, same engine, device-timed.

    python tools/sweep.py [--set mobilenet|densenet|config5|all] [--out profiles/r2_sweep.json]

* mobilenet: MobileNetV3-Small at 10/30/50/70/90/95 % -- batch-1 latency (median of
  per-replay CUDA events, graph replay), the paper's Fig. 1 / Table A.7 regime.
* densenet : DenseNet-121 @ 50 %, batch 128 throughput.
* config5  : EfficientNetV2-S and ResNet-101 at 30/50/70 %, batch 256 throughput.
Each line carries the step roofline (SURVEY.md 8d formulas over the exported graph) and
its fraction.  Inputs larger than L2 at batch >= 128; batch 1 is latency (L2-resident).
"""

from __future__ import annotations

import argparse
import json
import statistics
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import torch  # noqa: E402

from paper_2307_08771_b200 import engine as EN, export as E, plans as P  # noqa: E402
from paper_2307_08771_b200.configs import CONFIGS, MOBILENET_SWEEP, build_spatial_model  # noqa: E402


def peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        return json.loads(p.read_text())
    return {"hbm_gbs": 6650.0, "bf16_tflops_sustained": 1400.0}


def roofline_ms(eng, batch):
    pk = peaks()
    hbm, tc = pk["hbm_gbs"] * 1e9, pk["bf16_tflops_sustained"] * 1e12
    return sum(max(s.flops * batch / tc, (s.bytes + s.gather_bytes) * batch / hbm) for s in eng.conv_stats) * 1e3


def time_engine(sm, cfg, strategy, gather, batch, steps):
    plans = P.load_plans(cfg.asset_dir / f"plans_{strategy}.json")
    eg = E.export_graph(sm.graph, plans)
    eng = EN.from_plans(sm, eg, E.compose_maps(sm.graph, plans), batch=batch, gather_mode=gather)
    eng.capture()
    x = torch.randn(batch, 3, 224, 224, generator=torch.Generator().manual_seed(0))
    eng.input_buf.copy_(x.cuda())
    for _ in range(5):
        eng.replay(0)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if batch == 1:
        lat = []
        for _ in range(steps):
            a.record()
            eng.replay(0)
            b.record()
            b.synchronize()
            lat.append(a.elapsed_time(b))
        ms = statistics.median(lat)
    else:
        a.record()
        for _ in range(steps):
            eng.replay(0)
        b.record()
        torch.cuda.synchronize()
        ms = a.elapsed_time(b) / steps
    roof = roofline_ms(eng, batch)
    out = {"ms": round(ms, 4), "images_per_s": round(batch / (ms / 1e3), 1), "roofline_ms": round(roof, 4),
           "roofline_frac": round(roof / ms, 4), "launches": eng.n_launches,
           "copied_reads": P.copy_report(plans).copied, "total_reads": P.copy_report(plans).total_reads}
    del eng
    torch.cuda.empty_cache()
    return out


def run(names, batch_of, steps, out_lines):
    for name in names:
        cfg = CONFIGS[name]
        sm = build_spatial_model(cfg)
        batch = batch_of(cfg)
        t0 = time.time()
        up = time_engine(sm, cfg, "reorder", "fused", batch, steps)
        base = time_engine(sm, cfg, "baseline", "copy", batch, steps)
        rec = {"config": name, "model": cfg.model, "sparsity": cfg.sparsity, "batch": batch,
               "upscale": up, "baseline_copy": base, "upscale_speedup": round(base["ms"] / up["ms"], 4),
               "wall_s": round(time.time() - t0, 1)}
        print(json.dumps(rec), flush=True)
        out_lines.append(rec)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--set", default="all", choices=["mobilenet", "densenet", "config5", "all"])
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    lines = []
    if args.set in ("mobilenet", "all"):
        run([f"mobilenet_v3_small_s{round(s * 100):02d}" for s in MOBILENET_SWEEP], lambda c: 1, max(args.steps, 50),
            lines)
    if args.set in ("densenet", "all"):
        run(["densenet121_s50"], lambda c: c.batch, args.steps, lines)
    if args.set in ("config5", "all"):
        run(["resnet101_s30", "resnet101_s50", "resnet101_s70", "efficientnet_v2_s_s30", "efficientnet_v2_s_s50",
             "efficientnet_v2_s_s70"], lambda c: c.batch, args.steps, lines)
    if args.out:
        Path(args.out).write_text(json.dumps(lines, indent=1) + "\n")


if __name__ == "__main__":
    main()
