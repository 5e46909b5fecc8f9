#!/usr/bin/env python
"""Run an engine's ops one at a time with a device sync after each (CUDA_LAUNCH_BLOCKING
style) and compare every op's output with the oracle's value of the same node: finds the
first op that faults or diverges.  python tools/op_check.py <config> [strategy] [batch]"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from oracle.apply_plan_ref import apply_plans_spatial  # noqa: E402
from oracle.spatial_ref import run_spatial  # noqa: E402
from paper_2307_08771_b200 import engine as EN, export as E, plans as P  # noqa: E402
from paper_2307_08771_b200.configs import CONFIGS, build_spatial_model  # noqa: E402

name = sys.argv[1]
strategy = sys.argv[2] if len(sys.argv) > 2 else "reorder"
N = int(sys.argv[3]) if len(sys.argv) > 3 else 2
cfg = CONFIGS[name]
sm = build_spatial_model(cfg, randomize_bn=True)
plans = P.load_plans(cfg.asset_dir / f"plans_{strategy}.json")
eg = E.export_graph(sm.graph, plans)
eng = EN.from_plans(sm, eg, E.compose_maps(sm.graph, plans), batch=N)
x = torch.randn(N, 3, 224, 224, generator=torch.Generator().manual_seed(6))
w, v = apply_plans_spatial(plans, sm.graph, sm.weights, sm.vectors)
vals = {}
run_spatial(eg, sm.specs, w, v, x, dtype=torch.float32, values=vals)
eng.input_buf.copy_(x.cuda())
torch.cuda.synchronize()
for i, op in enumerate(eng.ops):
    try:
        op.launch()
        torch.cuda.synchronize()
    except Exception as exc:
        print(f"FAULT at op {i} {op.kind} {op.anchor} -> {op.output}: {exc}")
        raise
    if op.output in vals:
        got = eng._value(op.output).to_nchw().cpu()
        ref = vals[op.output].float()
        if ref.dim() == 2:
            ref = ref[:, :, None, None]
        err = float((got - ref).abs().max() / ref.abs().max().clamp_min(1e-6))
        flag = "  <<<" if err > 2e-2 else ""
        print(f"{i:3d} {op.kind:9s} {op.output:40s} {tuple(got.shape)} rel {err:.2e}{flag}", flush=True)
