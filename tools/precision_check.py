"""bf16 drift of the GPU engine vs the fp32 oracle, next to the drift of a bf16 CPU run of the
same oracle graph and of two GPU variants against each other (dev tool)."""
import sys, torch
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from oracle.apply_plan_ref import apply_plans_spatial
from oracle.spatial_ref import deviation, run_spatial, top1_agreement
from paper_2307_08771_b200 import engine as EN, export as E, plans as P
from paper_2307_08771_b200.configs import CONFIGS, build_spatial_model
for name in ["resnet50_s50", "resnet101_s50"]:
    cfg = CONFIGS[name]
    sm = build_spatial_model(cfg, randomize_bn=True)
    plans = P.load_plans(cfg.asset_dir / "plans_reorder.json")
    eg = E.export_graph(sm.graph, plans)
    maps = E.compose_maps(sm.graph, plans)
    x = torch.randn(2, 3, 224, 224, generator=torch.Generator().manual_seed(3))
    got = EN.from_plans(sm, eg, maps, batch=2).forward(x.cuda()).cpu()
    got_copy = EN.from_plans(sm, eg, maps, batch=2, gather_mode="copy", stem_s2d=False).forward(x.cuda()).cpu()
    w, v = apply_plans_spatial(plans, sm.graph, sm.weights, sm.vectors)
    ref = run_spatial(eg, sm.specs, w, v, x, dtype=torch.float32)
    ref16 = run_spatial(eg, sm.specs, w, v, x, dtype=torch.bfloat16).float()
    print(name, "gpu-vs-fp32", deviation(got, ref), "gpu-vs-gpu(copy,im2col stem)", deviation(got, got_copy),
          "bf16oracle-vs-fp32", deviation(ref16, ref), "gpu-vs-bf16oracle", deviation(got, ref16),
          "top1", top1_agreement(got, ref), "logit absmax", float(ref.abs().max()))
