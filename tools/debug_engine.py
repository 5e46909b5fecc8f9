"""Compare every engine value against the oracle's intermediate (dev tool)."""
import sys
from pathlib import Path
import torch
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from oracle.apply_plan_ref import apply_plans_spatial  # noqa: E402
from oracle.spatial_ref import run_spatial  # noqa: E402
from paper_2307_08771_b200 import engine as EN, export as E, plans as P  # noqa: E402
from paper_2307_08771_b200.configs import CONFIGS, build_spatial_model  # noqa: E402

cfg = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "resnet18_s50"]
strategy = sys.argv[2] if len(sys.argv) > 2 else "reorder"
gm = sys.argv[3] if len(sys.argv) > 3 else "fused"
N = int(sys.argv[4]) if len(sys.argv) > 4 else 4
sm = build_spatial_model(cfg, randomize_bn=True)
plans = P.load_plans(cfg.asset_dir / f"plans_{strategy}.json")
eg = E.export_graph(sm.graph, plans)
maps = E.compose_maps(sm.graph, plans)
x = torch.randn(N, 3, 224, 224, generator=torch.Generator().manual_seed(0))
eng = EN.from_plans(sm, eg, maps, batch=N, gather_mode=gm)
eng.forward(x.cuda())
torch.cuda.synchronize()
w, v = apply_plans_spatial(plans, sm.graph, sm.weights, sm.vectors)
vals = {}
run_spatial(eg, sm.specs, w, v, x, dtype=torch.float32, values=vals)
for op in eng.ops:
    a = eng._value(op.output)
    got = a.to_nchw().cpu() if a.H * a.W > 1 or a.buf.dtype == torch.bfloat16 else a.buf[:, :a.C].float().cpu()
    ref = vals[op.output]
    if ref.dim() == 2:
        ref = ref[:, :, None, None]
    got = got.reshape(ref.shape)
    err = float((got - ref).abs().max() / ref.abs().max().clamp_min(1e-6))
    print(f"{op.kind:8s} {op.output:28s} {tuple(ref.shape)} err {err:.2e} {'<<<' if err > 2e-2 else ''}"
          f" {op.info.get('read')} {eng.graph.layer(op.info['read']).params[:8] if op.info.get('read') else ''}")
