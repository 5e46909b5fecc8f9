#!/usr/bin/env python
"""One eager forward of the bench engine inside an NVTX range "step" -- the ncu target for
the per-launch list (ncu --nvtx --nvtx-include "step/" ...).
python tools/profile_step.py [config] [batch] [passes]"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2307_08771_b200 import engine as EN, export as E, plans as P  # noqa: E402
from paper_2307_08771_b200.configs import CONFIGS, build_spatial_model  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "resnet50_s50"
batch = int(sys.argv[2]) if len(sys.argv) > 2 else 256
passes = int(sys.argv[3]) if len(sys.argv) > 3 else 1
cfg = CONFIGS[name]
sm = build_spatial_model(cfg)
plans = P.load_plans(cfg.asset_dir / "plans_reorder.json")
eg = E.export_graph(sm.graph, plans)
eng = EN.from_plans(sm, eg, E.compose_maps(sm.graph, plans), batch=batch)
eng.capture()  # autotune + graph (as bench.py); the profiled passes run eagerly
eng.input_buf.copy_(torch.randn(batch, 3, 224, 224, generator=torch.Generator().manual_seed(0)).cuda())
eng.launch_all()
torch.cuda.synchronize()
for _ in range(passes):
    torch.cuda.nvtx.range_push("step")
    eng.launch_all(nvtx=True)
    torch.cuda.nvtx.range_pop()
torch.cuda.synchronize()
print("ok", eng.n_launches, "launches per pass")
