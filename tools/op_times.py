#!/usr/bin/env python
"""Per-op device time (CUDA events around each op's launches, eager, after warm-up) next to
its algorithmic roofline, for one config: python tools/op_times.py <config> [batch] [strategy] [gather]"""
import json
import sys
from collections import defaultdict
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2307_08771_b200 import engine as EN, export as E, plans as P  # noqa: E402
from paper_2307_08771_b200.configs import CONFIGS, build_spatial_model  # noqa: E402

name = sys.argv[1]
cfg = CONFIGS[name]
batch = int(sys.argv[2]) if len(sys.argv) > 2 else max(cfg.batch, 1)
strategy = sys.argv[3] if len(sys.argv) > 3 else "reorder"
gather = sys.argv[4] if len(sys.argv) > 4 else "fused"
sm = build_spatial_model(cfg)
plans = P.load_plans(cfg.asset_dir / f"plans_{strategy}.json")
eg = E.export_graph(sm.graph, plans)
eng = EN.from_plans(sm, eg, E.compose_maps(sm.graph, plans), batch=batch, gather_mode=gather)
eng.capture()
eng.input_buf.copy_(torch.randn(batch, 3, 224, 224, generator=torch.Generator().manual_seed(0)).cuda())
rows, total = bench.kernel_table(eng, batch, bench.peaks())
by_kernel = defaultdict(lambda: [0, 0.0, 0.0])
for r in rows:
    k = by_kernel[r["kernel"]]
    k[0] += 1
    k[1] += r["us"]
    k[2] += r["roofline_us"]
print(json.dumps({"config": name, "batch": batch, "strategy": strategy, "eager_sum_us": round(total * 1e3, 1),
                  "by_kernel": {k: {"launches": v[0], "us": round(v[1], 1), "roofline_us": round(v[2], 1)}
                                for k, v in sorted(by_kernel.items(), key=lambda kv: -kv[1][1])}}))

def t_us(fn, reps=10):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps * 1e3


for r in sorted(rows, key=lambda r: -r["us"])[:int(sys.argv[5]) if len(sys.argv) > 5 else 25]:
    op = next(o for o in eng.ops if o.info.get("conv", o.output) == r["op"])
    extra = {}
    pre = op.info.get("read_pre")
    if pre and op.info.get("variant"):
        fn = pre[op.info["variant"][0]]
        if fn is not None:
            extra["read_us"] = round(t_us(fn), 1)
    print(json.dumps({**r, "desc": op.info.get("desc", ""), "variant": op.info.get("variant"), **extra}))
