"""Batch-1 forward latency (CUDA-graph replay, median of events) for PDL on/off (dev tool)."""
import statistics
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2307_08771_b200 import engine as EN, export as E, plans as P  # noqa: E402
from paper_2307_08771_b200.configs import CONFIGS, build_spatial_model  # noqa: E402


def main():
    cfg = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "resnet50_s50"]
    N = int(sys.argv[2]) if len(sys.argv) > 2 else 1
    sm = build_spatial_model(cfg)
    plans = P.load_plans(cfg.asset_dir / "plans_reorder.json")
    eg = E.export_graph(sm.graph, plans)
    eng = EN.from_plans(sm, eg, E.compose_maps(sm.graph, plans), batch=N)
    eng.input_buf.copy_(torch.randn(N, 3, 224, 224))
    eng.capture()
    for _ in range(20):
        eng.replay()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    lat = []
    for _ in range(50):
        a.record()
        eng.replay()
        b.record()
        b.synchronize()
        lat.append(a.elapsed_time(b))
    print(f"batch {N}: median {statistics.median(lat) * 1e3:.1f} us, min {min(lat) * 1e3:.1f} us")


if __name__ == "__main__":
    main()
