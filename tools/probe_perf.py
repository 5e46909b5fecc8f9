"""Per-op timing probe for the engine (development tool, not the bench).

python tools/probe_perf.py [config] [batch] [strategy] [gather_mode]
Prints whole-forward time (CUDA graph replay) and a per-op table (events
around each launch, eager) with algorithmic bytes/FLOPs and roofline times.
"""

import json
import os
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2307_08771_b200 import engine as EN, export as E, plans as P  # noqa: E402
from paper_2307_08771_b200.configs import CONFIGS, build_spatial_model  # noqa: E402

PEAKS = {"hbm": 6554.6e9, "tc": 1398.9e12}


def main():
    cfg = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "resnet50_s50"]
    N = int(sys.argv[2]) if len(sys.argv) > 2 else 256
    strategy = sys.argv[3] if len(sys.argv) > 3 else "reorder"
    gm = sys.argv[4] if len(sys.argv) > 4 else "fused"
    sm = build_spatial_model(cfg)
    plans = P.load_plans(cfg.asset_dir / f"plans_{strategy}.json")
    eg = E.export_graph(sm.graph, plans)
    maps = E.compose_maps(sm.graph, plans)
    opts = {}
    for kv in os.environ.get("UB_ENGINE_OPTS", "").split(","):
        if "=" in kv:
            k, v = kv.split("=")
            opts[k] = v == "1"
    eng = EN.from_plans(sm, eg, maps, batch=N, gather_mode=gm, **opts)
    x = torch.randn(N, 3, 224, 224, device="cuda")
    eng.input_buf.copy_(x)
    # per-op eager timing
    for _ in range(3):
        eng.launch_all()
    torch.cuda.synchronize()
    eng.autotune()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in eng.ops]
    reps = 5
    times = [0.0] * len(eng.ops)
    for _ in range(reps):
        for op, (a, b) in zip(eng.ops, evs):
            a.record()
            op.launch()
            b.record()
        torch.cuda.synchronize()
        for i, (a, b) in enumerate(evs):
            times[i] += a.elapsed_time(b) / reps
    stats = {s.name: s for s in eng.conv_stats}
    rows = []
    for op, t in zip(eng.ops, times):
        name = op.info.get("conv", op.output)
        st = stats.get(name)
        if st is None and op.kind == "gather":
            st = stats.get(f"{op.output}(copy)")
        f = st.flops * N if st else 0.0
        b = (st.bytes + st.gather_bytes) * N if st else 0.0
        troof = max(f / PEAKS["tc"], b / PEAKS["hbm"]) * 1e3
        rows.append((op.kind, name, t, f / 1e9, b / 1e6, troof, op.info.get("desc", "")))
    tot = sum(r[2] for r in rows)
    troof = sum(r[5] for r in rows)
    for r in sorted(rows, key=lambda r: -r[2])[:int(sys.argv[5]) if len(sys.argv) > 5 else 25]:
        print(f"{r[0]:8s} {r[1]:24s} {r[2]*1e3:7.1f} us {r[3]:6.2f} GF {r[4]:6.1f} MB roof {r[5]*1e3:6.1f} us "
              f"frac {r[5]/max(r[2],1e-9):.2f}  {r[6]}")
    if len(sys.argv) > 6 and sys.argv[6] == "gap":
        print("--- by gap to roofline")
        for r in sorted(rows, key=lambda r: -(r[2] - r[5]))[:40]:
            print(f"{r[1]:24s} {r[2]*1e3:7.1f} us roof {r[5]*1e3:6.1f} gap {(r[2]-r[5])*1e3:6.1f}  {r[6]}")
    cats = {}
    for r in rows:
        d = r[6]
        key = r[0] if not d else (d.split()[0] + (" gather" if "gather" in d else ""))
        c = cats.setdefault(key, [0.0, 0.0, 0])
        c[0] += r[2]
        c[1] += r[5]
        c[2] += 1
    for k, (t, tr, n) in sorted(cats.items(), key=lambda kv: -kv[1][0]):
        print(f"  {k:16s} x{n:2d} {t*1e3:8.1f} us  roof {tr*1e3:7.1f} us  frac {tr/max(t,1e-9):.2f}")
    print(f"eager sum {tot:.3f} ms, roofline {troof:.3f} ms, frac {troof/tot:.3f}")
    eng.capture(autotune=False)
    for op in eng.ops:
        if "plans" in op.info and len(op.info["plans"]) > 1:
            print("  pick", op.info["conv"], op.info["plans"][op.info["variant"][0]], op.info["variant"][1])
    for _ in range(3):
        eng._graph_exec.replay()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(10):
        eng._graph_exec.replay()
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / 10
    print(json.dumps({"cfg": cfg.name, "N": N, "strategy": strategy, "gather": gm, "graph_ms": ms,
                      "img_s": N / ms * 1e3, "roof_ms": troof, "frac": troof / ms, "launches": len(eng.ops)}))


if __name__ == "__main__":
    main()
