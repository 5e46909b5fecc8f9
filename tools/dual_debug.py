"""Find consumers whose dual-store read plan disagrees with their cover/gather plan (dev tool)."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2307_08771_b200 import engine as EN, export as E, plans as P  # noqa: E402
from paper_2307_08771_b200.configs import CONFIGS, build_spatial_model  # noqa: E402

cfg = CONFIGS["resnet50_s50"]
sm = build_spatial_model(cfg)
plans = P.load_plans(cfg.asset_dir / "plans_reorder.json")
eg = E.export_graph(sm.graph, plans)
maps = E.compose_maps(sm.graph, plans)
eng = EN.from_plans(sm, eg, maps, batch=2)
eng.input_buf.copy_(torch.randn(2, 3, 224, 224))
eng.launch_all()
torch.cuda.synchronize()
for op in (eng.ops if "--plans" in sys.argv else []):
    if op.kind != "conv" or "plans" not in op.info or "dual" not in op.info["plans"]:
        continue
    outs = {}
    for pi, name in enumerate(op.info["plans"]):
        for v in (0, 1, 33, 65):
            op.info["variant"] = (pi, v)
            try:
                op.launch()
            except Exception as e:  # noqa: BLE001
                outs[(name, v)] = str(e)[:60]
                continue
            torch.cuda.synchronize()
            y = eng.values[op.output] if op.output in eng.values else None
            outs[(name, v)] = y.buf.float().clone() if y is not None else None
    ref = outs[("cover", 65)] if ("cover", 65) in outs and torch.is_tensor(outs[("cover", 65)]) else None
    line = []
    for k, t in outs.items():
        if torch.is_tensor(t) and ref is not None:
            line.append(f"{k[0]}/{k[1]}: {float((t - ref).abs().max()):.3g}")
        else:
            line.append(f"{k[0]}/{k[1]}: {t if not torch.is_tensor(t) else 'ok'}")
    print(op.info["conv"], op.info.get("desc", ""), "\n   ", "; ".join(line))

print("--- compact buffers vs their producers' outputs")
eng.launch_all()
torch.cuda.synchronize()
for vid, (comp, chans) in eng._dual_bufs.items():
    y = eng.values[vid]
    prod = [op for op in eng.ops if op.kind == "conv" and op.info.get("out") == vid]
    want = y.buf[:, [y.coff + c for c in chans]].float()
    got = comp.buf[:, :len(chans)].float()
    bad = (want != got)
    print(vid, "producers", [(p.info["conv"], p.info.get("variant"), p.info.get("desc")) for p in prod],
          "y", (y.cstride, y.coff, y.C), "bad", int(bad.sum()), "of", bad.numel(),
          "bad rows", bad.any(1).nonzero()[:3].flatten().tolist(), "bad cols", bad.any(0).nonzero()[:6].flatten().tolist())

print("--- buffer sharing")
ptrs = {}
for vid, a in eng.values.items():
    ptrs.setdefault(a.buf.data_ptr(), []).append((vid, a.coff, a.C))
for pt, lst in ptrs.items():
    if len(lst) > 1 or any("#compact" in v for v, _, _ in lst):
        print(hex(pt), lst)
import collections
for vid, (comp, chans) in eng._dual_bufs.items():
    y = eng.values[vid]
    lo, hi = comp.buf.data_ptr(), comp.buf.data_ptr() + comp.buf.numel() * 2
    for v2, a in eng.values.items():
        b0, b1 = a.buf.data_ptr(), a.buf.data_ptr() + a.buf.numel() * 2
        if a is not comp and b0 < hi and lo < b1:
            print("OVERLAP", vid, "compact with", v2)

print("--- bad channel detail")
for vid, (comp, chans) in eng._dual_bufs.items():
    y = eng.values[vid]
    want = y.buf[:, [y.coff + c for c in chans]].float()
    got = comp.buf[:, :len(chans)].float()
    bad = (want != got).any(0).nonzero().flatten().tolist()
    if bad:
        print(vid, "bad chans", [chans[k] for k in bad][:40], "cout", y.C)
        k = bad[0]
        print("   row0..3 got", got[:4, k].tolist(), "want", want[:4, k].tolist())
