"""Generate the committed per-config assets with the REFERENCE planner.

Run in the build container (where /root/reference exists):
    python tools/make_assets.py [config ...]

For each pinned config (paper_2307_08771_b200/configs.py) this script
  1. lowers the seeded torchvision model to the reference IR (our lowering),
  2. converts it to a live `reslice.ModelGraph` + float64 `WeightStore`,
  3. calls the reference's own `score_channels` / `make_masks` /
     `plan_model` / `export_model` (pipeline.py:99-146) for the `reorder`
     (UPSCALE) and `baseline` strategies,
  4. writes graph.json, masks.json, plans_<strategy>.json, export_<strategy>.json
     (the exported IR graph) and meta.json (timings, copy stats and a sha256 of
     every exported proxy tensor, which pins our apply_plan restatement).
Nothing here runs on the GPU hosts; they read the committed files.
"""

from __future__ import annotations

import hashlib
import json
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402

from paper_2307_08771_b200.ref import reslice  # noqa: E402

ref_graph_from_dict = reslice.graph.graph_from_dict
ref_plan_to_dict = reslice.planner.plan_to_dict

from paper_2307_08771_b200 import ir  # noqa: E402
from paper_2307_08771_b200.configs import CONFIGS, build_spatial_model  # noqa: E402


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.float64).tobytes()).hexdigest()[:16]


def make(name: str) -> None:
    cfg = CONFIGS[name]
    out = cfg.asset_dir
    out.mkdir(parents=True, exist_ok=True)
    sm = build_spatial_model(cfg)
    g_ref = ref_graph_from_dict(ir.graph_to_dict(sm.graph))
    diags = reslice.graph.validate(g_ref)
    assert not diags, diags
    store = reslice.WeightStore()
    for lid, arr in sm.proxy_weights().items():
        store[lid] = arr
    assert not reslice.graph.validate(g_ref, store)

    if cfg.native_planner:  # reference plan_model, native decompose/order core
        from paper_2307_08771_b200 import native_planner
        native_planner.install(reslice)
    t0 = time.time()
    scores = reslice.score_channels(g_ref, store.tensors, cfg.heuristic, side="input")
    masks = reslice.make_masks(g_ref, scores, cfg.sparsity, "unconstrained",
                               reslice.find_segments(g_ref), scope=cfg.scope)
    t_masks = time.time() - t0
    ir.save_graph(sm.graph, out / "graph.json", compact=True)
    ir.save_masks(masks, out / "masks.json", compact=True)
    meta = {"config": cfg.__dict__, "mask_seconds": round(t_masks, 3), "strategies": {},
            "proxy_sha256": {lid: sha(a) for lid, a in sorted(store.tensors.items())}}
    for strategy in ("reorder", "baseline"):
        t0 = time.time()
        plans, fallbacks = reslice.plan_model(g_ref, masks, "input", strategy, "baseline")
        t_plan = time.time() - t0
        t0 = time.time()
        res = reslice.export_model(g_ref, store, masks, "input", strategy, "baseline")
        t_export = time.time() - t0
        ir.dump_json({"version": 1, "segments": [ref_plan_to_dict(p) for p in sorted(plans, key=lambda p: p.segment)],
                      "totals": {"total_reads": res.totals.total_reads, "copied": res.totals.copied,
                                 "zero_copy_optimal": res.totals.zero_copy_optimal}},
                     out / f"plans_{strategy}.json", compact=True)
        ir.dump_json(reslice.graph.graph_to_dict(res.graph), out / f"export_{strategy}.json", compact=True)
        kinds = {}
        for lay in res.graph.layers:
            kinds[lay.kind.value] = kinds.get(lay.kind.value, 0) + 1
        meta["strategies"][strategy] = {
            "plan_seconds": round(t_plan, 3), "export_seconds": round(t_export, 3),
            "n_plans": len(plans), "fallbacks": list(fallbacks),
            "total_reads": res.totals.total_reads, "copied": res.totals.copied,
            "exported_kinds": kinds,
            "exported_sha256": {lid: sha(a) for lid, a in sorted(res.weights.tensors.items())},
        }
        print(f"{name} {strategy}: {len(plans)} plans, copied {res.totals.copied}/{res.totals.total_reads}, "
              f"plan {t_plan:.1f}s export {t_export:.1f}s, kinds {kinds}", flush=True)
    meta["native_planner"] = cfg.native_planner
    if cfg.native_planner:
        from paper_2307_08771_b200 import native_planner
        native_planner.uninstall()
    (out / "meta.json").write_text(json.dumps(meta, indent=1, sort_keys=True) + "\n")


if __name__ == "__main__":
    for n in sys.argv[1:] or ["resnet18_s50", "resnet50_s50"]:
        make(n)
