"""Export artifact round trip: graph, plans, specs and every exported
tensor come back bit-identical; runs on CPU (the permute kernels are stubbed by a torch
restatement here -- the artifact code is device-agnostic)."""

import torch

from paper_2307_08771_b200 import artifact, export as E, ir, plans as P
from paper_2307_08771_b200.configs import CONFIGS, build_spatial_model


def _cpu_export(sm, plans):
    """ExportResult with weights permuted by plain torch indexing (no GPU here)."""
    maps = E.compose_maps(sm.graph, plans)
    ew = E.ExportedWeights()
    for lid, w in sm.weights.items():
        rows = torch.tensor(list(maps.rows.get(lid, range(w.shape[0]))))
        cols = torch.tensor(list(maps.cols.get(lid, range(w.shape[1]))))
        out = w[rows.clamp_min(0)][:, cols.clamp_min(0)].clone()
        out[rows < 0] = 0
        out[:, cols < 0] = 0
        ew.mix[lid] = out.to(torch.bfloat16) if lid.endswith("conv1") else out
    for uid, named in sm.vectors.items():
        perm = maps.vec.get(uid)
        ew.vec[uid] = {k: (v[list(perm)] if perm is not None else v.clone()).double() for k, v in named.items()}
    return E.ExportResult(E.export_graph(sm.graph, plans), ew, tuple(plans), P.copy_report(plans), ("x",))


def test_export_artifact_round_trip(tmp_path):
    cfg = CONFIGS["resnet18_s50"]
    sm = build_spatial_model(cfg)
    plans = P.load_plans(cfg.asset_dir / "plans_reorder.json")
    res = _cpu_export(sm, plans)
    artifact.save_export(res, sm, tmp_path / "r18")
    back, model = artifact.load_export(tmp_path / "r18", device="cpu")
    assert ir.graph_to_dict(back.graph) == ir.graph_to_dict(res.graph)
    assert [P.plan_to_dict(p) for p in back.plans] == [P.plan_to_dict(p) for p in res.plans]
    assert back.totals == res.totals and back.fallbacks == res.fallbacks
    assert set(back.weights.mix) == set(res.weights.mix)
    for lid, t in res.weights.mix.items():
        assert back.weights.mix[lid].dtype == t.dtype and torch.equal(back.weights.mix[lid], t)
    for uid, named in res.weights.vec.items():
        for k, t in named.items():
            assert torch.equal(back.weights.vec[uid][k], t)
    assert model.input_chw == sm.input_chw
    for lid in (l.id for l in res.graph.layers):
        if lid in sm.specs:
            assert model.specs[lid] == sm.specs[lid]
