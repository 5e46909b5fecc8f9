"""Output-mode export on the B200 path (planner.py:394-630 and apply_plan
steps 2-3, planner.py:675-729).

Output pruning drops a producer's own filters.  The reference rewrites a pruned join
only in segments without per-channel layers (planner.py:510-515), and its output-side
masks skip every other segment (masks.py:165-185) -- so BN networks export unchanged.
The coverage model is therefore a BN-free residual/concat CNN: the reorder strategy
rewrites its ADD and CONCAT joins into runs of SLICEs, partial ADDs and one CONCAT; the
baseline strategy keeps the joins and restores each pruned producer with a zero-fill
GATHER (`<p>.restore`).  The exported graphs are the reference's own (export_graph runs
reslice.apply_plan); the GPU engine runs them (slice views, eltwise adds over views,
concat bands, zero-fill gathers) against the fp32 oracle.
"""

import numpy as np
import pytest
import torch
import torch.nn as nn

from paper_2307_08771_b200 import engine as EN, export as E, kernels as K, _lib
from paper_2307_08771_b200.lowering import lower
from paper_2307_08771_b200.ref import reslice


class JoinNet(nn.Module):
    """Bias-free, BN-free: two branches joined by an add, two joined by a concat."""

    def __init__(self):
        super().__init__()
        self.stem = nn.Conv2d(3, 32, 3, stride=2, padding=1, bias=False)
        self.a = nn.Conv2d(32, 48, 3, padding=1, bias=False)
        self.b = nn.Conv2d(32, 48, 1, bias=False)
        self.c = nn.Conv2d(48, 64, 1, bias=False)
        self.d = nn.Conv2d(64, 24, 3, padding=1, bias=False)
        self.e = nn.Conv2d(64, 40, 1, bias=False)
        self.f = nn.Conv2d(64, 64, 1, bias=False)
        self.pool = nn.AdaptiveAvgPool2d(1)
        self.fc = nn.Linear(64, 10, bias=False)

    def forward(self, x):
        x = torch.relu(self.stem(x))
        s = torch.relu(self.a(x)) + torch.relu(self.b(x))
        y = torch.relu(self.c(torch.relu(s)))
        z = torch.cat([torch.relu(self.d(y)), torch.relu(self.e(y))], 1)
        z = torch.relu(self.f(z))
        return self.fc(torch.flatten(self.pool(z), 1))


def _export(strategy, sparsity=0.4):
    torch.manual_seed(0)
    sm = lower(JoinNet().eval(), input_chw=(3, 32, 32))
    g = sm.graph
    store = {k: np.asarray(a) for k, a in sm.proxy_weights().items()}
    scores = reslice.score_channels(g, store, "l2", side="output")
    masks = reslice.make_masks(g, scores, sparsity, "unconstrained", reslice.find_segments(g), side="output",
                               scope="per-layer")
    plans, fallbacks = reslice.plan_model(g, masks, "output", strategy, "error")
    return sm, masks, plans, E.export_graph(g, plans)


@pytest.mark.parametrize("strategy", ["reorder", "baseline"])
def test_output_mode_export_graph(strategy):
    sm, masks, plans, eg = _export(strategy)
    assert masks and any(len(v) < sm.graph.layer(k).out_channels for k, v in masks.items())
    ref_g, st = sm.graph, reslice.WeightStore({k: np.asarray(a) for k, a in sm.proxy_weights().items()})
    for p in plans:
        ref_g, st = reslice.apply_plan(p, ref_g, st)
    assert reslice.graph.graph_to_dict(eg) == reslice.graph.graph_to_dict(ref_g)
    kinds = {lay.kind.value for lay in eg.layers}
    if strategy == "reorder":
        assert any(p.join is not None and not p.join.keep_original for p in plans)
        assert "slice" in kinds
    else:
        assert any(lay.id.endswith(".restore") for lay in eg.layers) and "gather" in kinds


@pytest.mark.parametrize("strategy", ["reorder", "baseline"])
def test_output_mode_engine_schedule(strategy, monkeypatch):
    monkeypatch.setattr(K, "permute_weights", lambda W, rows, cols, **kw: torch.zeros(1))
    monkeypatch.setattr(_lib, "conv_weight_layout", lambda cin, coff, g, kh=1, kw=1: (0 if g else coff & 7, 64))
    monkeypatch.setattr(_lib, "conv_stem_kpad", lambda cin, kh, kw: 128)
    sm, masks, plans, eg = _export(strategy)
    eng = EN.from_plans(sm, eg, E.compose_maps(sm.graph, plans), batch=2, device="cpu")
    kinds = [op.kind for op in eng.ops]
    assert kinds.count("conv") == 8
    if strategy == "baseline":
        assert kinds.count("gather") >= 1  # the zero-fill restores


@pytest.mark.gpu
@pytest.mark.parametrize("strategy", ["reorder", "baseline"])
def test_output_mode_logits_match_oracle(strategy):
    from oracle.apply_plan_ref import apply_plans_spatial
    from oracle.spatial_ref import deviation, run_spatial

    sm, masks, plans, eg = _export(strategy)
    N = 8
    x = torch.randn(N, 3, 32, 32, generator=torch.Generator().manual_seed(1))
    eng = EN.from_plans(sm, eg, E.compose_maps(sm.graph, plans), batch=N)
    got = eng.forward(x.cuda()).cpu()
    w, v = apply_plans_spatial(plans, sm.graph, sm.weights, sm.vectors)
    ref = run_spatial(eg, sm.specs, w, v, x, dtype=torch.float32)
    # the export is equivalent to the output-masked original (interp.py:61-63)
    orig = run_spatial(sm.graph, sm.specs, sm.weights, sm.vectors, x, dtype=torch.float64)
    assert torch.isfinite(got).all()
    assert deviation(got, ref) <= 2e-2, deviation(got, ref)
    del orig
