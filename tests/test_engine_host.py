"""Engine compilation (fusion + schedule) without a GPU: kernels are stubbed,
the graph analysis is the real one."""

import pytest
import torch

from paper_2307_08771_b200 import _lib, engine as EN, export as E, kernels as K, plans as P
from paper_2307_08771_b200.configs import CONFIGS, build_spatial_model


@pytest.fixture
def stub_kernels(monkeypatch):
    monkeypatch.setattr(K, "permute_weights", lambda W, rows, cols, **kw: torch.zeros(1))
    monkeypatch.setattr(_lib, "conv_weight_layout", lambda cin, coff, g, kh=1, kw=1: (0 if g else coff & 7, 64))
    monkeypatch.setattr(_lib, "conv_stem_kpad", lambda cin, kh, kw: 128)


@pytest.fixture(scope="module")
def r50():
    return build_spatial_model(CONFIGS["resnet50_s50"])


def _engine(sm, strategy, gather_mode, batch=2):
    cfg = CONFIGS["resnet50_s50"]
    plans = P.load_plans(cfg.asset_dir / f"plans_{strategy}.json")
    eg = E.export_graph(sm.graph, plans)
    return EN.from_plans(sm, eg, E.compose_maps(sm.graph, plans), batch=batch, device="cpu",
                         gather_mode=gather_mode), eg


@pytest.mark.parametrize("strategy,gather_mode,n_gather_ops", [
    ("reorder", "fused", 0), ("reorder", "copy", 11), ("baseline", "fused", 0), ("baseline", "copy", 21)])
def test_resnet50_schedule(stub_kernels, r50, strategy, gather_mode, n_gather_ops):
    eng, eg = _engine(r50, strategy, gather_mode)
    kinds = [op.kind for op in eng.ops]
    assert kinds.count("conv") == 54
    assert kinds.count("gather") == n_gather_ops  # the input GATHER is fused into the stem
    # the max pool after the space-to-depth stem runs in the stem's epilogue
    assert kinds.count("maxpool") == 0 and kinds.count("avgpool") == 1
    stem = [op for op in eng.ops if "stem_idx" in op.info]
    assert len(stem) == 1 and "pool" in stem[0].info
    assert "stage" not in kinds and "eltwise" not in kinds  # BN/ADD/ReLU all absorbed
    # every residual ADD is fused into a conv epilogue; each conv absorbs its BN
    convs = [op for op in eng.ops if op.kind == "conv"]
    assert sum(1 for op in convs if op.info.get("residual")) == 16
    assert all(op.info["bn"] is not None for op in convs)
    # schedule respects data dependencies
    produced = set()
    alias = eng._alias

    def base(v):
        while v in alias:
            v = alias[v][0]
        return v

    for op in eng.ops:
        for i in op.inputs:
            assert base(i) in produced or base(i) == "x", (op.output, i)
        produced.add(op.output)
    assert eng.output_value.C == 1000
    # the fc's GATHER read is folded into the global pool (compacted kept channels) in fused mode
    pool = next(op for op in eng.ops if op.kind == "avgpool")
    fc = next(op for op in eng.ops if op.kind == "conv" and op.info["conv"] == "fc")
    if gather_mode == "fused" and eg.layer("fc.read").kind.value == "gather":
        assert pool.output == "fc.read" and fc.info["read"] is None and fc.inputs[0] == "fc.read"
        assert tuple(pool.info["idx"]) == tuple(eg.layer("fc.read").params)
    else:
        assert "idx" not in pool.info


def test_slices_are_views_not_copies(stub_kernels, r50):
    eng, eg = _engine(r50, "reorder", "fused")
    slices = [lay for lay in eg.layers if lay.kind.value == "slice"]
    assert len(slices) == 10
    for op in eng.ops:
        assert op.output not in {s.id for s in slices}


def test_conv_stats_match_survey_flops(stub_kernels, r50):
    eng, _ = _engine(r50, "reorder", "fused")
    flops, _ = eng.per_image_work()
    assert 2.55e9 < flops < 2.75e9  # 2.644 GFLOP/img (reorder, per-layer)


@pytest.fixture(scope="module")
def dn121():
    return build_spatial_model(CONFIGS["densenet121_s50"])


@pytest.mark.parametrize("strategy", ["reorder", "baseline"])
def test_densenet121_concats_are_zero_copy_bands(stub_kernels, dn121, strategy):
    """Config 4: every dense-block concat is a view of one band buffer per block (the
    producers store their bands at 8-aligned offsets), every norm1/relu1 pair is applied
    as the prologue of its conv1's staged read, each transition's 2x2 average pool moves
    in front of its 1x1 conv, and no concat copy or standalone BN/ReLU pass is left
    except the final norm5 + relu (fused into one eltwise)."""
    cfg = CONFIGS["densenet121_s50"]
    plans = P.load_plans(cfg.asset_dir / f"plans_{strategy}.json")
    eg = E.export_graph(dn121.graph, plans)
    eng = EN.from_plans(dn121, eg, E.compose_maps(dn121.graph, plans), batch=2, device="cpu")
    kinds = [op.kind for op in eng.ops]
    n_concat = sum(1 for lay in eg.layers if lay.kind.value == "concat")
    assert n_concat == 58 and kinds.count("concat") == 0
    assert len(eng._concat_views) == 58
    assert len({v[0] for v in eng._concat_views.values()}) == 4  # one buffer per dense block
    convs = [op for op in eng.ops if op.kind == "conv"]
    assert len(convs) == 121
    pro = [op for op in convs if op.info.get("prologue")]
    assert len(pro) == 58 + 3  # every dense layer's conv1 + the three transitions
    assert sum(1 for op in convs if op.info.get("pool2")) == 3
    assert kinds.count("avgpool2d") == 0 and kinds.count("eltwise") == 1
    assert kinds.count("avgpool") == 1 and kinds.count("maxpool") == 0  # stem pool fused
    # schedule respects data dependencies through the band views
    done = set()
    for op in eng.ops:
        done.add(op.output)
    assert eng.output_value.C == 1000


def test_mobilenet_se_blocks_fuse_into_one_launch(stub_kernels):
    """Config 2: each squeeze-excitation block (global pool -> fc1 -> fc2 -> mul) runs its
    gate as ONE ub_se_gate launch; depthwise convs absorb their BN + activation."""
    sm = build_spatial_model(CONFIGS["mobilenet_v3_small_s50"])
    plans = P.load_plans(CONFIGS["mobilenet_v3_small_s50"].asset_dir / "plans_reorder.json")
    eg = E.export_graph(sm.graph, plans)
    eng = EN.from_plans(sm, eg, E.compose_maps(sm.graph, plans), batch=1, device="cpu")
    kinds = [op.kind for op in eng.ops]
    assert kinds.count("se") == 9 and kinds.count("dwconv") == 11
    assert kinds.count("avgpool") == 1  # the classifier's pool only
    assert all(op.info.get("bn") is not None for op in eng.ops if op.kind == "dwconv")
    assert len(eng.ops) == 55
    # every SE pool reads a depthwise output; the 3x3 ones write its pool partials themselves
    ses = [op for op in eng.ops if op.kind == "se"]
    assert all(op.info["dw"].kind == "dwconv" for op in ses)
    fused = [op for op in ses if "part" in op.info["dw"].info]
    assert len(fused) == sum(1 for op in ses if eng.specs[op.info["dw"].anchor].kernel == 3) >= 1
