"""Pin the CPU oracle and the integer half of the B200 export to the REFERENCE.

Fixtures in tests/golden/ were produced by running the reference `reslice`
(tools/make_golden.py, tools/make_assets.py); nothing here imports it.
  * exported graphs (SLICE/GATHER insertion, widths, ids, edge order) must be
    identical -- bit-exact integer contract;
  * exported weights from the oracle's numpy apply_plan restatement must be
    bit-identical (float.hex / sha256);
  * the oracle interpreter must reproduce the reference interp.run outputs;
  * the spatial oracle, run on the same channel-collapsed graphs, must agree
    with the interpreter (its op semantics are the reference's).
"""

import hashlib
import json
from pathlib import Path

import numpy as np
import pytest
import torch

from oracle import apply_plan_ref, interp_ref, spatial_ref
from paper_2307_08771_b200 import export as E, ir, plans as P
from paper_2307_08771_b200.configs import CONFIGS

GOLDEN = Path(__file__).resolve().parent / "golden"


def _unhex(xs, shape=None):
    a = np.array([float.fromhex(x) for x in xs], dtype=np.float64)
    return a.reshape(shape) if shape is not None else a


def _sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.float64).tobytes()).hexdigest()[:16]


def _weights(d):
    return {k: _unhex(v["hex"], tuple(v["shape"])) for k, v in d.items()}


def _regen_weights(graph, seed):
    """Restates pkg/tests/helpers.py:27-38 (build_model): seeded standard normals
    in layer order, (out, in) per CHANNEL_MIX, (out,) per PER_CHANNEL."""
    rng = np.random.default_rng(seed)
    w = {}
    for lay in graph.layers:
        if lay.kind is ir.LayerKind.CHANNEL_MIX:
            w[lay.id] = rng.standard_normal((lay.out_channels, lay.in_channels))
        elif lay.kind is ir.LayerKind.PER_CHANNEL:
            w[lay.id] = rng.standard_normal(lay.out_channels)
    return w


EXAMPLES = json.loads((GOLDEN / "reference_examples.json").read_text())
DAGS = json.loads((GOLDEN / "random_dags.json").read_text())


@pytest.mark.parametrize("ex", EXAMPLES, ids=[e["name"] for e in EXAMPLES])
def test_reference_examples(ex):
    g = ir.graph_from_dict(ex["graph"])
    plans = [P.plan_from_dict(d) for d in ex["plans"]]
    # integer contract: our graph rewrite == the reference's export
    assert ir.graph_to_dict(E.export_graph(g, plans)) == ex["export"]
    # weight math: numpy restatement, bit-exact
    got = apply_plan_ref.apply_plans_weights(plans, g, _weights(ex["weights"]))
    want = _weights(ex["export_weights"])
    assert set(got) == set(want)
    for k in want:
        assert np.array_equal(got[k], want[k]), k
    # interpreter restatement
    w0 = _weights(ex["weights"])
    eg = ir.graph_from_dict(ex["export"])
    masks = {k: tuple(v) for k, v in ex["masks"].items()}
    for x, y0, y1 in zip(ex["inputs"], ex["outputs_masked_original"], ex["outputs_export"]):
        x = _unhex(x)
        np.testing.assert_allclose(interp_ref.run(g, w0, x, masks), _unhex(y0), rtol=1e-12, atol=1e-12)
        np.testing.assert_allclose(interp_ref.run(eg, want, x), _unhex(y1), rtol=1e-12, atol=1e-12)


def test_reference_literals_fan_fixture():
    """The literal expectations of test_planner.py:220-240 / 35-54."""
    ex = next(e for e in EXAMPLES if e["name"] == "fan4_fixed_order_apply_plan")
    plan = P.plan_from_dict(ex["plans"][0])
    assert plan.producer_orders["A"] == (0, 2, 3, 1)
    acc = {a.consumer: a for a in plan.consumers}
    assert (acc["B"].mode, acc["B"].start, acc["B"].length, acc["B"].perm) == ("slice", 0, 3, (0, 2, 3))
    assert (acc["C"].mode, acc["C"].start, acc["C"].length, acc["C"].perm) == ("slice", 1, 3, (2, 3, 1))
    assert (acc["D"].mode, acc["D"].perm, acc["D"].indices) == ("gather", (0, 3), (0, 2))
    assert plan.stats == P.CopyStats(8, 2)
    w = _weights(ex["weights"])
    got = apply_plan_ref.apply_plans_weights([plan], ir.graph_from_dict(ex["graph"]), w)
    assert np.array_equal(got["A"], w["A"][[0, 2, 3, 1], :])
    assert np.array_equal(got["B"], w["B"][:, [0, 2, 3]])
    assert np.array_equal(got["C"], w["C"][:, [2, 3, 1]])
    assert np.array_equal(got["D"], w["D"][:, [0, 3]])
    reads = {lay.id: lay for lay in ir.graph_from_dict(ex["export"]).layers if lay.id.endswith(".read")}
    assert reads["B.read"].params == (0, 3) and reads["C.read"].params == (1, 3)
    assert reads["D.read"].kind is ir.LayerKind.GATHER and reads["D.read"].params == (0, 2)
    rescue = next(e for e in EXAMPLES if e["name"] == "zero_copy_rescue")
    assert P.plan_from_dict(rescue["plans"][0]).producer_orders["A"] == (0, 1, 2, 4, 3, 5)  # test_pipeline.py:78-96


@pytest.mark.parametrize("rec", DAGS, ids=[f"dag{r['seed']}" for r in DAGS])
def test_random_dags(rec):
    g = ir.graph_from_dict(rec["graph"])
    w = _regen_weights(g, rec["seed"])
    assert {k: _sha(v) for k, v in w.items()} == rec["weights_sha"], "weight regeneration drifted"
    for case in rec["cases"]:
        plans = [P.plan_from_dict(d) for d in case["plans"]]
        eg = E.export_graph(g, plans)
        assert ir.graph_to_dict(eg) == case["export"]
        ew = apply_plan_ref.apply_plans_weights(plans, g, w)
        assert {k: _sha(v) for k, v in ew.items()} == case["export_sha"]
        assert [P.copy_report(plans).total_reads, P.copy_report(plans).copied] == case["totals"]
        masks = {k: tuple(v) for k, v in case["masks"].items()}
        for x, y0, y1 in zip(case["inputs"], case["outputs_masked_original"], case["outputs_export"]):
            x = _unhex(x)
            np.testing.assert_allclose(interp_ref.run(g, w, x, masks), _unhex(y0), rtol=1e-12, atol=1e-12)
            np.testing.assert_allclose(interp_ref.run(eg, ew, x), _unhex(y1), rtol=1e-12, atol=1e-12)
            # spatial oracle with the reference's 1x1 semantics == interp
            sw = {k: torch.from_numpy(v).reshape(*v.shape, 1, 1) for k, v in ew.items() if v.ndim == 2}
            sv = {k: {"bias": torch.from_numpy(v)} for k, v in ew.items() if v.ndim == 1}
            xs = torch.from_numpy(x).reshape(1, -1, 1, 1)
            out = spatial_ref.run_spatial(eg, {}, sw, sv, xs)
            np.testing.assert_allclose(out.numpy().reshape(-1), _unhex(y1), rtol=1e-12, atol=1e-12)


@pytest.mark.parametrize("cfg_name", ["resnet18_s50", "resnet50_s50", "resnet101_s50"])
def test_resnet_assets_pin_lowering_and_apply(cfg_name):
    """Lowering is deterministic (proxy sha == reference run) and the oracle's
    apply_plan on the proxies reproduces the reference export bit-for-bit."""
    from paper_2307_08771_b200.configs import build_spatial_model

    cfg = CONFIGS[cfg_name]
    meta = json.loads((cfg.asset_dir / "meta.json").read_text())
    sm = build_spatial_model(cfg)
    proxy = sm.proxy_weights()
    assert {k: _sha(v) for k, v in proxy.items()} == meta["proxy_sha256"]
    g = ir.load_graph(cfg.asset_dir / "graph.json")
    assert ir.graph_to_dict(g) == ir.graph_to_dict(sm.graph)
    for st in ("reorder", "baseline"):
        plans = P.load_plans(cfg.asset_dir / f"plans_{st}.json")
        assert ir.graph_to_dict(E.export_graph(g, plans)) == json.loads(
            (cfg.asset_dir / f"export_{st}.json").read_text())
        ew = apply_plan_ref.apply_plans_weights(plans, g, proxy)
        assert {k: _sha(v) for k, v in ew.items()} == meta["strategies"][st]["exported_sha256"]
        assert P.copy_report(plans).copied == meta["strategies"][st]["copied"]


def test_spatial_oracle_export_equals_masked_original_fp64():
    """interp.py:98-121 metric on real spatial ResNet-18 (64x64 input, fp64):
    the exported network equals the mask-simulated original to ~1e-15."""
    from paper_2307_08771_b200.configs import build_spatial_model

    cfg = CONFIGS["resnet18_s50"]
    sm = build_spatial_model(cfg, randomize_bn=True)
    masks = ir.load_masks(cfg.asset_dir / "masks.json")
    x = torch.randn(2, 3, 64, 64, generator=torch.Generator().manual_seed(0), dtype=torch.float64)
    ref = spatial_ref.run_spatial(sm.graph, sm.specs, sm.weights, sm.vectors, x, masks=masks)
    for st in ("reorder", "baseline"):
        plans = P.load_plans(cfg.asset_dir / f"plans_{st}.json")
        eg = E.export_graph(sm.graph, plans)
        w, v = apply_plan_ref.apply_plans_spatial(plans, sm.graph, sm.weights, sm.vectors)
        got = spatial_ref.run_spatial(eg, sm.specs, w, v, x)
        assert spatial_ref.deviation(got, ref) <= 1e-12
        assert spatial_ref.top1_agreement(got, ref) == 1.0
