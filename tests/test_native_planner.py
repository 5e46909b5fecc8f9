"""Native planner core (csrc/planner.cpp) vs the reference planner.

* golden: the reference's decompose_paths + order_channels outputs on 120 random reorder
  graphs (tests/golden/planner_core.json, tools/make_planner_golden.py) -- no reference
  needed at test time;
* live (when the reference is importable here): random graphs, and whole `plan_model`
  runs on the committed ResNet configs with the native core installed give the same
  plans as the pure-Python planner.
"""

import json
import random
import sys
from pathlib import Path

import pytest

from paper_2307_08771_b200 import ir, native_planner as NP, plans as P

ROOT = Path(__file__).resolve().parents[1]
REF = Path("/root/reference/pkg/src")


def test_native_core_matches_reference_golden():
    data = json.loads((ROOT / "tests" / "golden" / "planner_core.json").read_text())
    for case in data["cases"]:
        paths, kept, dropped = NP.decompose_and_order(list(case["nodes"].items()), case["channel_space"])
        assert [[list(m), r, list(a)] for m, r, a in paths] == case["paths"]
        assert list(kept) == case["order"] and list(dropped) == case["dropped"]


def test_native_core_rejects_bad_graphs():
    with pytest.raises(ValueError):
        NP.decompose_and_order([("a", {5})], 4)  # channel out of range
    with pytest.raises(ValueError):
        NP.decompose_and_order([("a", set())], 4)  # empty retained set


def _reference():
    if not REF.exists():
        pytest.skip("reference not present (GPU box)")
    sys.path.insert(0, str(REF))
    import reslice

    return reslice


def test_native_core_matches_live_reference_random():
    reslice = _reference()
    from reslice.ordering import order_channels
    from reslice.path_search import decompose_paths
    from reslice.reorder_graph import reorder_graph_from_sets

    rng = random.Random(7)
    for _ in range(60):
        space = rng.choice([16, 64, 200])
        sets = {f"n{i}": rng.sample(range(space), rng.randint(1, space)) for i in range(rng.randint(1, 10))}
        rg = reorder_graph_from_sets(sets, space)
        paths = decompose_paths(rg)
        order = order_channels(rg, paths)
        npaths, kept, dropped = NP.decompose_and_order([(k, v.retained) for k, v in rg.nodes.items()], space)
        assert [(p.nodes, p.reward, p.covered_parents) for p in paths] == npaths
        assert order.order == kept and order.dropped == dropped
    assert reslice is not None


@pytest.mark.parametrize("cfg_name", ["resnet18_s50", "resnet50_s50"])
def test_plan_model_identical_with_native_core(cfg_name):
    reslice = _reference()
    from paper_2307_08771_b200.configs import CONFIGS

    cfg = CONFIGS[cfg_name]
    g = reslice.graph.graph_from_dict(json.loads((cfg.asset_dir / "graph.json").read_text()))
    masks = {k: tuple(v) for k, v in ir.load_masks(cfg.asset_dir / "masks.json").items()}
    NP.install(reslice)
    try:
        plans, _ = reslice.plan_model(g, masks, "input", "reorder", "error")
    finally:
        NP.uninstall()
    want = P.load_plans(cfg.asset_dir / "plans_reorder.json")  # made by the pure-Python reference
    got = [P.from_reference(p) for p in plans]
    assert [P.plan_to_dict(p) for p in got] == [P.plan_to_dict(p) for p in want]
