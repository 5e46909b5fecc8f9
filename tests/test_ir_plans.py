"""IR / masks / plan file formats (graph.py:316-441, planner.py:813-927) and the
export twin's host logic, without a GPU."""

import json

import pytest

from paper_2307_08771_b200 import export as E, ir, plans as P
from paper_2307_08771_b200.configs import CONFIGS

R50 = CONFIGS["resnet50_s50"].asset_dir


def test_graph_roundtrip_byte_identical(tmp_path):
    g = ir.load_graph(R50 / "graph.json")
    ir.save_graph(g, tmp_path / "a.json")
    ir.save_graph(ir.load_graph(tmp_path / "a.json"), tmp_path / "b.json")
    assert (tmp_path / "a.json").read_bytes() == (tmp_path / "b.json").read_bytes()
    assert not ir.validate(g)


def test_plans_roundtrip(tmp_path):
    plans = P.load_plans(R50 / "plans_reorder.json")
    P.save_plans(plans, tmp_path / "p.json")
    again = P.load_plans(tmp_path / "p.json")
    assert [P.plan_to_dict(p) for p in again] == [P.plan_to_dict(p) for p in plans]
    obj = json.loads((tmp_path / "p.json").read_text())
    assert obj["totals"]["copied"] == P.copy_report(plans).copied == 4610
    assert obj["totals"]["total_reads"] == 12290


def test_masks_roundtrip(tmp_path):
    m = ir.load_masks(R50 / "masks.json")
    ir.save_masks(m, tmp_path / "m.json")
    assert ir.load_masks(tmp_path / "m.json") == m
    g = ir.load_graph(R50 / "graph.json")
    assert not ir.validate_masks(g, m)
    assert ir.validate_masks(g, {"conv1": (5,)})  # index out of [0, 3)
    assert ir.validate_masks(g, {"bn1": (0,)})  # not a channel-mixing layer


def test_format_errors(tmp_path):
    (tmp_path / "bad.json").write_text("[1, 2]")
    with pytest.raises(ir.ModelFormatError):
        ir.load_graph(tmp_path / "bad.json")
    (tmp_path / "v.json").write_text(json.dumps({"version": 9, "layers": [], "edges": []}))
    with pytest.raises(ir.ModelFormatError):
        ir.load_graph(tmp_path / "v.json")
    with pytest.raises(ir.ModelFormatError):
        P.plan_from_dict({"segment": "x"})


def test_topological_order_file_order_ties():
    L = ir.LayerKind
    g = ir.ModelGraph([ir.Layer("in", L.INPUT, 2, 2), ir.Layer("b", L.CHANNEL_MIX, 2, 2),
                       ir.Layer("a", L.CHANNEL_MIX, 2, 2), ir.Layer("s", L.ADD, 2, 2),
                       ir.Layer("out", L.OUTPUT, 2, 2)],
                      [("in", "b"), ("in", "a"), ("a", "s"), ("b", "s"), ("s", "out")])
    assert g.topological_order() == ("in", "b", "a", "s", "out")
    assert g.predecessors("s") == ("a", "b")  # edge-file order is the operand order


def test_compose_maps_matches_sequential_plans():
    """Rows from a layer's output segment, columns from its input segment; the
    composition equals applying the plans one after another."""
    g = ir.load_graph(R50 / "graph.json")
    plans = P.load_plans(R50 / "plans_reorder.json")
    maps = E.compose_maps(g, plans)
    eg = E.export_graph(g, plans)
    for lid, rows in maps.rows.items():
        assert eg.layer(lid).out_channels == len(rows)
    for lid, cols in maps.cols.items():
        assert eg.layer(lid).in_channels == len(cols)
    # every per-channel permutation is a permutation of a subset of the vector
    for uid, perm in maps.vec.items():
        assert len(set(perm)) == len(perm) == eg.layer(uid).out_channels


def test_output_mode_export_graph_is_the_references():
    """Output mode (planner.py:479-607 + apply_plan steps 2-3): the exported graph is
    the reference's own apply_plan output, and the composed maps cover every
    rewritten layer (rows = kept filters, cols = full-slice permutations)."""
    from paper_2307_08771_b200.ref import reslice
    L = ir.LayerKind
    # two producers joined by an add, read by two consumers: no per-channel interior
    g = ir.ModelGraph(
        [ir.Layer("x", L.INPUT, 4, 4), ir.Layer("a", L.CHANNEL_MIX, 4, 6), ir.Layer("b", L.CHANNEL_MIX, 4, 6),
         ir.Layer("s", L.ADD, 6, 6), ir.Layer("r", L.PASS_THROUGH, 6, 6), ir.Layer("c", L.CHANNEL_MIX, 6, 3),
         ir.Layer("d", L.CHANNEL_MIX, 6, 2), ir.Layer("cat", L.CONCAT, 5, 5), ir.Layer("out", L.OUTPUT, 5, 5)],
        [("x", "a"), ("x", "b"), ("a", "s"), ("b", "s"), ("s", "r"), ("r", "c"), ("r", "d"),
         ("c", "cat"), ("d", "cat"), ("cat", "out")])
    masks = {"a": (0, 1, 4), "b": (1, 2, 4, 5)}
    for strategy in ("reorder", "baseline"):
        plans, _ = reslice.pipeline.plan_model(g, masks, "output", strategy, "baseline")
        st = E._shape_store(g)
        ref_g = g
        for pl in plans:
            ref_g, st = reslice.planner.apply_plan(pl, ref_g, st)
        eg = E.export_graph(g, plans)
        assert ir.graph_to_dict(eg) == ir.graph_to_dict(ref_g)
        maps = E.compose_maps(g, plans)
        assert eg.layer("a").out_channels == len(maps.rows["a"]) == 3
        assert eg.layer("b").out_channels == len(maps.rows["b"]) == 4
        kinds = {lay.kind for lay in eg.layers}
        if strategy == "baseline":
            assert L.GATHER in kinds  # zero-fill infill after each pruned producer
        else:
            assert "s" not in eg  # the join was rewritten into runs of slices + adds + a concat


def test_compose_maps_rejects_out_of_range_indices():
    g = ir.load_graph(R50 / "graph.json")
    plans = P.load_plans(R50 / "plans_reorder.json")
    bad = plans[0]
    p0 = bad.producers[-1]
    width = g.layer(p0).out_channels
    orders = dict(bad.producer_orders)
    orders[p0] = tuple(orders.get(p0, range(width)))[:-1] + (width,)
    import dataclasses
    with pytest.raises(ir.ValidationError):
        E.compose_maps(g, [dataclasses.replace(bad, producer_orders=orders)])


def test_reference_is_imported_unmodified():
    """ir/plans/export consume the reference package itself (no re-typed copy)."""
    import hashlib
    from pathlib import Path

    from paper_2307_08771_b200.ref import REF_SOURCE, reslice
    assert ir.ModelGraph is reslice.graph.ModelGraph and P.SegmentPlan is reslice.planner.SegmentPlan
    src = REF_SOURCE / "src" / "reslice"
    if src.exists():
        for f in ("graph.py", "planner.py", "pipeline.py", "interp.py"):
            here = Path(reslice.__file__).parent / f
            assert hashlib.sha256(here.read_bytes()).digest() == hashlib.sha256((src / f).read_bytes()).digest()


def test_live_plan_model_reproduces_the_committed_plans():
    """export.plan_model runs the reference planner itself (pipeline.py:99-132): on the
    ResNet-18 config it reproduces the committed plan file byte for byte."""
    from paper_2307_08771_b200.configs import CONFIGS

    cfg = CONFIGS["resnet18_s50"]
    g = ir.load_graph(cfg.asset_dir / "graph.json")
    masks = ir.load_masks(cfg.asset_dir / "masks.json")
    plans, fallbacks = E.plan_model(g, masks, "input", "reorder", "baseline")
    want = P.load_plans(cfg.asset_dir / "plans_reorder.json")
    assert [P.plan_to_dict(p) for p in sorted(plans, key=lambda p: p.segment)] == [P.plan_to_dict(p) for p in want]
