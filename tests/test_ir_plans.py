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


def test_output_mode_is_refused():
    g = ir.load_graph(R50 / "graph.json")
    with pytest.raises(NotImplementedError):
        E.export_model(g, {}, {}, {}, mode="output", plans=[])


def test_plan_model_without_reference_needs_plans(monkeypatch):
    import builtins

    real = builtins.__import__

    def no_reslice(name, *a, **k):
        if name.startswith("reslice"):
            raise ImportError("reslice hidden")
        return real(name, *a, **k)

    monkeypatch.setattr(builtins, "__import__", no_reslice)
    with pytest.raises(E.PlannerUnavailableError):
        E.plan_model(ir.load_graph(R50 / "graph.json"), {})
