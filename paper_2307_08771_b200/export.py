"""B200 twin of the reference export: `plan_model` -> `apply_plan` -> `export_model`.

* Planning is the REFERENCE's (pipeline.py:99-132), consumed unchanged: when
  `reslice` is importable its `plan_model` is called; otherwise plans come from
  the reference's own plan files (planner.py:907-927), e.g. the committed
  assets.  Nothing here re-derives an ordering.
* The graph half of `apply_plan` (planner.py:648-796, input mode) is restated
  on the integer IR: producer widths, interior widths, and `<consumer>.read`
  SLICE/GATHER insertion with the reference's id and edge order, so the
  exported graph is identical to the reference's.
* The weight half runs on the GPU (`ub_permute_weights`): all plans touching a
  layer are composed first (a conv's rows come from its output segment's plan,
  its columns from its input segment's plan, pipeline.py:140-142 applies them
  one after another), then ONE kernel pass per layer writes the result.
"""

from __future__ import annotations

import logging
from dataclasses import dataclass, field, replace
from typing import Mapping, Sequence

import torch

from .ir import ChannelMask, Layer, LayerKind, ModelGraph, ValidationError, graph_from_dict, graph_to_dict, \
    validate, validate_masks
from .plans import MODE_INPUT, STRATEGY_REORDER, CopyStats, SegmentPlan, copy_report, from_reference

log = logging.getLogger(__name__)


class PlannerUnavailableError(RuntimeError):
    """`reslice` is not importable here and no plans were supplied."""


@dataclass
class ExportedWeights:
    """Device-resident counterpart of the reference WeightStore after export:
    CHANNEL_MIX -> [O', I', kh, kw], PER_CHANNEL -> named vectors (BN keeps
    weight/bias/mean/var, all permuted by the same per_channel order)."""

    mix: dict[str, torch.Tensor] = field(default_factory=dict)
    vec: dict[str, dict[str, torch.Tensor]] = field(default_factory=dict)


@dataclass(frozen=True)
class ExportResult:
    """pipeline.py:41-47."""

    graph: ModelGraph
    weights: ExportedWeights
    plans: tuple[SegmentPlan, ...]
    totals: CopyStats
    fallbacks: tuple[str, ...]


# ------------------------------------------------------------------ planning
def plan_model(graph: ModelGraph, masks: ChannelMask, mode: str = MODE_INPUT, strategy: str = STRATEGY_REORDER,
               on_unsupported: str = "error") -> tuple[list[SegmentPlan], list[str]]:
    """Calls the reference planner (pipeline.py:99-132) on `graph`."""
    try:
        import reslice  # noqa: F401
        from reslice.graph import graph_from_dict as ref_from_dict
        from reslice.pipeline import plan_model as ref_plan_model
    except ImportError as exc:
        raise PlannerUnavailableError(
            "the reference planner `reslice` is not importable; pass plans= "
            "(e.g. paper_2307_08771_b200.plans.load_plans(...))") from exc
    plans, fallbacks = ref_plan_model(ref_from_dict(graph_to_dict(graph)), dict(masks), mode, strategy,
                                      on_unsupported)
    return [from_reference(p) for p in plans], list(fallbacks)


# ------------------------------------------------------------------ graph rewrite
def _fresh_id(taken: set[str], base: str) -> str:
    """planner.py:637-645."""
    if base not in taken:
        taken.add(base)
        return base
    k = 2
    while f"{base}_{k}" in taken:
        k += 1
    taken.add(f"{base}_{k}")
    return f"{base}_{k}"


def apply_plan_graph(plan: SegmentPlan, graph: ModelGraph) -> ModelGraph:
    """Integer half of apply_plan (planner.py:648-796) for input-mode plans."""
    if plan.infill or (plan.join is not None and not plan.join.keep_original):
        raise NotImplementedError(f"{plan.segment}: output-mode join rewrite / infill is not on the B200 path")
    layers: dict[str, Layer] = {lay.id: lay for lay in graph.layers}
    order = [lay.id for lay in graph.layers]
    edges = list(graph.edges)
    taken = set(order)
    # 1. producers (planner.py:661-673)
    for p in plan.producers:
        lay = layers[p]
        rows = tuple(plan.producer_orders.get(p, range(lay.out_channels)))
        if lay.kind is LayerKind.INPUT:
            if rows != tuple(range(lay.out_channels)):
                raise ValidationError([f"{p}: cannot permute a model input"])
            continue
        if rows != tuple(range(lay.out_channels)):
            layers[p] = replace(lay, out_channels=len(rows))
    # 4. interior widths (planner.py:734-753)
    prov = ModelGraph([layers[i] for i in order], edges)
    interior = set(u for u in plan.interior if u in layers)
    for u in prov.topological_order():
        if u not in interior:
            continue
        lay = layers[u]
        widths = [layers[q].out_channels for q in prov.predecessors(u)]
        if lay.kind is LayerKind.CONCAT:
            w = sum(widths)
        elif lay.kind is LayerKind.ADD:
            if len(set(widths)) != 1:
                raise ValidationError([f"{u}: add operands now differ in width {widths}"])
            w = widths[0]
        elif lay.kind in (LayerKind.PASS_THROUGH, LayerKind.PER_CHANNEL):
            w = widths[0]
        else:
            raise ValidationError([f"{u}: unexpected {lay.kind.value} interior layer"])
        layers[u] = replace(lay, in_channels=w, out_channels=w)
    # 5. consumers (planner.py:755-790)
    for acc in plan.consumers:
        c = acc.consumer
        lay = layers[c]
        pred = graph.predecessors(c)[0]
        perm = tuple(acc.perm)
        if perm != tuple(range(lay.in_channels)):
            layers[c] = replace(lay, in_channels=len(perm))
        src_w = layers[pred].out_channels
        if acc.mode == "slice":
            if acc.length != len(perm):
                raise ValidationError([f"{c}: slice length disagrees with its permutation"])
            if (acc.start, acc.length) == (0, src_w):
                continue
            nid = _fresh_id(taken, f"{c}.read")
            layers[nid] = Layer(nid, LayerKind.SLICE, src_w, acc.length, (acc.start, acc.length))
        else:
            if len(acc.indices) != len(perm):
                raise ValidationError([f"{c}: gather width disagrees with its permutation"])
            nid = _fresh_id(taken, f"{c}.read")
            layers[nid] = Layer(nid, LayerKind.GATHER, src_w, len(acc.indices), tuple(acc.indices))
        order.append(nid)
        try:
            k = edges.index((pred, c))
        except ValueError:
            raise ValidationError([f"{c}: expected edge from {pred} is missing"]) from None
        edges[k] = (nid, c)
        edges.append((pred, nid))
    out = ModelGraph([layers[i] for i in order], edges)
    diags = validate(out)
    if diags:
        raise ValidationError([f"plan {plan.segment} produced an inconsistent model"] + diags)
    return out


def export_graph(graph: ModelGraph, plans: Sequence[SegmentPlan]) -> ModelGraph:
    g = graph
    for p in plans:
        g = apply_plan_graph(p, g)
    return g


# ------------------------------------------------------------------ index composition
@dataclass
class LayerMaps:
    """Composed index maps of all plans: rows/cols per CHANNEL_MIX (-1 = zero
    row/column), per-channel permutations per PER_CHANNEL node.  None =
    identity (the layer is untouched by every plan)."""

    rows: dict[str, tuple[int, ...]] = field(default_factory=dict)
    cols: dict[str, tuple[int, ...]] = field(default_factory=dict)
    vec: dict[str, tuple[int, ...]] = field(default_factory=dict)


def compose_maps(graph: ModelGraph, plans: Sequence[SegmentPlan]) -> LayerMaps:
    maps = LayerMaps()
    for plan in plans:
        for p in plan.producers:
            if graph.layer(p).kind is LayerKind.INPUT:
                continue
            width = graph.layer(p).out_channels
            rows = list(plan.producer_orders.get(p, range(width)))
            for local in plan.zero_rows.get(p, ()):  # planner.py:672-673
                rows[rows.index(local)] = -1
            if p in maps.rows:
                raise ValidationError([f"{p}: rows rewritten by two plans"])
            if tuple(rows) != tuple(range(width)):
                maps.rows[p] = tuple(rows)
        for u, perm in plan.per_channel.items():  # planner.py:731-733
            maps.vec[u] = tuple(perm)
        for acc in plan.consumers:
            width = graph.layer(acc.consumer).in_channels
            cols = list(acc.perm)
            for local in plan.zero_columns.get(acc.consumer, ()):  # planner.py:766-767
                cols[list(acc.perm).index(local)] = -1
            if acc.consumer in maps.cols:
                raise ValidationError([f"{acc.consumer}: columns rewritten by two plans"])
            if tuple(cols) != tuple(range(width)):
                maps.cols[acc.consumer] = tuple(cols)
    return maps


# ------------------------------------------------------------------ weights on device
def _i32(seq, device):
    return torch.as_tensor(list(seq), dtype=torch.int32).to(device)


def export_weights(graph: ModelGraph, weights: Mapping[str, torch.Tensor],
                   vectors: Mapping[str, Mapping[str, torch.Tensor]], maps: LayerMaps,
                   device="cuda", out_dtype=torch.float32) -> ExportedWeights:
    """Weight half of apply_plan for every layer, one GPU pass per tensor."""
    from . import kernels as K

    ew = ExportedWeights()
    for lid, w in weights.items():
        O, I = w.shape[0], w.shape[1]
        rows = maps.rows.get(lid, range(O))
        cols = maps.cols.get(lid, range(I))
        wd = w.to(device).contiguous()
        ew.mix[lid] = K.permute_weights(wd, rows, cols, out_dtype=out_dtype)
    for uid, named in vectors.items():
        perm = maps.vec.get(uid)
        ew.vec[uid] = {}
        for k, v in named.items():
            vd = v.to(device).contiguous()
            ew.vec[uid][k] = K.permute_vector(vd, perm) if perm is not None else vd.clone()
    return ew


def export_model(graph: ModelGraph, weights: Mapping[str, torch.Tensor],
                 vectors: Mapping[str, Mapping[str, torch.Tensor]] | None, masks: ChannelMask,
                 mode: str = MODE_INPUT, strategy: str = STRATEGY_REORDER, on_unsupported: str = "error",
                 plans: Sequence[SegmentPlan] | None = None, fallbacks: Sequence[str] = (),
                 device="cuda", out_dtype=torch.float32) -> ExportResult:
    """pipeline.py:135-146 with the weight math on the GPU.  Pure: inputs are
    not modified.  `weights` are the 4-D CHANNEL_MIX tensors of the sidecar
    (2-D linear weights as [O, I, 1, 1])."""
    if mode != MODE_INPUT:
        raise NotImplementedError("output-mode export is outside the B200 hot path (SURVEY.md 8f-2)")
    diags = validate_masks(graph, masks, mode)
    if diags:
        raise ValidationError(diags)
    if plans is None:
        plans, fallbacks = plan_model(graph, masks, mode, strategy, on_unsupported)
    plans = list(plans)
    out_graph = export_graph(graph, plans)
    maps = compose_maps(graph, plans)
    ew = export_weights(graph, weights, vectors or {}, maps, device=device, out_dtype=out_dtype)
    return ExportResult(out_graph, ew, tuple(plans), copy_report(plans), tuple(fallbacks))
