"""B200 twin of the reference export: `plan_model` -> `apply_plan` -> `export_model`.

* Planning is the REFERENCE's (pipeline.py:99-132), consumed unchanged: the
  imported `reslice.pipeline.plan_model`, or the reference's own plan files
  (planner.py:907-927), e.g. the committed assets.  Nothing here re-derives an
  ordering.
* The graph half of `apply_plan` (planner.py:648-796) is the reference's own
  function, run on shape-only weights: producer widths, infill gathers, the
  output-mode join rewrite, interior widths and `<consumer>.read` SLICE/GATHER
  insertion all come out exactly as the reference exports them.
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

import numpy as np

from .ir import ChannelMask, LayerKind, ModelGraph, ValidationError, WeightStore, validate_masks
from .plans import MODE_INPUT, STRATEGY_REORDER, CopyStats, SegmentPlan, copy_report
from .ref import reslice

_ref_apply_plan = reslice.planner.apply_plan

log = logging.getLogger(__name__)


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
    plans, fallbacks = reslice.pipeline.plan_model(graph, dict(masks), mode, strategy, on_unsupported)
    return list(plans), list(fallbacks)


# ------------------------------------------------------------------ graph rewrite
def _shape_store(graph: ModelGraph) -> WeightStore:
    """Zero tensors with the reference WeightStore shapes (graph.py:150-161): the
    reference `apply_plan` validates weights against the graph, and only its graph
    half is used here -- the weight half runs on the GPU from the 4-D sidecar."""
    st = WeightStore()
    for lay in graph.layers:
        if lay.kind is LayerKind.CHANNEL_MIX:
            st[lay.id] = np.zeros((lay.out_channels, lay.in_channels))
        elif lay.kind is LayerKind.PER_CHANNEL:
            st[lay.id] = np.zeros((lay.out_channels,))
    return st


def export_graph(graph: ModelGraph, plans: Sequence[SegmentPlan]) -> ModelGraph:
    """The exported graph: the reference's own `apply_plan` (planner.py:648-796),
    applied plan by plan as `export_model` does (pipeline.py:140-142), on shape-only
    weights.  Input and output mode (infill gathers, join rewrite) alike."""
    g, st = graph, _shape_store(graph)
    for p in plans:
        g, st = _ref_apply_plan(p, g, st)
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
            if any(not (0 <= r < width) for r in plan.producer_orders.get(p, ())):
                raise ValidationError([f"{p}: producer order index out of [0, {width})"])
            if p in maps.rows:
                raise ValidationError([f"{p}: rows rewritten by two plans"])
            if tuple(rows) != tuple(range(width)):
                maps.rows[p] = tuple(rows)
        for u, perm in plan.per_channel.items():  # planner.py:731-733
            width = graph.layer(u).out_channels
            if any(not (0 <= i < width) for i in perm):
                raise ValidationError([f"{u}: per-channel index out of [0, {width})"])
            maps.vec[u] = tuple(perm)
        for acc in plan.consumers:
            width = graph.layer(acc.consumer).in_channels
            if any(not (0 <= i < width) for i in acc.perm):
                raise ValidationError([f"{acc.consumer}: column index out of [0, {width})"])
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
    from . import _lib
    bad = _lib.index_faults()
    if bad:
        raise ValidationError([f"export: {bad} plan indices outside their source tensors"])
    return ew


def apply_plan(plan: SegmentPlan, graph: ModelGraph, weights: ExportedWeights) -> tuple[ModelGraph, ExportedWeights]:
    """planner.py:648-796 with the reference's signature, on 4-D device weights.

    The graph half is the reference's own `apply_plan`; the weight half permutes, on the
    GPU, exactly the tensors this plan touches (its producers' rows, its consumers'
    columns, its per-channel vectors).  Pure, like the reference (planner.py:655): the
    input `weights` is not modified; untouched tensors are shared with the result."""
    from . import kernels as K

    g_out = export_graph(graph, [plan])
    maps = compose_maps(graph, [plan])
    new = ExportedWeights(mix=dict(weights.mix), vec={k: dict(v) for k, v in weights.vec.items()})
    for lid in sorted(set(maps.rows) | set(maps.cols)):
        W = weights.mix[lid]
        O, I = W.shape[0], W.shape[1]
        new.mix[lid] = K.permute_weights(W.contiguous(), maps.rows.get(lid, range(O)), maps.cols.get(lid, range(I)),
                                         out_dtype=W.dtype)
    for uid, perm in maps.vec.items():
        if uid in weights.vec:
            new.vec[uid] = {n: K.permute_vector(t.contiguous(), perm) for n, t in weights.vec[uid].items()}
    from . import _lib
    bad = _lib.index_faults()
    if bad:
        raise ValidationError([f"plan {plan.segment}: {bad} indices outside their source tensors"])
    return g_out, new


def export_model(graph: ModelGraph, weights: Mapping[str, torch.Tensor],
                 vectors: Mapping[str, Mapping[str, torch.Tensor]] | None, masks: ChannelMask,
                 mode: str = MODE_INPUT, strategy: str = STRATEGY_REORDER, on_unsupported: str = "error",
                 plans: Sequence[SegmentPlan] | None = None, fallbacks: Sequence[str] = (),
                 device="cuda", out_dtype=torch.float32) -> ExportResult:
    """pipeline.py:135-146 with the weight math on the GPU.  Pure: inputs are
    not modified.  `weights` are the 4-D CHANNEL_MIX tensors of the sidecar
    (2-D linear weights as [O, I, 1, 1])."""
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
