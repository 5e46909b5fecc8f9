"""Oracle: apply_plan's weight math restated in numpy (planner.py:648-796).

Input-mode plans, applied one plan after another over a dict-of-arrays store,
as export_model does (pipeline.py:140-142).  Works for 2-D (out, in) proxies
and for 4-D (out, in, kh, kw) tensors alike: rows index axis 0, columns axis 1.
Plans are duck-typed (ours or the reference's).
"""

from __future__ import annotations

from typing import Mapping

import numpy as np


def apply_plan_weights(plan, widths_out: Mapping[str, int], widths_in: Mapping[str, int],
                       kinds: Mapping[str, str], store: dict[str, np.ndarray]) -> dict[str, np.ndarray]:
    """One plan.  widths_* are the CURRENT layer widths (before this plan);
    kinds maps layer id -> LayerKind value.  Returns a new store (pure).
    Ids absent from `store` are skipped, so one call can permute a single
    named vector family (e.g. every BN running_mean) at a time."""
    new = {k: v.copy() for k, v in store.items()}  # planner.py:655
    # step 1: producer rows (planner.py:661-673)
    for p in plan.producers:
        width = widths_out[p]
        rows = tuple(plan.producer_orders.get(p, range(width)))
        if kinds[p] == "input" or p not in new:
            continue
        if rows != tuple(range(width)):
            new[p] = new[p][list(rows)]
        for local in plan.zero_rows.get(p, ()):
            new[p][rows.index(local)] = 0.0
    # step 4: per-channel vectors (planner.py:731-733)
    for u, perm in sorted(plan.per_channel.items()):
        if u in new:
            new[u] = new[u][list(perm)]
    # step 5: consumer columns (planner.py:755-767)
    for acc in plan.consumers:
        c = acc.consumer
        perm = tuple(acc.perm)
        if c not in new:
            continue
        if perm != tuple(range(widths_in[c])):
            new[c] = new[c][:, list(perm)]
        for local in plan.zero_columns.get(c, ()):
            new[c][:, perm.index(local)] = 0.0
    return new


def apply_plans_weights(plans, graph, store: Mapping[str, np.ndarray]) -> dict[str, np.ndarray]:
    """All plans in order; `graph` is the ORIGINAL IR graph (duck-typed).
    Widths are tracked as the reference's sequential rewrite changes them."""
    out_w = {lay.id: lay.out_channels for lay in graph.layers}
    in_w = {lay.id: lay.in_channels for lay in graph.layers}
    kinds = {lay.id: (lay.kind.value if hasattr(lay.kind, "value") else str(lay.kind)) for lay in graph.layers}
    cur = {k: np.asarray(v) for k, v in store.items()}
    for plan in plans:
        cur = apply_plan_weights(plan, out_w, in_w, kinds, cur)
        for p in plan.producers:
            if kinds[p] != "input" and p in plan.producer_orders:
                out_w[p] = len(plan.producer_orders[p])
        for acc in plan.consumers:
            in_w[acc.consumer] = len(acc.perm)
    return cur


def apply_plans_spatial(plans, graph, weights, vectors):
    """Exported 4-D sidecar: CHANNEL_MIX tensors (torch, any rank >= 2) and every
    named PER_CHANNEL vector family permuted through the same plans."""
    import torch

    mix = apply_plans_weights(plans, graph, {k: v.detach().double().cpu().numpy() for k, v in weights.items()})
    names = sorted({n for vv in vectors.values() for n in vv})
    vec: dict = {k: {} for k in vectors}
    for n in names:
        fam = {k: vv[n].detach().double().cpu().numpy() for k, vv in vectors.items() if n in vv}
        for k, v in apply_plans_weights(plans, graph, fam).items():
            vec[k][n] = torch.from_numpy(v)
    return {k: torch.from_numpy(v) for k, v in mix.items()}, vec
