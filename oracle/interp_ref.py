"""Oracle: the reference interpreter restated in numpy (interp.py:36-121).

One float64 activation vector per node, evaluated in the reference's Kahn
order (graph.py:128-147).  Masks simulate pruning on the original model:
input-side masks zero a consumer's input channels right before its matrix
(interp.py:59-60).  Graphs are duck-typed (ours or the reference's).
"""

from __future__ import annotations

from typing import Mapping

import numpy as np

DEFAULT_TOLERANCE = 1e-9  # interp.py:18
DEFAULT_TRIALS = 8  # interp.py:19


def _kind(lay) -> str:
    return lay.kind.value if hasattr(lay.kind, "value") else str(lay.kind)


def run(graph, weights: Mapping[str, np.ndarray], x, masks=None, mask_side: str = "input") -> np.ndarray:
    """interp.py:36-84."""
    x = np.asarray(x, dtype=np.float64)
    masks = masks or {}
    inputs = [lay.id for lay in graph.layers if _kind(lay) == "input"]
    outputs = [lay.id for lay in graph.layers if _kind(lay) == "output"]
    assert len(inputs) == 1 and len(outputs) == 1, "interpreter needs one input and one output"
    vals: dict[str, np.ndarray] = {}
    for lid in graph.topological_order():
        lay = graph.layer(lid)
        k = _kind(lay)
        ins = [vals[p] for p in graph.predecessors(lid)]
        if k == "input":
            out = x
        elif k == "channel_mix":
            v = ins[0]
            if mask_side == "input" and lid in masks:
                m = np.zeros(len(v))
                m[list(masks[lid])] = 1.0
                v = v * m
            out = weights[lid] @ v
            if mask_side == "output" and lid in masks:
                m = np.zeros(len(out))
                m[list(masks[lid])] = 1.0
                out = out * m
        elif k == "add":
            out = np.sum(ins, axis=0)
        elif k == "concat":
            out = np.concatenate(ins)
        elif k == "pass_through":
            out = np.maximum(0.0, ins[0])
        elif k == "per_channel":
            out = ins[0] + weights[lid]
        elif k == "slice":
            s, n = lay.params
            out = ins[0][s:s + n]
        elif k == "gather":
            out = np.array([ins[0][i] if i >= 0 else 0.0 for i in lay.params])
        else:
            out = ins[0]
        assert out.shape == (lay.out_channels,), f"{lid}: shape {out.shape}"
        vals[lid] = out
    return vals[outputs[0]]


def deviation(a: np.ndarray, b: np.ndarray) -> float:
    """The reference's equivalence metric (interp.py:119-120)."""
    scale = np.maximum(1.0, np.maximum(np.abs(a), np.abs(b)))
    return float(np.max(np.abs(a - b) / scale))


def check_equivalence(g0, w0, masks, g1, w1, trials=DEFAULT_TRIALS, seed=0, mask_side="input") -> float:
    """interp.py:98-121: max deviation over standard-normal inputs (seed 0)."""
    n_in = next(lay.out_channels for lay in g0.layers if _kind(lay) == "input")
    rng = np.random.default_rng(seed)
    worst = 0.0
    for _ in range(trials):
        x = rng.standard_normal(n_in)
        worst = max(worst, deviation(run(g0, w0, x, masks, mask_side), run(g1, w1, x)))
    return worst
