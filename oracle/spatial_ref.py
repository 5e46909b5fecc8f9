"""Oracle: interp.run's op dispatch (interp.py:52-83) over real spatial tensors.

Same topological schedule and per-kind semantics as the reference
interpreter; the channel-collapsed ops are replaced by their spatial
originals from the lowering sidecar (CHANNEL_MIX -> conv2d / linear,
PER_CHANNEL -> BatchNorm or bias, PASS_THROUGH -> relu / max pool / global
average pool / flatten).  Activations are [N, C, H, W] torch CPU tensors in
float64 (parity anchor) or float32 (the timed CPU reference path).  A graph
without specs (e.g. the reference's random DAG fixtures) runs with the
reference's 1x1 semantics (PASS_THROUGH = ReLU, PER_CHANNEL = + vector).
"""

from __future__ import annotations

from typing import Mapping

import torch
import torch.nn.functional as F


_ACTS = {"relu": torch.relu, "relu6": lambda v: v.clamp(0.0, 6.0), "hardswish": F.hardswish,
         "hardsigmoid": F.hardsigmoid, "silu": F.silu, "sigmoid": torch.sigmoid}


def _kind(lay) -> str:
    return lay.kind.value if hasattr(lay.kind, "value") else str(lay.kind)


def run_spatial(graph, specs: Mapping, weights: Mapping[str, torch.Tensor],
                vectors: Mapping[str, Mapping[str, torch.Tensor]], x: torch.Tensor,
                masks: Mapping[str, tuple] | None = None, dtype=torch.float64, values: dict | None = None,
                store_dtype=None) -> torch.Tensor:
    """Returns the OUTPUT node's value ([N, C] if spatially collapsed).  If
    `values` is a dict it receives every node's output (debugging aid).
    `store_dtype` (e.g. torch.bfloat16): every node's output is rounded to it and back
    -- the reference evaluated at a GPU's storage precision (a precision control for
    the parity tests, not a model of any particular kernel fusion)."""
    masks = masks or {}
    vals: dict[str, torch.Tensor] = {}
    out_id = None
    # values are dropped after their last reader (bounded memory at large batches)
    readers = {lid: len(graph.successors(lid)) for lid in graph.topological_order()}
    for lid in graph.topological_order():
        lay = graph.layer(lid)
        k = _kind(lay)
        spec = specs.get(lid)
        op = spec.op if spec is not None else None
        ins = [vals[p] for p in graph.predecessors(lid)]
        if k == "input":
            out = x.to(dtype)
        elif k == "channel_mix":
            v = ins[0]
            if lid in masks:  # interp.py:59-60
                m = torch.zeros(v.shape[1], dtype=dtype)
                m[list(masks[lid])] = 1.0
                v = v * m.view(1, -1, 1, 1)
            w = weights[lid].to(dtype)
            if op == "conv":
                out = F.conv2d(v, w, stride=spec.stride, padding=spec.pad)
            else:  # linear / 1x1 channel mix over a collapsed tensor
                out = F.conv2d(v, w)
        elif k == "add" and op == "mul":  # squeeze-excitation gate (lowered to a positional ADD)
            out = ins[0] * ins[1]
        elif k == "add":
            out = ins[0]
            for t in ins[1:]:
                out = out + t
        elif k == "concat":
            out = torch.cat(ins, dim=1)
        elif k == "pass_through":
            v = ins[0]
            if op == "maxpool":
                out = F.max_pool2d(v, spec.kernel, spec.stride, spec.pad)
            elif op == "avgpool":
                out = v.mean(dim=(2, 3), keepdim=True)
            elif op == "avgpool_k":
                out = F.avg_pool2d(v, spec.kernel, spec.stride, spec.pad)
            elif op in ("flatten", "identity"):
                out = v
            elif op in _ACTS:
                out = _ACTS[op](v)
            else:  # relu, and the reference's PASS_THROUGH semantics
                out = torch.clamp_min(v, 0.0)
        elif k == "per_channel":
            vec = vectors[lid]
            if op == "dwconv":  # depthwise conv lowered to a channel-wise node
                C = ins[0].shape[1]
                w = vec["dw"].to(dtype).view(C, 1, spec.kernel, spec.kernel)
                b = vec["bias"].to(dtype) if "bias" in vec else None
                out = F.conv2d(ins[0], w, b, stride=spec.stride, padding=spec.pad, groups=C)
            elif op == "bn":
                scale = vec["weight"].to(dtype) / torch.sqrt(vec["var"].to(dtype) + spec.eps)
                out = (ins[0] - vec["mean"].to(dtype).view(1, -1, 1, 1)) * scale.view(1, -1, 1, 1) \
                    + vec["bias"].to(dtype).view(1, -1, 1, 1)
            else:  # bias / the reference's "+ vector"
                out = ins[0] + vec["bias"].to(dtype).view(1, -1, 1, 1)
        elif k == "slice":
            s, n = lay.params
            out = ins[0][:, s:s + n]
        elif k == "gather":
            v = ins[0]
            idx = torch.tensor([max(i, 0) for i in lay.params], dtype=torch.long)
            out = v.index_select(1, idx)
            neg = [j for j, i in enumerate(lay.params) if i < 0]
            if neg:
                out[:, neg] = 0.0
        elif k == "output":
            out = ins[0]
            out_id = lid
        else:
            raise ValueError(f"{lid}: unknown kind {k}")
        if store_dtype is not None and k != "output":
            out = out.to(store_dtype).to(dtype)
        if out.shape[1] != lay.out_channels:
            raise ValueError(f"{lid}: produced {out.shape[1]} channels, expected {lay.out_channels}")
        vals[lid] = out
        if values is None:
            for p in graph.predecessors(lid):
                readers[p] -= 1
                if readers[p] == 0 and p in vals and _kind(graph.layer(p)) != "output":
                    del vals[p]
    if values is not None:
        values.update(vals)
    res = vals[out_id]
    if res.dim() == 4 and res.shape[2] == 1 and res.shape[3] == 1:
        res = res[:, :, 0, 0]
    return res


def deviation(a: torch.Tensor, b: torch.Tensor) -> float:
    """interp.py:119-120 over all elements."""
    a = a.double()
    b = b.double()
    scale = torch.clamp_min(torch.maximum(a.abs(), b.abs()), 1.0)
    return float(((a - b).abs() / scale).max())


def top1_agreement(a: torch.Tensor, b: torch.Tensor) -> float:
    return float((a.argmax(dim=1) == b.argmax(dim=1)).double().mean())
