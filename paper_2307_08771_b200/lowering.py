"""torch.fx lowering: a torchvision CNN -> reference IR + spatial sidecar.

The reference IR is channel-exact and spatially collapsed (graph.py:1-9): a
convolution is a CHANNEL_MIX matrix.  Planning only needs that view, so the
lowering emits
  * the IR graph (node ids = fx node names, edge order = argument order),
  * the 2-D proxy weights the reference scores masks on (conv: the L2 norm of
    each (out, in) filter slice over kh x kw; linear: W itself), and
  * a sidecar that keeps what the IR drops: 4-D conv weights, BN statistics,
    kernel/stride/padding and the concrete PASS_THROUGH op.

Mapping: Conv2d/Linear -> CHANNEL_MIX (+ a
PER_CHANNEL "<id>.bias" node if biased); BatchNorm2d -> PER_CHANNEL;
ReLU/MaxPool/AvgPool/flatten -> PASS_THROUGH; add -> ADD; cat -> CONCAT (a
one-input cat -> PASS_THROUGH, since the reference rejects 1-input CONCAT,
graph.py:224-225).
"""

from __future__ import annotations

import operator
from dataclasses import dataclass, field

import numpy as np
import torch
import torch.fx
import torch.nn as nn

from .ir import Layer, LayerKind, ModelGraph


@dataclass(frozen=True)
class OpSpec:
    op: str  # input|conv|linear|bn|bias|dwconv|relu|relu6|hardswish|hardsigmoid|silu|sigmoid|maxpool|avgpool|
    #          avgpool_k|flatten|identity|add|mul|concat|output
    kernel: int = 1
    stride: int = 1
    pad: int = 0
    eps: float = 1e-5


@dataclass
class SpatialModel:
    """IR graph + the spatial sidecar keyed by the same layer ids."""

    graph: ModelGraph
    specs: dict[str, OpSpec]
    weights: dict[str, torch.Tensor] = field(default_factory=dict)  # CHANNEL_MIX -> [O, I, kh, kw] fp32
    vectors: dict[str, dict[str, torch.Tensor]] = field(default_factory=dict)  # PER_CHANNEL -> named vectors
    input_chw: tuple[int, int, int] = (3, 224, 224)

    def proxy_weights(self) -> dict[str, np.ndarray]:
        """The reference WeightStore content (float64, graph.py:150-161)."""
        out: dict[str, np.ndarray] = {}
        for lid, w in self.weights.items():
            w64 = w.detach().to(torch.float64).cpu()
            if self.specs[lid].op == "linear":
                out[lid] = w64[:, :, 0, 0].numpy()
            else:
                out[lid] = torch.sqrt((w64 * w64).sum(dim=(2, 3))).numpy()
        for lid, vec in self.vectors.items():
            if "dw" in vec:  # depthwise filter bank: one L2 norm per channel (a (C,) vector)
                w64 = vec["dw"].detach().to(torch.float64).cpu()
                out[lid] = torch.sqrt((w64 * w64).sum(dim=1)).numpy()
            else:
                out[lid] = vec["bias"].detach().to(torch.float64).cpu().numpy()
        return out


ACT_MODULES = {nn.ReLU: "relu", nn.ReLU6: "relu6", nn.Hardswish: "hardswish", nn.Hardsigmoid: "hardsigmoid",
               nn.SiLU: "silu", nn.Sigmoid: "sigmoid"}


def _is_add(node: torch.fx.Node) -> bool:
    if node.op == "call_function" and node.target in (operator.add, torch.add, operator.iadd):
        return True
    return node.op == "call_method" and node.target in ("add", "add_")


def lower(model: nn.Module, input_chw=(3, 224, 224)) -> SpatialModel:
    """Lower an eval-mode torchvision CNN (ResNet/DenseNet family)."""
    model = model.eval()
    gm = torch.fx.symbolic_trace(model)
    mods = dict(gm.named_modules())
    layers: list[Layer] = []
    edges: list[tuple[str, str]] = []
    specs: dict[str, OpSpec] = {}
    weights: dict[str, torch.Tensor] = {}
    vectors: dict[str, dict[str, torch.Tensor]] = {}
    width: dict[str, int] = {}  # fx node name -> IR id of its value
    alias: dict[str, str] = {}  # fx node -> IR node producing its value

    def add_layer(lid, kind, cin, cout, spec, srcs):
        layers.append(Layer(lid, kind, cin, cout))
        specs[lid] = spec
        for s in srcs:
            edges.append((s, lid))
        width[lid] = cout

    def src(arg) -> str:
        return alias[arg.name]

    for node in gm.graph.nodes:
        if node.op == "placeholder":
            c = input_chw[0]
            add_layer(node.name, LayerKind.INPUT, c, c, OpSpec("input"), [])
            alias[node.name] = node.name
        elif node.op == "call_module":
            m = mods[node.target]
            s = src(node.args[0])
            cin = width[s]
            if isinstance(m, nn.Conv2d) and m.groups != 1:
                # depthwise (groups == channels, multiplier 1): channel-wise, so a PER_CHANNEL-like
                # interior node whose "vector" is the filter bank; the planner
                # permutes it with the channel order like a BN vector
                if not (m.groups == m.in_channels == m.out_channels == cin):
                    raise NotImplementedError(f"{node.name}: grouped conv other than depthwise")
                assert m.kernel_size[0] == m.kernel_size[1] and m.stride[0] == m.stride[1]
                assert m.padding[0] == m.padding[1] and m.dilation == (1, 1)
                add_layer(node.name, LayerKind.PER_CHANNEL, cin, cin,
                          OpSpec("dwconv", m.kernel_size[0], m.stride[0], m.padding[0]), [s])
                vec = {"dw": m.weight.detach().float().reshape(cin, -1).contiguous()}
                if m.bias is not None:
                    vec["bias"] = m.bias.detach().float()
                vectors[node.name] = vec
                alias[node.name] = node.name
            elif isinstance(m, nn.Conv2d):
                assert m.kernel_size[0] == m.kernel_size[1] and m.stride[0] == m.stride[1]
                assert m.padding[0] == m.padding[1] and m.dilation == (1, 1) and cin == m.in_channels
                add_layer(node.name, LayerKind.CHANNEL_MIX, cin, m.out_channels,
                          OpSpec("conv", m.kernel_size[0], m.stride[0], m.padding[0]), [s])
                weights[node.name] = m.weight.detach().float().contiguous()
                alias[node.name] = node.name
                if m.bias is not None:
                    bid = f"{node.name}.bias"
                    add_layer(bid, LayerKind.PER_CHANNEL, m.out_channels, m.out_channels, OpSpec("bias"), [node.name])
                    vectors[bid] = {"bias": m.bias.detach().float()}
                    alias[node.name] = bid
            elif isinstance(m, nn.Linear):
                assert cin == m.in_features
                add_layer(node.name, LayerKind.CHANNEL_MIX, cin, m.out_features, OpSpec("linear"), [s])
                weights[node.name] = m.weight.detach().float().reshape(m.out_features, m.in_features, 1, 1).contiguous()
                alias[node.name] = node.name
                if m.bias is not None:
                    bid = f"{node.name}.bias"
                    add_layer(bid, LayerKind.PER_CHANNEL, m.out_features, m.out_features, OpSpec("bias"), [node.name])
                    vectors[bid] = {"bias": m.bias.detach().float()}
                    alias[node.name] = bid
            elif isinstance(m, nn.BatchNorm2d):
                add_layer(node.name, LayerKind.PER_CHANNEL, cin, cin, OpSpec("bn", eps=float(m.eps)), [s])
                vectors[node.name] = {"weight": m.weight.detach().float(), "bias": m.bias.detach().float(),
                                      "mean": m.running_mean.detach().float(), "var": m.running_var.detach().float()}
                alias[node.name] = node.name
            elif isinstance(m, tuple(ACT_MODULES)):
                op = next(v for t, v in ACT_MODULES.items() if isinstance(m, t))
                add_layer(node.name, LayerKind.PASS_THROUGH, cin, cin, OpSpec(op), [s])
                alias[node.name] = node.name
            elif isinstance(m, nn.MaxPool2d):
                k, st, p = (m.kernel_size, m.stride, m.padding)
                k = k if isinstance(k, int) else k[0]
                st = st if isinstance(st, int) else st[0]
                p = p if isinstance(p, int) else p[0]
                add_layer(node.name, LayerKind.PASS_THROUGH, cin, cin, OpSpec("maxpool", k, st, p), [s])
                alias[node.name] = node.name
            elif isinstance(m, nn.AvgPool2d):
                k, st, p = (m.kernel_size, m.stride, m.padding)
                k = k if isinstance(k, int) else k[0]
                st = st if isinstance(st, int) else st[0]
                p = p if isinstance(p, int) else p[0]
                add_layer(node.name, LayerKind.PASS_THROUGH, cin, cin, OpSpec("avgpool_k", k, st, p), [s])
                alias[node.name] = node.name
            elif isinstance(m, nn.AdaptiveAvgPool2d):
                osz = m.output_size
                assert osz in (1, (1, 1)), "only global average pooling is supported"
                add_layer(node.name, LayerKind.PASS_THROUGH, cin, cin, OpSpec("avgpool"), [s])
                alias[node.name] = node.name
            elif isinstance(m, (nn.Identity, nn.Dropout)):
                alias[node.name] = s
            else:
                raise NotImplementedError(f"{node.name}: module {type(m).__name__}")
        elif node.op in ("call_function", "call_method"):
            if _is_add(node):
                ins = [src(a) for a in node.args[:2]]
                w = width[ins[0]]
                add_layer(node.name, LayerKind.ADD, w, w, OpSpec("add"), ins)
                alias[node.name] = node.name
            elif node.target in (operator.mul, torch.mul):
                # squeeze-excitation `scale * x`: a positional join of two C-wide values, i.e. an
                # ADD in the reference IR -- both operands must share one order
                ins = [src(a) for a in node.args[:2]]
                w = width[ins[0]]
                assert width[ins[1]] == w, f"{node.name}: mul of different widths"
                add_layer(node.name, LayerKind.ADD, w, w, OpSpec("mul"), ins)
                alias[node.name] = node.name
            elif getattr(node.target, "__name__", "") == "stochastic_depth":
                alias[node.name] = src(node.args[0])  # identity in eval mode
            elif node.target in (torch.flatten,) or (node.op == "call_method" and node.target in ("flatten", "view")):
                s = src(node.args[0])
                add_layer(node.name, LayerKind.PASS_THROUGH, width[s], width[s], OpSpec("flatten"), [s])
                alias[node.name] = node.name
            elif node.target in (torch.nn.functional.adaptive_avg_pool2d,):
                s = src(node.args[0])
                osz = node.args[1] if len(node.args) > 1 else node.kwargs.get("output_size")
                assert osz in (1, (1, 1)), "only global average pooling is supported"
                add_layer(node.name, LayerKind.PASS_THROUGH, width[s], width[s], OpSpec("avgpool"), [s])
                alias[node.name] = node.name
            elif node.target in (torch.relu, torch.nn.functional.relu):
                s = src(node.args[0])
                add_layer(node.name, LayerKind.PASS_THROUGH, width[s], width[s], OpSpec("relu"), [s])
                alias[node.name] = node.name
            elif node.target is torch.cat:
                ins = [src(a) for a in node.args[0]]
                if len(ins) == 1:
                    add_layer(node.name, LayerKind.PASS_THROUGH, width[ins[0]], width[ins[0]], OpSpec("identity"), ins)
                else:
                    w = sum(width[i] for i in ins)
                    add_layer(node.name, LayerKind.CONCAT, w, w, OpSpec("concat"), ins)
                alias[node.name] = node.name
            else:
                raise NotImplementedError(f"{node.name}: {node.op} {node.target}")
        elif node.op == "output":
            s = src(node.args[0])
            add_layer("output", LayerKind.OUTPUT, width[s], width[s], OpSpec("output"), [s])
        else:
            raise NotImplementedError(f"{node.name}: {node.op}")
    return SpatialModel(ModelGraph(layers, edges), specs, weights, vectors, tuple(input_chw))


def randomize_bn(sm: SpatialModel, seed: int = 0) -> None:
    """Non-trivial BN statistics, so a mis-permuted per-channel vector shows up
    in parity tests (default init gamma=1, beta=0, mean=0, var=1 hides it)."""
    g = torch.Generator().manual_seed(seed)
    for lid in sorted(sm.vectors):
        v = sm.vectors[lid]
        if "mean" not in v:
            continue
        n = v["bias"].numel()
        v["weight"] = 0.5 + torch.rand(n, generator=g)
        v["bias"] = 0.2 * torch.randn(n, generator=g)
        v["mean"] = 0.2 * torch.randn(n, generator=g)
        v["var"] = 0.5 + torch.rand(n, generator=g)
