"""Inference engine: executes an exported IR graph on B200 with fused kernels.

This is the spatial, batched twin of the reference interpreter `run`
(interp.py:36-84).  The graph is compiled once into a launch schedule:

  * CHANNEL_MIX + its `<c>.read` node + its epilogue chain
      (PER_CHANNEL bias/BN -> ADD -> ReLU, each single-consumer) -> ONE
      `ub_conv_fwd` launch.  SLICE reads are channel-offset views (zero copy);
      GATHER reads are fused into the A-operand staging (gather_mode="fused")
      or materialised by `ub_channel_gather` first (gather_mode="copy", the
      baseline export's copy-then-conv behaviour).
  * BN scale is folded into the weight rows at compile time (one permute
    kernel pass per layer writes the bf16 K-major GEMM operand).
  * INPUT (+ a GATHER reading it) -> `ub_stage_input`; max/avg pools and any
    node the conv epilogue cannot absorb -> standalone kernels.
  * The op list is topologically scheduled (residual producers first), every
    value gets its own NHWC buffer, and the whole forward can be captured in a
    CUDA graph.
"""

from __future__ import annotations

import os
import ctypes
from dataclasses import dataclass, field
from typing import Callable, Mapping, Sequence

import torch

from . import _lib
from . import kernels as K
from .ir import LayerKind, ModelGraph

# PASS_THROUGH ops that are activations (ub_eltwise act codes, _lib.UB_ACT)
ACTS = ("relu", "relu6", "hardswish", "hardsigmoid", "silu", "sigmoid")


@dataclass
class _Op:
    kind: str                     # conv | stage | gather | maxpool | avgpool | eltwise
    anchor: str                   # node id giving the topological position
    inputs: list[str]             # value ids read
    output: str                   # value id written
    launch: Callable[[], None] | None = None
    info: dict = field(default_factory=dict)


@dataclass
class ConvStats:
    """Algorithmic work of one conv launch (SURVEY.md 8d formulas)."""

    name: str
    flops: float
    bytes: float
    gather_bytes: float


class Engine:
    """Compiled forward pass of one exported graph at a fixed batch size.

    weight_source(lid) -> (W [O,I,kh,kw] fp32 device tensor, rows, cols)
    vector_source(uid) -> (named vectors dict on CPU/device, perm or None)
    `rows`/`cols`/`perm` are the composed plan index maps (None = identity).
    """

    def __init__(self, graph: ModelGraph, specs: Mapping, weight_source, vector_source, batch: int,
                 input_chw=(3, 224, 224), device="cuda", gather_mode: str = "fused", fuse_stem: bool = True,
                 stem_s2d: bool = True, stem_pool: bool = True, cover_ratio: float = 2.5,
                 dual_store: bool = False, stem_pack_fused: bool = False, pool_gather: bool = True,
                 se_fuse: bool = True):
        assert gather_mode in ("fused", "copy")
        self.fuse_stem = fuse_stem
        self.stem_s2d = stem_s2d
        self.stem_pool = stem_pool
        self.cover_ratio = cover_ratio
        self.dual_store = dual_store
        self.stem_pack_fused = stem_pack_fused
        self.pool_gather = pool_gather
        self.se_fuse = se_fuse
        self.graph = graph
        # nodes the reference's apply_plan adds (join-rewrite ADD / CONCAT runs, SLICE / GATHER
        # reads) carry no spatial spec: they get the plain op of their kind
        from .lowering import OpSpec
        defaults = {LayerKind.ADD: "add", LayerKind.CONCAT: "concat", LayerKind.SLICE: "slice",
                    LayerKind.GATHER: "gather"}
        self.specs = dict(specs)
        for lay in graph.layers:
            if lay.id not in self.specs and lay.kind in defaults:
                self.specs[lay.id] = OpSpec(defaults[lay.kind])
        self.batch = batch
        self.device = torch.device(device)
        self.gather_mode = gather_mode
        self.input_chw = tuple(input_chw)
        self.values: dict[str, K.Act] = {}
        self.ops: list[_Op] = []
        self.conv_stats: list[ConvStats] = []
        self._keep: list[torch.Tensor] = []  # device tensors referenced by launches
        self._graph_exec = None
        self._shapes = self._infer_shapes()
        self._compile(weight_source, vector_source)
        bad = _lib.index_faults() if self.device.type == "cuda" else 0
        if bad:
            raise ValueError(f"engine: {bad} plan indices outside their source tensors")

    # ------------------------------------------------------------------ shapes
    def _infer_shapes(self) -> dict[str, tuple[int, int, int]]:
        g, sp = self.graph, self.specs
        shp: dict[str, tuple[int, int, int]] = {}
        for lid in g.topological_order():
            lay = g.layer(lid)
            preds = g.predecessors(lid)
            spec = sp.get(lid)
            if lay.kind is LayerKind.INPUT:
                c, h, w = self.input_chw
                shp[lid] = (lay.out_channels, h, w)
                continue
            _, h, w = shp[preds[0]]
            if lay.kind is LayerKind.ADD:  # an SE `mul` broadcasts its [N, C, 1, 1] gate
                h, w = max(shp[q][1] for q in preds), max(shp[q][2] for q in preds)
            if lay.kind is LayerKind.CHANNEL_MIX and spec is not None and spec.op == "conv":
                h = (h + 2 * spec.pad - spec.kernel) // spec.stride + 1
                w = (w + 2 * spec.pad - spec.kernel) // spec.stride + 1
            elif lay.kind is LayerKind.CHANNEL_MIX:
                assert (h, w) == (1, 1), f"{lid}: linear layer on a spatial tensor"
            elif lay.kind is LayerKind.PER_CHANNEL and spec is not None and spec.op == "dwconv":
                h = (h + 2 * spec.pad - spec.kernel) // spec.stride + 1
                w = (w + 2 * spec.pad - spec.kernel) // spec.stride + 1
            elif lay.kind is LayerKind.PASS_THROUGH and spec is not None:
                if spec.op == "maxpool":
                    h = (h + 2 * spec.pad - spec.kernel) // spec.stride + 1
                    w = (w + 2 * spec.pad - spec.kernel) // spec.stride + 1
                elif spec.op == "avgpool":
                    h, w = 1, 1
                elif spec.op == "avgpool_k":
                    h = (h + 2 * spec.pad - spec.kernel) // spec.stride + 1
                    w = (w + 2 * spec.pad - spec.kernel) // spec.stride + 1
            shp[lid] = (lay.out_channels, h, w)
        return shp

    # ------------------------------------------------------------------ helpers
    def _single_succ(self, lid: str) -> str | None:
        s = self.graph.successors(lid)
        return s[0] if len(s) == 1 else None

    def _alloc(self, vid: str, C: int, fp32: bool = False, shape_of: str | None = None,
               cmap: tuple | None = None) -> K.Act:
        _, h, w = self._shapes[shape_of or vid]
        if vid in getattr(self, "_place", {}):  # the value is a band of a zero-copy concat
            assert not fp32 and cmap is None
            key, off = self._place[vid]
            a = K.Act(self._band_buffer(key), self.batch, h, w, C, off)
            self.values[vid] = a
            return a
        width = C if cmap is None else (cmap[-1] + 1)
        cs = K.pad8(width) if not fp32 else (width + 3) // 4 * 4
        buf = torch.zeros((self.batch * h * w, cs), dtype=torch.float32 if fp32 else torch.bfloat16,
                          device=self.device)
        a = K.Act(buf, self.batch, h, w, C, 0, cmap)
        self.values[vid] = a
        return a

    def _act_code(self, node: str | None) -> int:
        if node is None:
            return 0
        return _lib.UB_ACT[self.specs[node].op]

    def _f32(self, seq) -> torch.Tensor:
        t = torch.as_tensor(list(seq), dtype=torch.float32, device=self.device)
        self._keep.append(t)
        return t

    def _i32(self, seq) -> torch.Tensor:
        t = torch.as_tensor(list(seq), dtype=torch.int32, device=self.device)
        self._keep.append(t)
        return t

    # ------------------------------------------------------------------ compile
    def _compile(self, weight_source, vector_source):
        g = self.graph
        kinds = {lay.id: lay.kind for lay in g.layers}
        absorbed: set[str] = set()   # nodes executed inside another op
        alias: dict[str, tuple[str, int, int]] = {}  # value -> (base value, start, length) views
        ops: list[_Op] = []
        topo = g.topological_order()
        pos = {lid: i for i, lid in enumerate(topo)}
        output_feed = {g.predecessors(lid)[0] for lid in topo if kinds[lid] is LayerKind.OUTPUT}

        # --- conv groups -------------------------------------------------------
        for lid in topo:
            if kinds[lid] is not LayerKind.CHANNEL_MIX:
                continue
            spec = self.specs[lid]
            read = g.predecessors(lid)[0]
            info = {"conv": lid, "read": None, "bn": None, "add": None, "relu": None}
            src = read
            if kinds[read] in (LayerKind.SLICE, LayerKind.GATHER) and read.endswith(".read") \
                    and len(g.successors(read)) == 1:
                info["read"] = read
                src = g.predecessors(read)[0]
                absorbed.add(read)
            # pre-activation prologue (DenseNet: norm -> relu -> conv.read -> conv): a BN and/or
            # ReLU between the value and this conv's read, read by nothing else and not already
            # absorbed by its producer's epilogue, is applied while the read stages the operand
            pro_bn = pro_relu = None
            s_ = src
            if (kinds[s_] is LayerKind.PASS_THROUGH and self.specs[s_].op == "relu" and s_ not in absorbed
                    and len(g.successors(s_)) == 1 and s_ not in output_feed):
                pro_relu, s_ = s_, g.predecessors(s_)[0]
            if (kinds[s_] is LayerKind.PER_CHANNEL and self.specs[s_].op in ("bn", "bias") and s_ not in absorbed
                    and len(g.successors(s_)) == 1 and s_ not in output_feed):
                pro_bn, s_ = s_, g.predecessors(s_)[0]
            # ... unless the value comes straight from a conv / depthwise conv, whose epilogue
            # takes the BN and activation instead (MobileNet: dw -> bn -> act -> conv)
            src_k = kinds[s_]
            fusable_src = ((src_k is LayerKind.CHANNEL_MIX or (src_k is LayerKind.PER_CHANNEL
                                                                and self.specs[s_].op == "dwconv"))
                           and len(g.successors(s_)) == 1)
            if (pro_bn or pro_relu) and not fusable_src:
                info["prologue"] = (pro_bn, pro_relu)
                absorbed.update(x for x in (pro_bn, pro_relu) if x)
                src = s_
            cur = lid
            nxt = self._single_succ(cur)
            if nxt is not None and kinds[nxt] is LayerKind.PER_CHANNEL and cur not in output_feed:
                info["bn"] = nxt
                absorbed.add(nxt)
                cur = nxt
                nxt = self._single_succ(cur)
            if nxt is not None and kinds[nxt] is LayerKind.ADD and len(g.predecessors(nxt)) == 2 \
                    and nxt not in absorbed and cur not in output_feed:
                others = [p for p in g.predecessors(nxt) if p != cur]
                if len(others) == 1:
                    info["add"] = nxt
                    info["residual"] = others[0]
                    absorbed.add(nxt)
                    cur = nxt
                    nxt = self._single_succ(cur)
            if nxt is not None and kinds[nxt] is LayerKind.PASS_THROUGH and self.specs[nxt].op in ACTS \
                    and cur not in output_feed:
                info["relu"] = nxt  # the epilogue activation (UB_ACT_* code; ReLU for ResNet/DenseNet)
                absorbed.add(nxt)
                cur = nxt
                nxt = self._single_succ(cur)
            # a 2x2/s2 average pool right after a 1x1/s1 conv (DenseNet transition, no ReLU in
            # between): pool and conv are both linear, so the pool moves in front of the conv
            # into the operand staging and the conv runs on a quarter of the pixels
            ps = self.specs.get(nxt) if nxt is not None else None
            if (ps is not None and ps.op == "avgpool_k" and (ps.kernel, ps.stride, ps.pad) == (2, 2, 0)
                    and info["relu"] is None and info["add"] is None and cur not in output_feed
                    and spec.op == "conv" and (spec.kernel, spec.stride, spec.pad) == (1, 1, 0)):
                info["pool2"] = nxt
                absorbed.add(nxt)
                cur = nxt
            info["src"] = src
            info["out"] = cur
            inputs = [src] + ([info["residual"]] if info.get("residual") else [])
            ops.append(_Op("conv", lid, inputs, cur, info=info))
            del spec

        # --- remaining nodes ---------------------------------------------------
        for lid in topo:
            k = kinds[lid]
            if lid in absorbed or k is LayerKind.CHANNEL_MIX:
                continue
            spec = self.specs.get(lid)
            preds = g.predecessors(lid)
            if k is LayerKind.INPUT:
                succ = g.successors(lid)
                idx = None
                out = lid
                # fused stem: the only reader of the model input is one spatial conv (directly or
                # through its GATHER read) -> im2col from the fp32 input inside the conv kernel
                stem_op = None
                for op in ops:
                    if op.kind == "conv" and op.info["src"] == lid and self.specs[op.anchor].op == "conv":
                        stem_op = op
                if stem_op is not None and len(succ) == 1 and self.fuse_stem:
                    rd = stem_op.info["read"]
                    if rd is not None and kinds[rd] is LayerKind.GATHER:
                        stem_op.info["stem_idx"] = g.layer(rd).params
                    elif rd is None:
                        stem_op.info["stem_idx"] = tuple(range(g.layer(lid).out_channels))
                    if "stem_idx" in stem_op.info:
                        stem_op.info["read"] = None
                        stem_op.inputs = []
                        continue
                if len(succ) == 1 and kinds[succ[0]] is LayerKind.GATHER:
                    idx = g.layer(succ[0]).params
                    out = succ[0]
                    absorbed.add(succ[0])
                    # the conv that read this gather now reads the staged tensor
                    for op in ops:
                        if op.info.get("read") == succ[0]:
                            op.info["read"] = None
                            op.info["src"] = out
                            op.inputs[0] = out
                ops.append(_Op("stage", lid, [], out, info={"idx": idx}))
            elif k is LayerKind.OUTPUT:
                alias[lid] = (preds[0], 0, -1)
            elif k is LayerKind.PASS_THROUGH and spec is not None and spec.op in ("flatten", "identity"):
                alias[lid] = (preds[0], 0, -1)
            elif k is LayerKind.SLICE:
                s, n = g.layer(lid).params
                alias[lid] = (preds[0], s, n)
            elif k is LayerKind.PASS_THROUGH and spec is not None and spec.op == "maxpool":
                ops.append(_Op("maxpool", lid, [preds[0]], lid, info={"spec": spec}))
            elif k is LayerKind.PASS_THROUGH and spec is not None and spec.op == "avgpool":
                ops.append(_Op("avgpool", lid, [preds[0]], lid))
            elif k is LayerKind.PASS_THROUGH and spec is not None and spec.op == "avgpool_k":
                ops.append(_Op("avgpool2d", lid, [preds[0]], lid, info={"spec": spec}))
            elif k is LayerKind.GATHER:
                ops.append(_Op("gather", lid, [preds[0]], lid, info={"idx": g.layer(lid).params}))
            elif k is LayerKind.PER_CHANNEL and spec is not None and spec.op == "dwconv":
                # depthwise conv + its BN + activation in one launch (ub_dwconv)
                info = {"bn": None, "act": None}
                cur = lid
                nxt = self._single_succ(cur)
                if (nxt is not None and nxt not in absorbed and kinds[nxt] is LayerKind.PER_CHANNEL
                        and self.specs[nxt].op == "bn" and cur not in output_feed):
                    info["bn"] = nxt
                    absorbed.add(nxt)
                    cur = nxt
                    nxt = self._single_succ(cur)
                if (nxt is not None and nxt not in absorbed and kinds[nxt] is LayerKind.PASS_THROUGH
                        and self.specs[nxt].op in ACTS and cur not in output_feed):
                    info["act"] = nxt
                    absorbed.add(nxt)
                    cur = nxt
                ops.append(_Op("dwconv", lid, [preds[0]], cur, info=info))
            elif k is LayerKind.CONCAT:
                # zero-copy when every operand can be stored straight into its band (_plan_concats)
                ops.append(_Op("concat", lid, list(preds), lid))
            elif k in (LayerKind.PASS_THROUGH, LayerKind.PER_CHANNEL, LayerKind.ADD):
                info = {"kind": k}
                out = lid
                # a standalone BN / add followed by its only reader, an activation: one pass
                nxt = self._single_succ(lid)
                if (k is not LayerKind.PASS_THROUGH and nxt is not None and nxt not in absorbed
                        and kinds[nxt] is LayerKind.PASS_THROUGH and self.specs[nxt].op in ACTS
                        and lid not in output_feed):
                    info["act"] = self.specs[nxt].op
                    absorbed.add(nxt)
                    out = nxt
                ops.append(_Op("eltwise", lid, list(preds), out, info=info))
            else:
                raise NotImplementedError(f"{lid}: {k.value} has no B200 kernel in this build")

        # copy-mode gathers: materialise the read before the conv
        if self.gather_mode == "copy":
            extra = []
            for op in ops:
                r = op.info.get("read") if op.kind == "conv" else None
                if r and kinds[r] is LayerKind.GATHER:
                    extra.append(_Op("gather", r, [op.info["src"]], r, info={"idx": g.layer(r).params}))
                    op.info["read"] = None
                    op.info["src"] = r
                    op.inputs[0] = r
            ops.extend(extra)

        def base(v):
            while v in alias:
                v = alias[v][0]
            return v

        # --- stem -> max pool fusion: when the space-to-depth stem's only reader is a
        # 3x3/s2/p1 max pool, the pool runs in the stem's epilogue (ub_conv_s2d_maxpool)
        if self.stem_pool:
            for sop in [o for o in ops if o.kind == "conv" and "stem_idx" in o.info]:
                readers = [o for o in ops if any(base(i) == sop.output for i in o.inputs)]
                if len(readers) != 1 or readers[0].kind != "maxpool":
                    continue
                mp = readers[0]
                sp, cs = mp.info["spec"], self.specs[sop.info["conv"]]
                _, ho, wo = self._shapes[sop.output]
                cout = g.layer(sop.info["conv"]).out_channels
                if ((sp.kernel, sp.stride, sp.pad) == (3, 2, 1) and base(mp.inputs[0]) == sop.output
                        and self._act_code(sop.info["relu"]) in (0, _lib.UB_ACT["relu"])
                        and self._s2d_ok(len(sop.info["stem_idx"]), cs, cout) and cout <= 64
                        and ho % 2 == 0 and wo % 2 == 0 and wo <= 128):
                    sop.info["pool"] = sp
                    sop.info["out"] = mp.output
                    sop.output = mp.output
                    ops.remove(mp)

        # --- squeeze-excitation gate: global pool -> fc1 (+bias, act) -> fc2 (+bias, act) whose
        # only reader is an SE `mul` becomes ONE launch (ub_se_gate, one CTA per image)
        if self.se_fuse:
            self._fuse_se(ops, base, kinds)

        # --- global avg pool -> GATHER read fusion: when a pool's only reader is a conv that
        # GATHERs its channels (ResNet: avgpool -> flatten -> fc.read -> fc), the pool writes
        # the gathered channels compacted (ub_avgpool_gather) and the conv reads them densely
        if self.pool_gather and self.gather_mode == "fused":
            for pop in [o for o in ops if o.kind == "avgpool"]:
                readers = [o for o in ops if any(base(i) == pop.output for i in o.inputs)]
                if len(readers) != 1 or readers[0].kind != "conv":
                    continue
                cop = readers[0]
                r = cop.info.get("read")
                if (r is None or kinds[r] is not LayerKind.GATHER or "stem_idx" in cop.info
                        or base(cop.info["src"]) != pop.output or cop.info.get("residual")
                        or g.layer(pop.anchor).out_channels % 8):
                    continue
                pop.info["idx"] = g.layer(r).params
                pop.output = r
                cop.info["read"] = None
                cop.info["src"] = r
                cop.inputs[0] = r

        # --- concat buffer planning (zero-copy bands)
        self._plan_concats(ops, alias, base, pos, output_feed)
        ops = [op for op in ops if not (op.kind == "concat" and op.output in self._concat_views)]

        # --- schedule: Kahn over value dependencies, ties by topological position
        produced = {op.output: op for op in ops}

        def producers(v, seen=None):
            v = base(v)
            if v in produced:
                return {id(produced[v])}
            if v in self._concat_views:  # a zero-copy concat depends on every operand's producer
                out = set()
                for u in self._concat_views[v][3]:
                    out |= producers(u)
                return out
            return set()

        deps = {id(op): set().union(*[producers(i) for i in op.inputs]) if op.inputs else set() for op in ops}
        done: set[int] = set()
        sched: list[_Op] = []
        remaining = sorted(ops, key=lambda o: pos[o.anchor])
        while remaining:
            for i, op in enumerate(remaining):
                if deps[id(op)] <= done:
                    sched.append(op)
                    done.add(id(op))
                    remaining.pop(i)
                    break
            else:
                raise RuntimeError("engine schedule has a cycle")
        self._alias = alias
        self.ops = sched

        # --- allocate + bind launches -------------------------------------------
        self.input_buf = torch.zeros((self.batch, *self.input_chw), dtype=torch.float32, device=self.device)
        self.input_bufs = [self.input_buf]
        self._graphs: list = []
        self._plan_dual_stores()
        for op in self.ops:
            getattr(self, f"_bind_{op.kind}")(op, weight_source, vector_source, output_feed)
        out_id = next(lid for lid in topo if kinds[lid] is LayerKind.OUTPUT)
        self.output_value = self._value(out_id)

    def _fuse_se(self, ops, base, kinds) -> None:
        def readers(v):
            return [o for o in ops if any(base(i) == v for i in o.inputs)]

        for pop in [o for o in ops if o.kind == "avgpool" and "idx" not in o.info]:
            r1 = readers(pop.output)
            if len(r1) != 1 or r1[0].kind != "conv":
                continue
            a = r1[0]
            r2 = readers(a.output)
            if len(r2) != 1 or r2[0].kind != "conv":
                continue
            b = r2[0]
            r3 = readers(b.output)
            if not r3 or any(o.kind != "eltwise" or self.specs.get(o.anchor) is None or
                             self.specs[o.anchor].op != "mul" for o in r3):
                continue
            ok = all(c.info.get(k) is None for c in (a, b) for k in ("residual", "prologue", "pool2"))
            ok = ok and all(self.specs[c.info["conv"]].op in ("conv", "linear") and
                            (self.specs[c.info["conv"]].op == "linear" or
                             (self.specs[c.info["conv"]].kernel, self.specs[c.info["conv"]].stride) == (1, 1))
                            for c in (a, b))
            ok = ok and base(a.info["src"]) == pop.output and base(b.info["src"]) == a.output
            if not ok:
                continue
            se = _Op("se", pop.anchor, list(pop.inputs), b.output, info={"pool": pop, "fc1": a, "fc2": b})
            # the pool reads a depthwise conv's output: that launch also writes per-tile channel
            # sums (ub_dwconv_pool) and the gate pools from them instead of re-reading the tensor
            src = base(pop.inputs[0])
            dw = next((o for o in ops if o.kind == "dwconv" and base(o.output) == src), None)
            if dw is not None and not os.environ.get("UB_SE_NOFUSEPOOL"):
                dw.info["se_part"] = True
                se.info["dw"] = dw
            idx = ops.index(pop)
            for o in (pop, a, b):
                ops.remove(o)
            ops.insert(idx, se)

    def _linear_dense(self, op, ws, vs, src_width: int):
        """A 1x1 CHANNEL_MIX over an [N, C, 1, 1] value as a dense fp32 matrix over ALL of its
        source's channels (its SLICE / GATHER read folded in as zero columns), with the BN
        scale folded into the rows; returns (W [O, src_width], bias [O] or None, act code)."""
        info = op.info
        lid = info["conv"]
        W, rows, cols = ws(lid)
        Wf = W.detach().float().cpu()[:, :, 0, 0]
        O, I = Wf.shape
        rows = list(rows if rows is not None else range(O))
        cols = list(cols if cols is not None else range(I))
        read = info["read"]
        if read is None:
            src = list(range(len(cols)))
        else:
            rl = self.graph.layer(read)
            src = list(range(rl.params[0], rl.params[0] + rl.params[1])) if rl.kind is LayerKind.SLICE \
                else list(rl.params)
        Wd = torch.zeros(len(rows), src_width)
        for k, (c, s_) in enumerate(zip(cols, src)):
            if c >= 0 and s_ >= 0:
                Wd[:, s_] += torch.where(torch.tensor(rows) >= 0, Wf[torch.tensor(rows).clamp_min(0), c], 0.0)
        scale = bias = None
        if info["bn"] is not None:
            vec, perm = vs(info["bn"])
            scale, bias = self._affine(info["bn"], vec, perm)
            if self.specs[info["bn"]].op == "bn":
                Wd = Wd * scale.cpu().view(-1, 1)
        return Wd, bias, self._act_code(info["relu"])

    def _bind_se(self, op, ws, vs, output_feed):
        x = self._value(op.inputs[0])
        assert x.cmap is None, "SE pool over a column-mapped value"
        a, b = op.info["fc1"], op.info["fc2"]
        C = x.C
        W1, b1, act1 = self._linear_dense(a, ws, vs, C)
        C1 = W1.shape[0]
        W2, b2, act2 = self._linear_dense(b, ws, vs, C1)
        C2 = W2.shape[0]

        def pack(Wd):
            t = torch.zeros(Wd.shape[0], K.pad8(Wd.shape[1]), dtype=torch.bfloat16)
            t[:, :Wd.shape[1]] = Wd.to(torch.bfloat16)
            t = t.to(self.device).contiguous()
            self._keep.append(t)
            return t

        w1, w2 = pack(W1), pack(W2)
        gate = self._alloc(b.info["out"], C2)
        xd = self._dense(x)
        dw = op.info.get("dw")
        part, nparts = dw.info.get("part", (None, 0)) if dw is not None else (None, 0)
        op.launch = lambda: K.se_gate(xd, w1, C1, b1, act1, w2, C2, b2, act2, gate, part, nparts)
        self.conv_stats.append(ConvStats(f"{op.anchor}(se)", 0.0, 2.0 * C * x.H * x.W, 0.0))

    def _plan_concats(self, ops, alias, base, pos, output_feed) -> None:
        """CONCAT as buffer planning: each operand's producer stores its
        band straight into one shared buffer, so the concat itself launches nothing.
        Bands start on 8-channel (16-byte) boundaries -- the producers' TMA stores need
        aligned bases -- so a concat of pruned widths is a view with a column map
        (Act.cmap) over a buffer with up to 7 pad columns per band.  Concats are planned
        largest-first (reverse topological order): DenseNet's per-layer concats are
        prefixes of the block's last one and all become views of one buffer.  A concat
        whose operands cannot be placed consistently (already placed elsewhere, an
        fp32/model-input/view operand) keeps a copy op."""
        self._place: dict[str, tuple[str, int]] = {}      # value -> (buffer key, physical offset)
        self._bands: dict[str, list] = {}                  # buffer key -> [width, shape_of, occupied]
        self._concat_views: dict[str, tuple] = {}          # concat -> (key, base, cmap, operands)
        self._band_bufs: dict[str, torch.Tensor] = {}
        producer_of = {op.output: op for op in ops}
        placeable_kinds = ("conv", "maxpool", "avgpool", "avgpool2d", "eltwise", "gather", "stage", "dwconv")
        g = self.graph

        def operand(v):  # full-width aliases (identity / flatten) resolve to their base
            while v in alias and alias[v][2] < 0:
                v = alias[v][0]
            return v

        def placeable(v):
            op = producer_of.get(v)
            return (op is not None and op.kind in placeable_kinds and v not in output_feed
                    and v not in self._place and v not in alias)

        def free(key, lo, hi):
            return all(hi <= a or lo >= b for a, b in self._bands[key][2])

        for c in sorted([op for op in ops if op.kind == "concat"], key=lambda o: -pos[o.anchor]):
            ins = [operand(v) for v in c.inputs]
            widths = [g.layer(v).out_channels if v in g else self._value_width(v) for v in ins]
            offs, o = [], 0
            for w_ in widths:
                offs.append(o)
                o += (w_ + 7) // 8 * 8
            placed = [(i, self._place[v]) for i, v in enumerate(ins) if v in self._place]
            if len(set(ins)) != len(ins):
                continue
            if not placed:
                if not all(placeable(v) for v in ins):
                    continue
                key, base_off = c.output, 0
                self._bands[key] = [0, c.output, []]
            else:
                key = placed[0][1][0]
                base_off = placed[0][1][1] - offs[placed[0][0]]
                ok = base_off >= 0 and all(k_ == key and off == base_off + offs[i] for i, (k_, off) in placed)
                ok = ok and all(placeable(v) and free(key, base_off + offs[i], base_off + offs[i] + widths[i])
                                for i, v in enumerate(ins) if v not in self._place)
                if not ok:
                    continue
            for i, v in enumerate(ins):
                if v not in self._place:
                    self._place[v] = (key, base_off + offs[i])
                    self._bands[key][2].append((base_off + offs[i], base_off + offs[i] + widths[i]))
            band = self._bands[key]
            band[0] = max(band[0], base_off + offs[-1] + widths[-1])
            cmap = tuple(offs[i] + j for i, w_ in enumerate(widths) for j in range(w_))
            dense = all(w_ % 8 == 0 for w_ in widths[:-1])
            self._concat_views[c.output] = (key, base_off, None if dense else cmap, ins)

    def _value_width(self, v: str) -> int:
        return self.graph.layer(v).out_channels

    def _band_buffer(self, key: str) -> torch.Tensor:
        if key not in self._band_bufs:
            width, shape_of, _ = self._bands[key]
            _, h, w = self._shapes[shape_of]
            self._band_bufs[key] = torch.zeros((self.batch * h * w, K.pad8(width)), dtype=torch.bfloat16,
                                               device=self.device)
        return self._band_bufs[key]

    def _plan_dual_stores(self) -> None:
        """Producer side of GATHER reads: a conv whose output is gathered by later 1x1 convs
        also stores the gathered channels compacted (ascending source order, the union when
        several consumers gather different sets) in its epilogue (ub_conv_desc.y2); the
        consumers are offered a dense "dual" read plan over that copy.  Off by default
        (dual_store=False): the kept sets of the ResNet-50 export are fragmented (~0.8 runs
        per channel), so the per-element compaction in the producer's epilogue costs more
        (+60..160 us per producer) than the consumers save (-10..25 us each); DESIGN.md 5."""
        self._dual: dict[str, list[int]] = {}
        self._dual_bufs: dict[str, tuple] = {}
        if self.gather_mode != "fused" or not self.dual_store:
            return
        need: dict[str, set] = {}
        for op in self.ops:
            if op.kind != "conv" or "stem_idx" in op.info or op.info["read"] is None:
                continue
            rl = self.graph.layer(op.info["read"])
            spec = self.specs[op.info["conv"]]
            kk = spec.kernel if spec.op == "conv" else 1
            if rl.kind is LayerKind.GATHER and kk == 1:
                need.setdefault(op.info["src"], set()).update(c for c in rl.params if c >= 0)
        producers = {op.info["out"] for op in self.ops if op.kind == "conv" and "stem_idx" not in op.info}
        for vid, chans in need.items():
            if vid in producers and vid not in self._alias:
                self._dual[vid] = sorted(chans)

    def _value(self, vid: str) -> K.Act:
        if vid in self.values:
            return self.values[vid]
        if vid in getattr(self, "_concat_views", {}):
            key, off, cmap, ins = self._concat_views[vid]
            _, h, w = self._shapes[vid]
            a = K.Act(self._band_buffer(key), self.batch, h, w, self.graph.layer(vid).out_channels, off, cmap)
            self.values[vid] = a
            return a
        if vid in self._alias:
            b, s, n = self._alias[vid]
            a = self._value(b)
            if n < 0:
                return a
            return a.view(s, n)
        raise KeyError(f"value {vid} not computed")

    # ------------------------------------------------------------------ binders
    def _bind_stage(self, op, ws, vs, output_feed):
        idx = op.info["idx"]
        C = len(idx) if idx is not None else self.input_chw[0]
        y = self._alloc(op.output, C)
        idx_dev = self._i32(idx) if idx is not None else None
        # the model input is read through self.input_buf at launch time (capture() records
        # one graph per input buffer for the pipelined Runner)
        op.launch = lambda: K.stage_input(self.input_buf, y, idx_dev)

    @staticmethod
    def _dense(a: K.Act) -> K.Act:
        """The physical columns a (possibly column-mapped) value spans, as a dense view."""
        return a if a.cmap is None else K.Act(a.buf, a.N, a.H, a.W, a.width, a.coff)

    def _alloc_like(self, vid: str, a: K.Act) -> K.Act:
        """Output of a layout-preserving op (pool / per-channel / activation): the same
        column map as its input, so a padded concat needs no compaction pass."""
        if a.cmap is None:
            return self._alloc(vid, a.C)
        if vid in getattr(self, "_place", {}):
            raise NotImplementedError(f"{vid}: a column-mapped value cannot be stored into a concat band")
        return self._alloc(vid, a.C, cmap=a.cmap)

    def _bind_maxpool(self, op, ws, vs, output_feed):
        sp = op.info["spec"]
        x = self._value(op.inputs[0])
        y = self._alloc_like(op.output, x)
        xd, yd = self._dense(x), self._dense(y)
        op.launch = lambda: K.maxpool(xd, sp.kernel, sp.stride, sp.pad, yd)

    def _bind_avgpool2d(self, op, ws, vs, output_feed):
        sp = op.info["spec"]
        x = self._value(op.inputs[0])
        y = self._alloc_like(op.output, x)
        xd, yd = self._dense(x), self._dense(y)
        op.launch = lambda: K.avgpool2d(xd, sp.kernel, sp.stride, sp.pad, yd)

    def _bind_avgpool(self, op, ws, vs, output_feed):
        x = self._value(op.inputs[0])
        idx = op.info.get("idx")
        xd = self._dense(x)
        if idx is not None:  # fused GATHER read of the consumer: compacted kept channels
            y = self._alloc(op.output, len(idx))
            idx_dev = self._i32([x.phys(i) for i in idx])
            op.launch = lambda: K.avgpool_gather(xd, idx_dev, y)
            return
        y = self._alloc_like(op.output, x)
        yd = self._dense(y)
        groups = (xd.C + 7) // 8
        if (self.batch * ((groups + 127) // 128) < _lib.num_sms_hint() and xd.coff % 8 == 0
                and xd.cstride % 8 == 0 and x.H * x.W >= 16):
            op.launch = lambda: K.avgpool_split(xd, yd)  # few images: split the pixels over threads
            op.info["split"] = True
        else:
            op.launch = lambda: K.avgpool_global(xd, yd)

    def _bind_gather(self, op, ws, vs, output_feed):
        x = self._value(op.inputs[0])
        idx = op.info["idx"]
        y = self._alloc(op.output, len(idx))
        idx_p = [x.phys(i) for i in idx]
        idx_dev = self._i32(idx_p)
        win = K.gather_window(idx_p)
        xd = self._dense(x)
        op.launch = lambda: K.gather_rows(xd, idx_dev, win, 1, y)
        n_img_pix = x.H * x.W
        self.conv_stats.append(ConvStats(f"{op.output}(copy)", 0.0, 0.0, 2 * 2 * len(idx) * n_img_pix))

    def _bind_concat(self, op, ws, vs, output_feed):
        """A concat _plan_concats could not make zero-copy: each operand is copied into its
        16-byte aligned band of a fresh buffer (the copy the reference's CONCAT implies)."""
        ins = [self._value(v) for v in op.inputs]
        widths = [a.C for a in ins]
        offs, o = [], 0
        for w_ in widths:
            offs.append(o)
            o += K.pad8(w_)
        dense = all(w_ % 8 == 0 for w_ in widths[:-1])
        cmap = None if dense else tuple(offs[i] + j for i, w_ in enumerate(widths) for j in range(w_))
        y = self._alloc(op.output, sum(widths), cmap=cmap)
        copies = []
        for a, off in zip(ins, offs):
            idx_p = [a.phys(i) for i in range(a.C)]
            copies.append((self._dense(a), self._i32(idx_p), K.gather_window(idx_p),
                           K.Act(y.buf, y.N, y.H, y.W, a.C, y.coff + off)))

        def launch():
            for xa, idx_dev, win, dst in copies:
                K.gather_rows(xa, idx_dev, win, 1, dst)

        op.launch = launch

    def _bind_dwconv(self, op, ws, vs, output_feed):
        """Depthwise conv (PER_CHANNEL-like node; its filters follow the planner's per-channel
        permutation like any vector) with the following BN folded: W' = s*W, b' = s*b + t."""
        lid = op.anchor
        sp = self.specs[lid]
        x = self._value(op.inputs[0])
        assert x.cmap is None, f"{lid}: depthwise conv over a column-mapped value"
        vec, perm = vs(lid)
        C = self.graph.layer(lid).out_channels

        def p(v):
            v = v.detach().float().cpu()
            return v[list(perm)] if perm is not None else v

        wdw = p(vec["dw"])  # [C, k*k]
        b = p(vec["bias"]) if "bias" in vec else torch.zeros(C)
        if op.info["bn"] is not None:
            bvec, bperm = vs(op.info["bn"])
            sc, sh = self._affine(op.info["bn"], bvec, bperm)
            sc, sh = sc.cpu(), sh.cpu()
            wdw = wdw * sc.view(-1, 1)
            b = b * sc + sh
        k = sp.kernel
        wt = torch.zeros(k * k, K.pad8(C))
        wt[:, :C] = wdw.t()
        wt, b = wt.to(self.device).contiguous(), b.to(self.device).contiguous()
        self._keep += [wt, b]
        act = self.specs[op.info["act"]].op if op.info["act"] else "none"
        y = self._alloc(op.output, C)
        part = None
        if op.info.get("se_part"):
            nparts = K.dwconv_pool_parts(k, sp.stride, y.H, y.W)
            if nparts > 0:
                part = torch.empty(y.N * nparts, K.pad8(C), dtype=torch.float32, device=self.device)
                op.info["part"] = (part, nparts)
        op.launch = lambda: K.dwconv(x, wt, b, k, sp.stride, sp.pad, act, y, part)
        # roofline bookkeeping: 2*k*k flops per output, input + output bytes
        self.conv_stats.append(ConvStats(lid, 2.0 * k * k * C * y.H * y.W, 2.0 * C * (x.H * x.W + y.H * y.W), 0.0))

    def _bind_eltwise(self, op, ws, vs, output_feed):
        """PER_CHANNEL / ADD / activation nodes no conv absorbed (plus a fused trailing
        activation): ub_eltwise over the physical columns of the operands."""
        kind = op.info["kind"]
        lid = op.anchor
        a = self._value(op.inputs[0])
        scale = shift = None
        others: list[K.Act] = []
        act = op.info.get("act", "none")
        gate = None
        if kind is LayerKind.PER_CHANNEL:
            vec, perm = vs(lid)
            scale, shift = self._affine(lid, vec, perm)
        elif kind is LayerKind.ADD:
            others = [self._value(v) for v in op.inputs[1:]]
            if self.specs[lid].op == "mul":  # squeeze-excitation gate (per image x channel)
                assert len(others) == 1
                gate, others = others[0], []
                if a.H * a.W == 1 and gate.H * gate.W > 1:
                    a, gate = gate, a
        else:
            act = self.specs[lid].op if self.specs[lid].op in ACTS else "relu"
        y = self._alloc_like(op.output, a)
        if a.cmap is not None:  # column-mapped operand: expand the vectors over the pad columns
            assert all(b.cmap == a.cmap for b in others), f"{lid}: operands with different layouts"
            if scale is not None:
                full_s = torch.zeros(a.width, device=self.device)
                full_t = torch.zeros(a.width, device=self.device)
                idx = torch.tensor(a.cmap, device=self.device)
                full_s[idx], full_t[idx] = scale, shift
                scale, shift = full_s, full_t
                self._keep += [scale, shift]
        ad, yd = self._dense(a), self._dense(y)
        od = [self._dense(b) for b in others]
        gd = self._dense(gate) if gate is not None else None

        def launch():
            if not od:
                K.eltwise(ad, yd, scale, shift, None, act, gd)
                return
            K.eltwise(ad, yd, scale, shift, od[0], act if len(od) == 1 else "none", gd)
            for k_, b in enumerate(od[1:]):
                K.eltwise(yd, yd, None, None, b, act if k_ == len(od) - 2 else "none")

        op.launch = launch

    def _affine(self, uid, vec, perm):
        spec = self.specs[uid]

        def p(v):
            v = v.detach().float().cpu()
            return v[list(perm)] if perm is not None else v

        if spec.op == "bn":
            scale = p(vec["weight"]) / torch.sqrt(p(vec["var"]) + spec.eps)
            shift = p(vec["bias"]) - p(vec["mean"]) * scale
        else:
            scale = torch.ones_like(p(vec["bias"]))
            shift = p(vec["bias"])
        s, t = scale.to(self.device), shift.to(self.device)
        self._keep += [s, t]
        return s, t

    def _bind_conv(self, op, ws, vs, output_feed):
        info = op.info
        lid = info["conv"]
        spec = self.specs[lid]
        lay = self.graph.layer(lid)
        if "stem_idx" in info:
            return self._bind_stem(op, ws, vs, output_feed)
        x = self._value(info["src"])
        read = info["read"]
        gather = None  # reference GATHER params (channel indices into x)
        if read is not None:
            rl = self.graph.layer(read)
            if rl.kind is LayerKind.SLICE:
                s0, n = rl.params
                x = x.view(s0, n)
            else:
                gather = list(rl.params)
        cin = len(gather) if gather is not None else x.C
        assert cin == lay.in_channels, f"{lid}: reads {cin} channels, layer has {lay.in_channels}"
        cout = lay.out_channels
        kk = spec.kernel if spec.op == "conv" else 1
        st = spec.stride if spec.op == "conv" else 1
        pd = spec.pad if spec.op == "conv" else 0
        W, rows, cols = ws(lid)
        scale = bias = None
        if info["bn"] is not None:
            vec, perm = vs(info["bn"])
            scale, bias = self._affine(info["bn"], vec, perm)
            if self.specs[info["bn"]].op != "bn":
                scale = None
        O, I = W.shape[0], W.shape[1]
        rows = list(rows if rows is not None else range(O))
        cols = list(cols if cols is not None else range(I))

        # Read plans for this layer's input (autotune() times them):
        #   ("slice", ...)  contiguous window -- zero-copy view (UPSCALE's contiguous read)
        #   ("gather", ...) fused gather: producer warps gather the channels; internal K order is
        #                   the gathered channels sorted by source position (a GEMM is invariant to
        #                   a consistent K permutation), the exported (perm, indices) stay the
        #                   reference's
        #   ("cover", ...)  the gather's covering window read as a slice, with zero weight columns
        #                   for the channels the gather drops (same result; cp.async operand path)
        #   ("copy", ...)   1x1 gathers: one kernel gathers the channels (and the strided pixels)
        #                   into a compact buffer, then a dense 1x1 / stride-1 GEMM over it -- half
        #                   the MMA work of "cover" when half the channels are kept
        plans = []

        def add_plan(kind, xv, gidx, wcols, width, pre=None, st_eff=None):
            lead, cpad = _lib.conv_weight_layout(width, xv.coff, gidx is not None, kk, kk)
            wg = K.permute_weights(W, rows, wcols, row_scale=scale, layout="gemm", lead=lead, cpad=cpad,
                                   out_dtype=torch.bfloat16)
            self._keep.append(wg)
            plans.append((kind, xv, gidx, lead, cpad, wg, pre, st if st_eff is None else st_eff))

        residual_id = info.get("residual")
        if (kk == 1 and st == 1 and pd == 0 and self.batch * x.H * x.W <= 16 and residual_id is None
                and info.get("prologue") is None and info.get("pool2") is None and info["out"] not in self._dual):
            return self._bind_small_linear(op, x, gather, W, rows, cols, scale, bias, cin, cout, output_feed)
        staged = info.get("prologue") is not None or info.get("pool2") is not None or x.cmap is not None
        if staged:
            # the read is staged by ub_gather_rows_ex into a compact buffer -- the gather (through
            # the concat's column map), the reader's BN/ReLU prologue and a moved 2x2 pool in one
            # pass -- and the conv reads it densely
            idx = gather if gather is not None else list(range(x.C))
            # internal K order = ascending source column (a GEMM is invariant to a consistent
            # permutation of K; the exported (perm, indices) stay the reference's): the staged
            # read's shared-memory gathers then touch distinct banks
            k_order = sorted(range(len(idx)), key=lambda k: (idx[k] < 0, x.phys(idx[k]), k))
            idx = [idx[k] for k in k_order]
            cols = [cols[k] for k in k_order]
            idx_p = [x.phys(i) for i in idx]
            xb = K.Act(x.buf, x.N, x.H, x.W, x.width, x.coff)
            pscale = pshift = None
            prelu = False
            if info.get("prologue") is not None:
                pro_bn, pro_relu = info["prologue"]
                prelu = pro_relu is not None
                if pro_bn is not None:
                    vec, perm = vs(pro_bn)
                    sc, sh = self._affine(pro_bn, vec, perm)
                    sc, sh = sc.cpu(), sh.cpu()
                    pscale = self._f32([float(sc[i]) if i >= 0 else 0.0 for i in idx])
                    pshift = self._f32([float(sh[i]) if i >= 0 else 0.0 for i in idx])
                else:
                    pscale = self._f32([1.0] * len(idx))
                    pshift = self._f32([0.0] * len(idx))
            pool2 = info.get("pool2") is not None
            st_g = st if (kk == 1 and pd == 0 and not pool2) else 1
            if pool2:
                ho, wo = x.H // 2, x.W // 2
            else:
                ho, wo = (x.H - 1) // st_g + 1, (x.W - 1) // st_g + 1
            scratch = K.empty_act(self.batch, ho, wo, cin, self.device)
            self._keep.append(scratch.buf)
            gdev = self._i32(idx_p)
            win = K.gather_window(idx_p)

            def pre(xb=xb, gdev=gdev, scratch=scratch, win=win, st_g=st_g, pool2=pool2, pscale=pscale,
                    pshift=pshift, prelu=prelu):
                K.gather_rows_ex(xb, gdev, win, st_g, scratch, pool2=pool2, scale=pscale, shift=pshift, relu=prelu)

            add_plan("copy", scratch, None, cols, cin, pre=pre, st_eff=st if st_g == 1 else 1)
        elif gather is None:
            add_plan("slice", x, None, cols, cin)
        else:
            k_order = sorted(range(cin), key=lambda k: (gather[k], k))
            add_plan("gather", x, self._i32([gather[k] for k in k_order]), [cols[k] for k in k_order], cin)
            if self.gather_mode == "fused":
                # copy plan: compact the gathered channels (1x1 / pad 0: only the pixels a strided
                # conv reads), then a dense conv -- for k x k convs the dense operand also makes
                # the halo kernel eligible (it takes no fused gather)
                st_g = st if (kk == 1 and pd == 0) else 1
                ho, wo = (x.H - 1) // st_g + 1, (x.W - 1) // st_g + 1
                k_order = sorted(range(cin), key=lambda k: (gather[k] < 0, gather[k], k))
                g_sorted = [gather[k] for k in k_order]
                scratch = K.empty_act(self.batch, ho, wo, cin, self.device)
                self._keep.append(scratch.buf)
                gdev = self._i32(g_sorted)
                win = K.gather_window(g_sorted)

                def pre(x=x, gdev=gdev, scratch=scratch, win=win, st_g=st_g):
                    K.gather_rows(x, gdev, win, st_g, scratch)

                add_plan("copy", scratch, None, [cols[k] for k in k_order], cin, pre=pre,
                         st_eff=1 if st_g != 1 else st)
            lo, hi = min(gather), max(gather)
            width = hi - lo + 1
            if (self.gather_mode == "fused" and lo >= 0 and len(set(gather)) == cin
                    and width <= self.cover_ratio * cin):
                pos = {c: k for k, c in enumerate(gather)}
                wcols = [cols[pos[lo + j]] if (lo + j) in pos else -1 for j in range(width)]
                add_plan("cover", x.view(lo, width), None, wcols, width)
            if kk == 1 and info["src"] in self._dual_bufs:  # the producer's compacted copy
                comp, col_of = self._dual_bufs[info["src"]]
                pos = {c: k for k, c in enumerate(gather)}
                wcols = [-1] * comp.C
                for c, j in col_of.items():
                    if c in pos:
                        wcols[j] = cols[pos[c]]
                add_plan("dual", comp, None, wcols, comp.C)
        residual = self._value(info["residual"]) if info.get("residual") else None
        fp32_out = info["out"] in output_feed
        y = self._alloc(info["out"], cout, fp32=fp32_out)
        y2 = y2_map = None
        if info["out"] in self._dual and not fp32_out:  # producer side of a later GATHER
            # ub_conv_desc.y2 layout: each 64-channel group's kept channels consecutive from
            # an 8-aligned column (zero columns pad the group to a multiple of 8)
            col_of, width = {}, 0
            for grp in range(0, cout, 64):
                kept = [c for c in self._dual[info["out"]] if grp <= c < grp + 64]
                for k, c in enumerate(kept):
                    col_of[c] = width + k
                width += K.pad8(len(kept))
            y2 = self._alloc(info["out"] + "#compact", width, shape_of=info["out"])
            m = [-1] * cout
            for c, j in col_of.items():
                m[c] = j
            y2_map = self._i32(m)
            self._dual_bufs[info["out"]] = (y2, col_of)
        relu = self._act_code(info["relu"])
        # variant = (plan index, ub_conv_desc.variant bits: producer width 1 = 256 / 2 = 512
        # threads; +4 re-load the weights per tile instead of keeping them resident; +16 weights
        # by cp.async instead of TMA; +32 1x1 activations by cp.async instead of TMA;
        # +64 one epilogue warpgroup instead of two on the TMA-fed 1x1 path; +65536 32-channel
        # N tiles for an fp32 output without residual (the classifier);
        # +8 no halo-tile kernel for a 3x3 (stride 1 or 2); +128 halo kernel with two epilogue groups)
        halo = kk == 3 and st in (1, 2) and pd == 1

        def gen_for(st_p):
            tiled = kk == 1 and st_p == 1
            gen = [pw | nb | bt | at | e1 for pw in (1, 2) for nb in (0, 4) for bt in (0, 16)
                   for at in ((0, 32) if tiled else (32,)) for e1 in ((0, 64) if tiled else (0,))]
            if kk == 1 and cout > 192:  # +8192: N tiles of <= 128 channels (weights may stay resident)
                gen = gen + [v | 8192 for v in gen if not v & 4]
            # (+32768 pair mode -- two M tiles per streamed weight box -- is not offered: it
            # measured slower on every wide-K 1x1 of ResNet-50)
            if fp32_out and residual is None:  # +65536: 32-channel N tiles (fp32 classifier)
                gen = gen + [v | 65536 for v in gen if not v & 8192]
            if halo:  # the halo kernel ignores the generic bits; offer it twice, then the generic kernel
                gen = [0, 128] + [v | 8 for v in gen]
            return gen

        op.info["halo"] = halo
        op.info["read_pre"] = [pl[6] for pl in plans]  # staged-read launches (tools time them apart)
        op.info["variants"] = [(pi, v) for pi, pl in enumerate(plans) for v in gen_for(pl[7])]
        op.info["variant"] = (len(plans) - 1, 0)  # cover when offered, else the only plan
        op.info["plans"] = [pl[0] for pl in plans]

        def launch():
            pi, pw = op.info["variant"]
            _, xv, gidx, lead, cpad, wg, pre, st_p = plans[pi]
            if pre is not None:
                pre()
            K.conv(xv, wg, lead, cpad, cout, kk, kk, st_p, pd, y, gather_idx=gidx, bias=bias, residual=residual,
                   relu=relu, y_fp32=fp32_out, variant=pw, y2=y2, y2_map=y2_map)

        op.launch = launch
        op.info["desc"] = (f"{kk}x{kk}s{st} {cin}->{cout} {x.H}x{x.W}"
                           f"{' gather' if gather is not None else ''}{' +res' if residual is not None else ''}"
                           f" [coff {plans[-1][1].coff} cs {plans[-1][1].cstride} lead {plans[-1][3]}"
                           f" cpad {plans[-1][4]}]")
        # roofline bookkeeping (per image)
        _, hi, wi = self._shapes[info["src"]] if info["src"] in self._shapes else (0, x.H, x.W)
        ho, wo = y.H, y.W
        flops = 2.0 * cout * cin * kk * kk * ho * wo
        byts = 2.0 * (cin * x.H * x.W + cout * ho * wo) + (2.0 * cout * cin * kk * kk) / self.batch
        if residual is not None:
            byts += 2.0 * cout * ho * wo
        self.conv_stats.append(ConvStats(lid, flops, byts, 0.0))

    def _bind_small_linear(self, op, x, gather, W, rows, cols, scale, bias, cin, cout, output_feed):
        """CHANNEL_MIX over at most 16 rows (images x pixels): ub_linear_small on CUDA cores,
        the read (SLICE / GATHER / column map) folded into its column offsets."""
        info = op.info
        idx = gather if gather is not None else list(range(x.C))
        xcol = self._i32([x.coff + x.phys(i) if i >= 0 else -1 for i in idx])
        wd = K.permute_weights(W, rows, cols, row_scale=scale, layout="dense", cpad=K.pad8(cin),
                               out_dtype=torch.bfloat16)
        self._keep.append(wd)
        fp32_out = info["out"] in output_feed
        y = self._alloc(info["out"], cout, fp32=fp32_out)
        act = self._act_code(info["relu"])
        xb = K.Act(x.buf, x.N, x.H, x.W, x.width, 0)
        op.launch = lambda: K.linear_small(xb, xcol, wd, cout, y, bias=bias, act=act, y_fp32=fp32_out)
        op.info.update(variants=[], variant=(0, 0), plans=["small"], halo=False,
                       desc=f"linear_small {cin}->{cout} M={self.batch * x.H * x.W}")
        self.conv_stats.append(ConvStats(info["conv"], 2.0 * cout * cin * x.H * x.W,
                                         2.0 * (cin * x.H * x.W + cout * x.H * x.W) + 2.0 * cout * cin / self.batch,
                                         0.0))

    def _s2d_ok(self, cin: int, spec, cout: int) -> bool:
        """Stem shapes the space-to-depth kernel takes (the folded 2x2 pixel fits 16 bytes)."""
        kk = spec.kernel
        return self.stem_s2d and spec.stride == 2 and kk >= 2 and (kk + 1) // 2 <= 4 and 4 * cin <= 8 and cout <= 128

    def _bind_stem(self, op, ws, vs, output_feed):
        info = op.info
        lid = info["conv"]
        spec = self.specs[lid]
        lay = self.graph.layer(lid)
        idx = info["stem_idx"]
        idx_dev = self._i32(idx)
        cin = len(idx)
        assert cin == lay.in_channels
        W, rows, cols = ws(lid)
        scale = bias = None
        if info["bn"] is not None:
            vec, perm = vs(info["bn"])
            scale, bias = self._affine(info["bn"], vec, perm)
            if self.specs[info["bn"]].op != "bn":
                scale = None
        O, I = W.shape[0], W.shape[1]
        rows = rows if rows is not None else range(O)
        cols = cols if cols is not None else range(I)
        assert info.get("residual") is None and info["out"] not in output_feed
        y = self._alloc(info["out"], lay.out_channels)
        relu = self._act_code(info["relu"])
        cout, kk, st, pd = lay.out_channels, spec.kernel, spec.stride, spec.pad
        ci, hi, wi = self.input_chw
        # space-to-depth stem when the folded 2x2 pixel fits 16 bytes (ub_conv_s2d); else the
        # single-launch im2col stem.  info["pool"]: the following max pool is fused.  The s2d
        # kernels' epilogues know ReLU only; other activations (MobileNetV3's hardswish stem)
        # take the im2col stem on the generic conv kernel.
        s2d = (self._s2d_ok(cin, spec, cout) and y.cstride % 8 == 0 and y.coff % 8 == 0
               and relu in (0, _lib.UB_ACT["relu"]))
        if "pool" in info:
            assert s2d, "stem/max-pool fusion needs the space-to-depth stem"
            wg = K.permute_weights(W, rows, cols, row_scale=scale, layout="s2d", out_dtype=torch.bfloat16)
            self._keep.append(wg)
            if self.stem_pack_fused:  # one launch: the kernel folds the fp32 input itself
                op.launch = lambda: K.stem_maxpool(self.input_buf, idx_dev, wg, cout, kk, pd, y, bias=bias, relu=relu)
                op.info["stem_kind"] = "s2d+maxpool+pack"
            else:
                sbuf = K.s2d_buffer(self.batch, hi, wi, kk, pd, self.device)
                self._keep.append(sbuf)
                op.launch = lambda: K.stem_s2d_maxpool(self.input_buf, idx_dev, sbuf, wg, cout, kk, pd, y, bias=bias,
                                                       relu=relu)
                op.info["stem_kind"] = "s2d+maxpool"
            wbytes = 2.0 * wg.numel()
        elif s2d:
            wg = K.permute_weights(W, rows, cols, row_scale=scale, layout="s2d", out_dtype=torch.bfloat16)
            sbuf = K.s2d_buffer(self.batch, hi, wi, kk, pd, self.device)
            self._keep += [wg, sbuf]
            op.launch = lambda: K.stem_s2d(self.input_buf, idx_dev, sbuf, wg, cout, kk, pd, y, bias=bias, relu=relu)
            op.info["stem_kind"] = "s2d"
            wbytes = 2.0 * wg.numel()
        elif cin <= 8 and kk <= 3 and cout <= 256 and y.coff % 8 == 0 and y.cstride % 8 == 0:
            # few input channels and a small filter (MobileNetV3 / EfficientNetV2 3x3/s2 stems):
            # direct conv on CUDA cores, the input read once (the im2col operand would be k*k times
            # the input); a 7x7 stem on 3 planes (ResNet at low sparsity) stays on the tensor cores
            Wf = W.detach().float().cpu()
            rr = torch.tensor([r_ for r_ in rows], dtype=torch.long)
            cc = torch.tensor([c_ for c_ in cols], dtype=torch.long)
            Wsel = Wf[rr.clamp_min(0)][:, cc.clamp_min(0)] * (rr >= 0).view(-1, 1, 1, 1) * (cc >= 0).view(1, -1, 1, 1)
            if scale is not None:
                Wsel = Wsel * scale.detach().float().cpu().view(-1, 1, 1, 1)
            wd = torch.zeros(kk * kk, cin, _lib.load().ub_conv_direct_wcols(cout))
            wd[:, :, :cout] = Wsel.permute(2, 3, 1, 0).reshape(kk * kk, cin, cout)
            wd = wd.to(self.device).contiguous()
            self._keep.append(wd)
            op.launch = lambda: K.conv_direct(self.input_buf, idx_dev, wd, bias, cout, kk, st, pd, relu, y)
            op.info["stem_kind"] = "direct"
            wbytes = 4.0 * wd.numel()
        else:
            kpad = _lib.conv_stem_kpad(cin, kk, kk)
            wg = K.permute_weights(W, rows, cols, row_scale=scale, layout="dense", cpad=kpad,
                                   out_dtype=torch.bfloat16)
            self._keep.append(wg)
            op.launch = lambda: K.conv_stem(self.input_buf, idx_dev, wg, kpad, cout, kk, st, pd, y, bias=bias, relu=relu)
            op.info["stem_kind"] = "im2col"
            wbytes = 2.0 * cout * kpad
        pooled = "pool" in info
        ho, wo = (2 * y.H, 2 * y.W) if pooled else (y.H, y.W)  # conv output (the pool halves it)
        flops = 2.0 * cout * cin * kk * kk * ho * wo
        byts = 4.0 * cin * hi * wi + 2.0 * cout * y.H * y.W + wbytes / self.batch
        self.conv_stats.append(ConvStats(lid, flops, byts, 0.0))

    # ------------------------------------------------------------------ execution
    def launch_all(self, nvtx: bool = False) -> None:
        """Enqueue the forward.  nvtx=True wraps every op in an NVTX range named after its
        exported node (for nsys / ncu --nvtx filtering; eager runs only)."""
        if not nvtx:
            for op in self.ops:
                op.launch()
            return
        for op in self.ops:
            torch.cuda.nvtx.range_push(f"{op.kind}:{op.anchor}")
            op.launch()
            torch.cuda.nvtx.range_pop()

    def forward(self, x: torch.Tensor) -> torch.Tensor:
        """x: [N, C, H, W] fp32 (device or host).  Returns logits (device)."""
        self.input_buf.copy_(x, non_blocking=True)
        if self._graph_exec is not None:
            self._graph_exec.replay()
        else:
            self.launch_all()
        return self.output_tensor()

    def kept_input_channels(self) -> list[int]:
        """Input channels any op reads (the INPUT node's GATHER; all when none)."""
        kept = set()
        for op in self.ops:
            if "stem_idx" in op.info:
                kept.update(op.info["stem_idx"])
            elif op.kind == "stage":
                idx = op.info["idx"]
                kept.update(idx if idx is not None else range(self.input_chw[0]))
        return sorted(kept) if kept else list(range(self.input_chw[0]))

    def replay(self, slot: int = 0) -> None:
        """Run the captured forward that reads input buffer `slot`."""
        self._graphs[slot].replay()

    def output_tensor(self) -> torch.Tensor:
        o = self.output_value
        t = o.buf[:, o.coff:o.coff + o.C]
        if o.H * o.W != 1:
            t = t.reshape(o.N, o.H, o.W, o.C).permute(0, 3, 1, 2)
        return t.float()

    def autotune(self, reps: int = 5) -> dict[str, tuple]:
        """Pick, per conv layer, the read plan (fused gather vs covering slice) and the
        producer width (256 vs 512 cp.async threads) by timing every combination on this
        engine's own buffers (CUDA events, after a warm-up)."""
        picks = {}
        for op in self.ops:
            if op.kind != "conv" or "stem_idx" in op.info or not op.info.get("variants"):
                continue
            best = None
            for v in op.info["variants"]:
                op.info["variant"] = v
                op.launch()
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record()
                for _ in range(reps):
                    op.launch()
                b.record()
                b.synchronize()
                t = a.elapsed_time(b)
                if best is None or t < best[0]:
                    best = (t, v)
            op.info["variant"] = best[1]
            picks[op.info["conv"]] = best[1]
        return picks

    def capture(self, autotune: bool = True, n_inputs: int = 1) -> None:
        """Capture the launch sequence in a CUDA graph (static buffers); optionally
        autotune the conv variants first.  n_inputs > 1 allocates that many input
        buffers and captures one graph per buffer (double-buffered input for the
        pipelined Runner.run_many)."""
        if autotune and self.batch >= 16:  # at small batches eager timings are launch-bound noise
            self.launch_all()
            self.autotune()
        s = torch.cuda.Stream(device=self.device)
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            _lib.reset_launch_count()
            self.launch_all()  # warm-up (first-launch attribute setup)
            self._launches = _lib.launch_count()
        torch.cuda.current_stream().wait_stream(s)
        torch.cuda.synchronize()
        while len(self.input_bufs) < n_inputs:
            self.input_bufs.append(torch.zeros_like(self.input_bufs[0]))
        self._graphs = []
        for k in range(max(n_inputs, 1)):
            self.input_buf = self.input_bufs[k]
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                self.launch_all()
            self._graphs.append(g)
        self.input_buf = self.input_bufs[0]
        self._graph_exec = self._graphs[0]

    @property
    def n_launches(self) -> int:
        """Library kernel launches per forward, counted by the C ABI (ub_launch_count) over
        one eager pass; before any pass, the op count (one launch per op, two for the
        space-to-depth stem)."""
        if getattr(self, "_launches", None) is None:
            return sum(2 if op.info.get("stem_kind", "") in ("s2d", "s2d+maxpool") else 1 for op in self.ops)
        return self._launches

    def kernel_label(self, op) -> str:
        """Which library kernel(s) one op launches with its current variant."""
        if op.kind == "conv":
            if "stem_idx" in op.info:
                return "stem_" + op.info.get("stem_kind", "")
            pi, pw = op.info["variant"]
            if op.info.get("halo") and not pw & 8:
                return "conv_halo3_kernel"
            plan = op.info["plans"][pi]
            if plan == "small":
                return "linear_small_kernel"
            return "conv_tc_kernel+gather_rows" if plan == "copy" else "conv_tc_kernel"
        return {"gather": "gather_rows_kernel", "stage": "stage_input_kernel", "maxpool": "maxpool_kernel",
                "avgpool": "avgpool_gather_kernel" if "idx" in op.info else (
                    "avgpool_split_kernel" if op.info.get("split") else "avgpool_kernel"),
                "eltwise": "eltwise_kernel", "dwconv": "dwconv_kernel", "avgpool2d": "avgpool2d_kernel",
                "concat": "gather_rows_kernel", "se": "se_gate_kernel"}.get(op.kind, op.kind)

    def per_image_work(self) -> tuple[float, float]:
        f = sum(c.flops for c in self.conv_stats)
        b = sum(c.bytes + c.gather_bytes for c in self.conv_stats)
        return f, b


# ---------------------------------------------------------------------- builders
def from_plans(sm, exported_graph: ModelGraph, maps, batch: int, device="cuda", gather_mode="fused",
               masks: Mapping[str, Sequence[int]] | None = None, **engine_opts) -> Engine:
    """One-pass export: original sidecar weights + composed plan maps -> GEMM operands.
    With `masks` and an identity export this runs the mask-simulated original
    (interp.py:59-60: masked input channels == zero weight columns)."""
    dev = torch.device(device)
    cache: dict[str, torch.Tensor] = {}

    def ws(lid):
        if lid not in cache:
            cache[lid] = sm.weights[lid].to(dev).contiguous()
        cols = maps.cols.get(lid) if maps is not None else None
        if masks is not None and lid in masks:
            keep = set(masks[lid])
            base = cols if cols is not None else range(sm.weights[lid].shape[1])
            cols = tuple(c if c in keep else -1 for c in base)
        return cache[lid], (maps.rows.get(lid) if maps is not None else None), cols

    def vs(uid):
        return sm.vectors[uid], (maps.vec.get(uid) if maps is not None else None)

    return Engine(exported_graph, sm.specs, ws, vs, batch, sm.input_chw, device, gather_mode, **engine_opts)


def from_export(sm, result, batch: int, device="cuda", gather_mode="fused") -> Engine:
    """Engine over an ExportResult (weights already permuted on device)."""

    def ws(lid):
        return result.weights.mix[lid].float().contiguous(), None, None

    def vs(uid):
        return result.weights.vec[uid], None

    return Engine(result.graph, sm.specs, ws, vs, batch, sm.input_chw, device, gather_mode)
