"""Plan and weight serialisation off the hot path.

An exported model as a self-contained directory, loadable without the original
weights or the planner:

    graph.json    the exported IR graph (graph.py:389-441 JSON schema, ir.graph_to_dict)
    plans.json    the SegmentPlans that produced it (planner.py:840-927 schema)
    specs.json    the spatial sidecar's per-layer op specs (kernel/stride/pad/eps) + input CHW
    weights.bin   every exported tensor, raw little-endian, 64-byte aligned
    index.json    name -> (kind, key, dtype, shape, byte offset) for weights.bin, totals, fallbacks

The reference's JSON weight format (graph.py:379-386) stores float64 lists and is
unusable at 25 M parameters; here the 4-D CHANNEL_MIX tensors and the per-channel
vectors are one binary blob that `load_export` maps straight into device memory.
Round trip is bit-exact (the bytes of each tensor are copied, not converted).
"""

from __future__ import annotations

import json
from dataclasses import asdict
from pathlib import Path

import numpy as np
import torch

from . import export as E
from . import ir
from . import plans as P
from .lowering import OpSpec, SpatialModel

FORMAT = "upscale-b200-export/1"
_ALIGN = 64
_DTYPES = {torch.float32: "f32", torch.float64: "f64", torch.bfloat16: "bf16", torch.float16: "f16"}
_TORCH = {v: k for k, v in _DTYPES.items()}


def save_export(result: E.ExportResult, model: SpatialModel, path: str | Path) -> Path:
    """Write `result` (exported graph, device weights, plans) plus the spatial op specs."""
    out = Path(path)
    out.mkdir(parents=True, exist_ok=True)
    ir.save_graph(result.graph, out / "graph.json")
    P.save_plans(result.plans, out / "plans.json")
    specs = {lid: asdict(s) for lid, s in model.specs.items() if lid in {l.id for l in result.graph.layers}}
    (out / "specs.json").write_text(json.dumps({"input_chw": list(model.input_chw), "specs": specs}, indent=1))
    entries = []
    for lid, t in result.weights.mix.items():
        entries.append(("mix", lid, "", t))
    for uid, named in result.weights.vec.items():
        for k, t in named.items():
            entries.append(("vec", uid, k, t))
    index, off = [], 0
    with open(out / "weights.bin", "wb") as f:
        for kind, key, sub, t in entries:
            t = t.detach().contiguous().cpu()
            if t.dtype not in _DTYPES:
                raise ir.ModelFormatError([f"{key}{'.' + sub if sub else ''}: unsupported dtype {t.dtype}"])
            raw = t.view(torch.uint8).numpy().tobytes() if t.dtype == torch.bfloat16 else t.numpy().tobytes()
            pad = (-off) % _ALIGN
            f.write(b"\0" * pad)
            off += pad
            f.write(raw)
            index.append({"kind": kind, "key": key, "name": sub, "dtype": _DTYPES[t.dtype],
                          "shape": list(t.shape), "offset": off, "nbytes": len(raw)})
            off += len(raw)
    meta = {"format": FORMAT, "tensors": index,
            "totals": asdict(result.totals),
            "fallbacks": list(result.fallbacks)}
    (out / "index.json").write_text(json.dumps(meta, indent=1))
    return out


def load_export(path: str | Path, device="cuda") -> tuple[E.ExportResult, SpatialModel]:
    """Inverse of save_export: (ExportResult with device weights, SpatialModel carrying the
    exported graph + op specs, for engine.from_export)."""
    src = Path(path)
    meta = json.loads((src / "index.json").read_text())
    if meta.get("format") != FORMAT:
        raise ir.ModelFormatError([f"{src}: not an {FORMAT} artifact"])
    graph = ir.load_graph(src / "graph.json")
    plans = P.load_plans(src / "plans.json")
    sj = json.loads((src / "specs.json").read_text())
    specs = {lid: OpSpec(**d) for lid, d in sj["specs"].items()}
    blob = np.fromfile(src / "weights.bin", dtype=np.uint8)
    ew = E.ExportedWeights()
    for e in meta["tensors"]:
        raw = torch.from_numpy(blob[e["offset"]:e["offset"] + e["nbytes"]].copy())
        dt = _TORCH[e["dtype"]]
        t = raw.view(dt).reshape(e["shape"]).to(device)
        if e["kind"] == "mix":
            ew.mix[e["key"]] = t
        else:
            ew.vec.setdefault(e["key"], {})[e["name"]] = t
    totals = P.CopyStats(**meta["totals"])
    result = E.ExportResult(graph, ew, tuple(plans), totals, tuple(meta["fallbacks"]))
    model = SpatialModel(graph, specs, {}, {}, tuple(sj["input_chw"]))
    return result, model
