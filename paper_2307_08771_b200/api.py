"""Reference-facing API: the drop-in for `reslice`'s export + inference path.

    from paper_2307_08771_b200 import api
    model = api.load_config("resnet50_s50")          # lowered torchvision model + masks
    plans, fallbacks = api.plan_model(model.graph, model.masks, strategy="reorder")
    res = api.export_model(model, model.masks, plans=plans)   # GPU permute kernel
    logits = api.run(res, x)                          # B200 engine, numpy in/out

Names and argument meaning follow pipeline.py:99-146 and interp.py:36-84; the
extra argument everywhere is the spatial sidecar (`SpatialModel`), because the
reference IR collapses the spatial dimensions a real CNN needs.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Mapping, Sequence

import numpy as np
import torch

from . import engine as EN
from . import export as E
from . import ir
from . import plans as P
from .configs import CONFIGS, Config, build_spatial_model
from .lowering import SpatialModel

plan_model = E.plan_model


@dataclass
class LoadedConfig:
    cfg: Config
    model: SpatialModel
    masks: ir.ChannelMask

    @property
    def graph(self) -> ir.ModelGraph:
        return self.model.graph

    def plans(self, strategy: str = "reorder") -> list[P.SegmentPlan]:
        """The reference planner's committed output for this config."""
        return P.load_plans(self.cfg.asset_dir / f"plans_{strategy}.json")


def load_config(name: str, randomize_bn: bool = False) -> LoadedConfig:
    cfg = CONFIGS[name]
    sm = build_spatial_model(cfg, randomize_bn=randomize_bn)
    return LoadedConfig(cfg, sm, ir.load_masks(cfg.asset_dir / "masks.json"))


@dataclass
class Exported:
    """ExportResult plus what the engine needs to run it."""

    result: E.ExportResult
    model: SpatialModel
    maps: E.LayerMaps

    @property
    def graph(self) -> ir.ModelGraph:
        return self.result.graph


def export_model(model: SpatialModel, masks: ir.ChannelMask, mode: str = "input", strategy: str = "reorder",
                 on_unsupported: str = "error", plans: Sequence[P.SegmentPlan] | None = None,
                 device="cuda") -> Exported:
    """pipeline.py:135-146 over the spatial sidecar; weights permuted on the GPU."""
    res = E.export_model(model.graph, model.weights, model.vectors, masks, mode, strategy, on_unsupported,
                         plans=plans, device=device)
    return Exported(res, model, E.compose_maps(model.graph, list(res.plans)))


class Runner:
    """Compiled engine cache keyed by batch size (one CUDA graph per size)."""

    def __init__(self, exported: Exported, gather_mode: str = "fused", device="cuda"):
        self.exported = exported
        self.gather_mode = gather_mode
        self.device = device
        self._engines: dict[int, EN.Engine] = {}
        self._host_out: dict[int, torch.Tensor] = {}

    def engine(self, batch: int) -> EN.Engine:
        if batch not in self._engines:
            ex = self.exported
            eng = EN.from_plans(ex.model, ex.graph, ex.maps, batch, device=self.device, gather_mode=self.gather_mode)
            eng.capture()
            self._engines[batch] = eng
        return self._engines[batch]

    def run(self, x) -> np.ndarray:
        """x: host array/tensor [N, C, H, W] float32 -> logits [N, classes] (host).
        Pinned host tensors are copied asynchronously; the D2H lands in a
        pinned buffer and the call returns after the stream drains."""
        xt = torch.as_tensor(x, dtype=torch.float32)
        eng = self.engine(xt.shape[0])
        out = eng.forward(xt)  # H2D into the engine's static input buffer
        host = self._host_out.get(eng.batch)
        if host is None or host.shape != out.shape:
            host = torch.empty(out.shape, dtype=torch.float32, pin_memory=True)
            self._host_out[eng.batch] = host
        host.copy_(out, non_blocking=True)
        torch.cuda.current_stream().synchronize()
        return host.numpy().copy()


def run(exported: Exported, x, gather_mode: str = "fused") -> np.ndarray:
    """interp.py:36 analogue: evaluate the exported model on a batch of images."""
    return Runner(exported, gather_mode).run(x)
