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
from . import kernels as K
from . import export as E
from . import ir
from . import plans as P
from .configs import CONFIGS, Config, build_spatial_model
from .lowering import SpatialModel

plan_model = E.plan_model
apply_plan = E.apply_plan


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
    """Compiled engine cache keyed by batch size (CUDA graphs per size).

    The host side of interp.run for batches: the H2D copy carries only the input
    channels the exported model reads (the INPUT node's GATHER, applied to the copy:
    ub_h2d_input_channels), and run_many() pipelines consecutive batches -- the copy
    of batch i+1 runs on its own stream while the forward of batch i replays its
    graph (two input buffers, one graph each)."""

    def __init__(self, exported: Exported, gather_mode: str = "fused", device="cuda"):
        self.exported = exported
        self.gather_mode = gather_mode
        self.device = device
        self._engines: dict[int, EN.Engine] = {}
        self._host_out: dict[tuple, torch.Tensor] = {}
        self._copy_stream = None
        self.h2d_bytes = 0  # bytes moved host -> device by the last run / run_many step

    def engine(self, batch: int) -> EN.Engine:
        if batch not in self._engines:
            ex = self.exported
            eng = EN.from_plans(ex.model, ex.graph, ex.maps, batch, device=self.device, gather_mode=self.gather_mode)
            eng.capture(n_inputs=2)
            self._engines[batch] = eng
        eng = self._engines[batch]
        if len(eng._graphs) < 2:  # an engine captured elsewhere with one input buffer
            eng.capture(autotune=False, n_inputs=2)
        return eng

    def _pinned_out(self, eng, slot):
        key = (eng.batch, slot)
        if key not in self._host_out:
            o = eng.output_tensor()
            self._host_out[key] = torch.empty(o.shape, dtype=torch.float32, pin_memory=True)
        return self._host_out[key]

    def _h2d(self, eng, xt, slot) -> int:
        if xt.is_pinned() and xt.is_contiguous():
            return K.h2d_input_channels(xt, eng.input_bufs[slot], eng.kept_input_channels())
        eng.input_bufs[slot].copy_(xt, non_blocking=True)
        return xt.numel() * 4

    def run(self, x) -> np.ndarray:
        """x: host array/tensor [N, C, H, W] float32 -> logits [N, classes] (host).
        Pinned host tensors are copied asynchronously (kept channels only); the D2H
        lands in a pinned buffer and the call returns after the stream drains."""
        xt = torch.as_tensor(x, dtype=torch.float32)
        eng = self.engine(xt.shape[0])
        self.h2d_bytes = self._h2d(eng, xt, 0)
        eng.replay(0)
        host = self._pinned_out(eng, 0)
        host.copy_(eng.output_tensor(), non_blocking=True)
        torch.cuda.current_stream().synchronize()
        return host.numpy().copy()

    def run_many(self, batches):
        """Pipelined run over an iterable of equally-sized pinned host batches; yields
        the logits of each batch (host numpy) in order.  Batch i+1's H2D overlaps batch
        i's forward; every batch still crosses PCIe and every result comes back.  A host
        batch is no longer read once the next one is pulled from `batches` (its copy has
        landed), so a loader may refill one pinned buffer in place."""
        compute = torch.cuda.current_stream()
        if self._copy_stream is None:
            self._copy_stream = torch.cuda.Stream(device=self.device)
        copy = self._copy_stream
        eng = None
        consumed = [None, None]  # event: the forward that read input buffer k finished
        pending = None           # (event, host buffer) of the previous batch's D2H
        for i, x in enumerate(batches):
            xt = torch.as_tensor(x, dtype=torch.float32)
            if eng is None:
                eng = self.engine(xt.shape[0])
            slot = i & 1
            with torch.cuda.stream(copy):
                if consumed[slot] is not None:
                    copy.wait_event(consumed[slot])
                self.h2d_bytes = self._h2d(eng, xt, slot)
                landed = torch.cuda.Event()
                landed.record(copy)
            compute.wait_event(landed)
            eng.replay(slot)
            done = torch.cuda.Event()
            done.record(compute)
            consumed[slot] = done
            host = self._pinned_out(eng, slot)
            host.copy_(eng.output_tensor(), non_blocking=True)
            d2h = torch.cuda.Event()
            d2h.record(compute)
            # the caller may refill the host tensor it just handed over once we pull the
            # next batch: its H2D must have landed first
            landed.synchronize()
            if pending is not None:
                pending[0].synchronize()
                yield pending[1].numpy().copy()
            pending = (d2h, host)
        if pending is not None:
            pending[0].synchronize()
            yield pending[1].numpy().copy()


def run(exported: Exported, x, gather_mode: str = "fused") -> np.ndarray:
    """interp.py:36 analogue: evaluate the exported model on a batch of images."""
    return Runner(exported, gather_mode).run(x)
