"""Pinned benchmark/parity configurations (BASELINE.json `configs`).

Models are torchvision architectures with `weights=None` built after
`torch.manual_seed(seed)` in eval mode; masks come from the reference's
`score_channels(..., "l2", side="input")` + `make_masks(..., "unconstrained",
scope="per-layer")`.  The reference default scope `global` leaves ResNet-50's
fc with 1 of 2048 inputs at random init, so per-layer is pinned.
Plans and masks for each config are generated once by tools/make_assets.py with
the reference planner and committed under assets/<config>/.
"""

from __future__ import annotations

from dataclasses import dataclass
from pathlib import Path

import torch

ASSETS = Path(__file__).resolve().parent / "assets"


@dataclass(frozen=True)
class Config:
    name: str
    model: str
    sparsity: float
    scope: str = "per-layer"
    heuristic: str = "l2"
    batch: int = 1
    seed: int = 0
    native_planner: bool = False

    @property
    def asset_dir(self) -> Path:
        return ASSETS / self.name


CONFIGS = {
    # BASELINE.json configs[0]: the reference's CPU-runnable case (batch-1 oracle)
    "resnet18_s50": Config("resnet18_s50", "resnet18", 0.5, batch=1),
    # BASELINE.json configs[2]: the north-star metric
    "resnet50_s50": Config("resnet50_s50", "resnet50", 0.5, batch=256),
    # BASELINE.json configs[4] (ResNet-101 half of the throughput sweep)
    "resnet101_s50": Config("resnet101_s50", "resnet101", 0.5, batch=256),
    # BASELINE.json configs[3]: concat-heavy, maximal gather pressure.  The pure-Python
    # reference planner does not finish at 0.5; the plans are the
    # reference plan_model's with the native planner core installed (same search,
    # csrc/planner.cpp), which plans it in 0.2 s.
    "densenet121_s50": Config("densenet121_s50", "densenet121", 0.5, batch=128, native_planner=True),
}

NORTH_STAR = "resnet50_s50"


def build_torch_model(cfg: Config) -> torch.nn.Module:
    import torchvision

    torch.manual_seed(cfg.seed)
    return getattr(torchvision.models, cfg.model)(weights=None).eval()


def build_spatial_model(cfg: Config, randomize_bn: bool = False):
    from .lowering import lower, randomize_bn as _rbn

    sm = lower(build_torch_model(cfg))
    if randomize_bn:
        _rbn(sm, cfg.seed)
    return sm
