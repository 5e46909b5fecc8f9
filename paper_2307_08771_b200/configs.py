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
# BASELINE.json configs[1]: the MobileNetV3-Small batch-1 latency sweep, UPSCALE vs baseline
# export (depthwise convs + squeeze-excitation lowered per SURVEY.md A.5)
MOBILENET_SWEEP = (0.1, 0.3, 0.5, 0.7, 0.9, 0.95)
for _s in MOBILENET_SWEEP:
    _n = f"mobilenet_v3_small_s{round(_s * 100):02d}"
    CONFIGS[_n] = Config(_n, "mobilenet_v3_small", _s, batch=1, native_planner=True)
# BASELINE.json configs[4]: EfficientNetV2-S / ResNet-101 at 30/50/70 %, batch 256
for _s in (0.3, 0.5, 0.7):
    _n = f"efficientnet_v2_s_s{round(_s * 100):02d}"
    CONFIGS[_n] = Config(_n, "efficientnet_v2_s", _s, batch=256, native_planner=True)
for _s in (0.3, 0.7):
    _n = f"resnet101_s{round(_s * 100):02d}"
    CONFIGS[_n] = Config(_n, "resnet101", _s, batch=256, native_planner=True)

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
