"""The torch.fx lowering (lowering.py) is exact: the lowered graph run by the spatial
oracle (interp.py's dispatch with real conv / BN / pool / depthwise / SE ops) equals the
torchvision model itself in fp64, for every model family the configs use -- this pins the
depthwise -> PER_CHANNEL-like node and SE mul -> positional ADD lowerings,
the DenseNet concats / transition pools and the ResNet blocks before any pruning."""

import pytest
import torch

from oracle.spatial_ref import run_spatial
from paper_2307_08771_b200.lowering import lower, randomize_bn
from paper_2307_08771_b200.ref import reslice


@pytest.mark.parametrize("name,size", [("resnet18", 64), ("densenet121", 64), ("mobilenet_v3_small", 96),
                                       ("efficientnet_v2_s", 64)])
def test_lowering_matches_torchvision_fp64(name, size):
    import torchvision

    torch.manual_seed(0)
    m = getattr(torchvision.models, name)(weights=None).eval().double()
    sm = lower(m, input_chw=(3, size, size))
    assert not reslice.graph.validate(sm.graph)
    randomize_bn(sm, 1)  # non-trivial statistics, copied back into the torch model
    for mod_name, mod in m.named_modules():
        lid = mod_name.replace(".", "_")
        if lid in sm.vectors and isinstance(mod, torch.nn.BatchNorm2d):
            v = sm.vectors[lid]
            mod.weight.data, mod.bias.data = v["weight"].double(), v["bias"].double()
            mod.running_mean.data, mod.running_var.data = v["mean"].double(), v["var"].double()
    x = torch.randn(2, 3, size, size, generator=torch.Generator().manual_seed(2), dtype=torch.float64)
    with torch.no_grad():
        ref = m(x)
        got = run_spatial(sm.graph, sm.specs, sm.weights, sm.vectors, x, dtype=torch.float64)
    assert float((ref - got).abs().max() / ref.abs().max()) < 1e-10
