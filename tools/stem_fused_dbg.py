"""Run the fused-pack stem once at N=1 (dev tool, for compute-sanitizer)."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2307_08771_b200 import kernels as K  # noqa: E402

dev = "cuda"
N = int(sys.argv[1]) if len(sys.argv) > 1 else 1
x = torch.randn(N, 3, 224, 224, device=dev)
idx = torch.tensor([2, 0], dtype=torch.int32, device=dev)
Wt = torch.randn(64, 2, 7, 7, device=dev) / 10
wg = K.permute_weights(Wt, list(range(64)), [0, 1], layout="s2d", out_dtype=torch.bfloat16)
y = K.empty_act(N, 56, 56, 64, dev)
K.stem_maxpool(x, idx, wg, 64, 7, 3, y, bias=torch.zeros(64, device=dev), relu=True)
torch.cuda.synchronize()
print("ok", float(y.buf.float().abs().sum()))
