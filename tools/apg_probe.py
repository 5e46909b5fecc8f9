"""ub_avgpool_gather at the ResNet-50 size (256 x 7 x 7 x 1816 -> 1024 kept), for ncu (dev tool)."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2307_08771_b200 import kernels as K  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 256
x = K.empty_act(N, 7, 7, 1816, "cuda")
x.buf.normal_()
idx = torch.arange(0, 1816, 2, dtype=torch.int32, device="cuda")[:1024].contiguous()
y = K.empty_act(N, 1, 1, 1024, "cuda")
for _ in range(3):
    K.avgpool_gather(x, idx, y)
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
ts = []
for _ in range(10):
    flush.zero_()
    a.record()
    K.avgpool_gather(x, idx, y)
    b.record()
    torch.cuda.synchronize()
    ts.append(a.elapsed_time(b) * 1e3)
ts.sort()
print(f"avgpool_gather N={N}: median {ts[5]:.1f} us (L2 flushed), {N * 49 * 1816 * 2 / ts[5] / 1e3:.0f} GB/s")
