"""H2D bandwidth of the input copy (dev tool): contiguous pinned vs per-channel 2-D copies."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2307_08771_b200 import kernels as K  # noqa: E402


def t(fn, reps=10):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    fn()
    torch.cuda.synchronize()
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


host = torch.randn(256, 3, 224, 224).pin_memory()
dev = torch.empty(256, 3, 224, 224, device="cuda")
nb = host.numel() * 4
ms = t(lambda: dev.copy_(host, non_blocking=True))
print(f"contiguous 3ch {nb / 1e6:.0f} MB: {ms:.3f} ms  {nb / ms / 1e6:.1f} GB/s")
ms = t(lambda: K.h2d_input_channels(host, dev, [0, 2]))
print(f"2 channels (2-D copies) {nb * 2 / 3 / 1e6:.0f} MB: {ms:.3f} ms  {nb * 2 / 3 / ms / 1e6:.1f} GB/s")
h2 = torch.randn(256, 2, 224, 224).pin_memory()
d2 = torch.empty(256, 2, 224, 224, device="cuda")
ms = t(lambda: d2.copy_(h2, non_blocking=True))
print(f"contiguous 2ch {h2.numel() * 4 / 1e6:.0f} MB: {ms:.3f} ms  {h2.numel() * 4 / ms / 1e6:.1f} GB/s")
