"""Graph-timed squeeze-excitation gate (dev tool): ub_se_gate at EfficientNetV2-S / MobileNetV3 shapes,
pooling from the tensor and from ub_dwconv_pool partials.  python tools/bench_se.py"""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
sys.path.insert(0, str(Path(__file__).resolve().parent))
from paper_2307_08771_b200 import _lib, kernels as K  # noqa: E402
from bench_stem import timeit  # noqa: E402


def main():
    dev = "cuda"
    for N, H, C, C1 in ((256, 7, 1159, 64), (256, 14, 710, 40), (256, 14, 387, 16), (1, 7, 576, 144)):
        x = K.empty_act(N, H, H, C, dev)
        x.buf.normal_()
        w1 = torch.randn(C1, K.pad8(C), device=dev).to(torch.bfloat16)
        w2 = torch.randn(C, K.pad8(C1), device=dev).to(torch.bfloat16)
        gate = K.empty_act(N, 1, 1, C, dev)
        nparts = K.dwconv_pool_parts(3, 1, H, H)
        part = torch.randn(N * nparts, K.pad8(C), device=dev)
        a = (w1, C1, None, _lib.UB_ACT["silu"], w2, C, None, _lib.UB_ACT["sigmoid"], gate)
        t0 = timeit(lambda: K.se_gate(x, *a))
        t1 = timeit(lambda: K.se_gate(x, *a, part, nparts))
        print(f"se_gate N{N} {H}x{H} C{C} C1 {C1}: pool {t0:6.1f} us, partials {t1:6.1f} us")


if __name__ == "__main__":
    main()
