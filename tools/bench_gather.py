#!/usr/bin/env python
"""Micro-benchmark of the staged read (ub_gather_rows_ex) and the dense conv behind it on
DenseNet-like shapes: python tools/bench_gather.py"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2307_08771_b200 import _lib, kernels as K  # noqa: E402


def t_us(fn, reps=20):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps * 1e3


dev = "cuda"
g = torch.Generator().manual_seed(0)
for (N, H, cs, width, n, cout) in [(128, 56, 232, 225, 64, 64), (128, 56, 232, 225, 112, 64), (128, 28, 520, 513, 240, 64),
                                   (128, 14, 1024, 1016, 496, 64), (128, 56, 232, 225, 128, 127)]:
    x = K.Act(torch.randn(N * H * H, cs, generator=g).to(torch.bfloat16).to(dev), N, H, H, width, 0)
    idx = sorted(torch.randperm(width, generator=g)[:n].tolist())
    idx_d = torch.tensor(idx, dtype=torch.int32, device=dev)
    sc = torch.rand(n, device=dev) + 0.5
    sh = torch.randn(n, device=dev)
    y = K.empty_act(N, H, H, n, dev)
    tg = t_us(lambda: K.gather_rows_ex(x, idx_d, K.gather_window(idx), 1, y, scale=sc, shift=sh, relu=True))
    lead, cpad = _lib.conv_weight_layout(n, 0, False, 1, 1)
    wg = K.permute_weights(torch.randn(cout, n, 1, 1, device=dev), list(range(cout)), list(range(n)), layout="gemm",
                           lead=lead, cpad=cpad, out_dtype=torch.bfloat16)
    out = K.empty_act(N, H, H, cout, dev)
    best = min((t_us(lambda v=v: K.conv(y, wg, lead, cpad, cout, 1, 1, 1, 0, out, relu=True, variant=v)), v)
               for v in (0, 1, 2, 32, 33, 34, 64, 65, 66))
    gbytes = N * H * H * (width + n) * 2
    cbytes = N * H * H * (n + cout) * 2
    print(f"N{N} {H}x{H} width {width} -> {n} -> {cout}: gather {tg:.1f} us ({gbytes / tg / 1e3:.0f} GB/s), "
          f"conv {best[0]:.1f} us ({cbytes / best[0] / 1e3:.0f} GB/s, variant {best[1]})", flush=True)
