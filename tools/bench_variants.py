#!/usr/bin/env python
"""Graph-timed conv variants on one shape: python tools/bench_variants.py N H W cs coff cin cout k stride [variants...]
(variant 0 = default choice (halo when eligible), 8 = generic implicit GEMM, +1/+2 producer width ...)"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2307_08771_b200 import _lib, kernels as K  # noqa: E402


def timeit(fn, reps=10):
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        for _ in range(2):
            fn()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            for _ in range(reps):
                fn()
    torch.cuda.current_stream().wait_stream(s)
    g.replay()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    a.record()
    g.replay()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps * 1e3


N, H, W, cs, coff, cin, cout, k, st = map(int, sys.argv[1:10])
variants = [int(v) for v in sys.argv[10:]] or [0, 8, 9, 10, 40, 41, 42]
dev = "cuda"
g = torch.Generator().manual_seed(0)
x = K.Act(torch.randn(N * H * W, cs, generator=g).to(torch.bfloat16).to(dev), N, H, W, cin, coff)
lead, cpad = _lib.conv_weight_layout(cin, coff, False, k, k)
wg = K.permute_weights(torch.randn(cout, cin, k, k, device=dev), list(range(cout)), list(range(cin)), layout="gemm",
                       lead=lead, cpad=cpad, out_dtype=torch.bfloat16)
pad = k // 2
Ho, Wo = (H + 2 * pad - k) // st + 1, (W + 2 * pad - k) // st + 1
y = K.empty_act(N, Ho, Wo, cout, dev)
flops = 2 * N * Ho * Wo * cout * cin * k * k
byts = 2 * N * (H * W * cin + Ho * Wo * cout)
for v in variants:
    try:
        t = timeit(lambda: K.conv(x, wg, lead, cpad, cout, k, k, st, pad, y, relu=True, variant=v))
        print(f"variant {v:6d}: {t:8.1f} us  {flops / t / 1e6:7.1f} TF/s  {byts / t / 1e3:7.1f} GB/s")
    except Exception as exc:  # noqa: BLE001
        print(f"variant {v:6d}: {exc}")
