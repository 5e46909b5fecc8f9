#!/usr/bin/env python
"""Launch one conv (or gather) of a given shape a few times -- an ncu target.
python tools/one_conv.py conv N H W cin cout k stride [cstride coff variant] | gather N H cstride width n"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2307_08771_b200 import _lib, kernels as K  # noqa: E402

dev = "cuda"
g = torch.Generator().manual_seed(0)
a = sys.argv[1:]
if a[0] == "conv":
    N, H, W, cin, cout, k, st = map(int, a[1:8])
    cs = int(a[8]) if len(a) > 8 else K.pad8(cin)
    coff = int(a[9]) if len(a) > 9 else 0
    var = int(a[10]) if len(a) > 10 else 0
    x = K.Act(torch.randn(N * H * W, cs, generator=g).to(torch.bfloat16).to(dev), N, H, W, cin, coff)
    lead, cpad = _lib.conv_weight_layout(cin, coff, False, k, k)
    wg = K.permute_weights(torch.randn(cout, cin, k, k, device=dev), list(range(cout)), list(range(cin)),
                           layout="gemm", lead=lead, cpad=cpad, out_dtype=torch.bfloat16)
    pad = k // 2
    Ho, Wo = (H + 2 * pad - k) // st + 1, (W + 2 * pad - k) // st + 1
    y = K.empty_act(N, Ho, Wo, cout, dev)
    for _ in range(3):
        K.conv(x, wg, lead, cpad, cout, k, k, st, pad, y, relu=True, variant=var)
elif a[0] == "dw":
    N, H, C, k, st = map(int, a[1:6])
    x = K.Act(torch.randn(N * H * H, K.pad8(C), generator=g).to(torch.bfloat16).to(dev), N, H, H, C, 0)
    Ho = (H + 2 * (k // 2) - k) // st + 1
    y = K.empty_act(N, Ho, Ho, C, dev)
    wt = torch.randn(k * k, K.pad8(C), device=dev)
    b = torch.randn(C, device=dev)
    for _ in range(3):
        K.dwconv(x, wt, b, k, st, k // 2, "silu", y)
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    ev[0].record()
    for _ in range(20):
        K.dwconv(x, wt, b, k, st, k // 2, "silu", y)
    ev[1].record()
    torch.cuda.synchronize()
    print(f"dwconv N{N} {H}x{H} C{C} k{k} s{st}: {ev[0].elapsed_time(ev[1]) / 20 * 1e3:.1f} us")
else:
    N, H, cs, width, n = map(int, a[1:6])
    x = K.Act(torch.randn(N * H * H, cs, generator=g).to(torch.bfloat16).to(dev), N, H, H, width, 0)
    idx = sorted(torch.randperm(width, generator=g)[:n].tolist())
    idx_d = torch.tensor(idx, dtype=torch.int32, device=dev)
    y = K.empty_act(N, H, H, n, dev)
    sc = torch.rand(n, device=dev)
    for _ in range(3):
        K.gather_rows_ex(x, idx_d, K.gather_window(idx), 1, y, scale=sc, shift=sc, relu=True)
torch.cuda.synchronize()
print("ok")
