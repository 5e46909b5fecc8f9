"""Compare one halo conv case against torch and print where it differs (dev tool).
python tools/halo_debug.py N H W cs coff cin cout stride [variant]"""
import os
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2307_08771_b200 import _lib, kernels as K  # noqa: E402

N, H, W, cs, coff, cin, cout, st = [int(v) for v in sys.argv[1:9]]
dev = "cuda"
g = torch.Generator().manual_seed(0)
xfull = torch.randn(N, cs, H, W, generator=g)
x = K.act_from_nchw(xfull.to(dev))
x.C = cs
xa = x.view(coff, cin)
Wt = torch.randn(cout, cin, 3, 3, generator=g) / (cin * 9) ** 0.5
lead, cpad = _lib.conv_weight_layout(cin, coff, False, 3, 3)
wg = K.permute_weights(Wt.to(dev).contiguous(), list(range(cout)), list(range(cin)), layout="gemm", lead=lead,
                       cpad=cpad, out_dtype=torch.bfloat16)
Ho = (H + 2 - 3) // st + 1
Wo = (W + 2 - 3) // st + 1
y = K.empty_act(N, Ho, Wo, cout, dev)
y.buf.fill_(float("nan"))
K.conv(xa, wg, lead, cpad, cout, 3, 3, st, 1, y)
torch.cuda.synchronize()
ref = torch.nn.functional.conv2d(xfull[:, coff:coff + cin].to(torch.bfloat16).float(),
                                 Wt.to(torch.bfloat16).float(), stride=st, padding=1)
out = y.to_nchw().cpu().float()
err = (out - ref).abs()
bad = ~(err < 0.05)
print("lead", lead, "cpad", cpad, "bad", int(bad.sum()), "of", bad.numel())
if bad.any():
    idx = bad.nonzero()
    print("images", sorted(set(idx[:, 0].tolist()))[:10])
    print("channels", sorted(set(idx[:, 1].tolist()))[:20])
    print("rows", sorted(set(idx[:, 2].tolist())))
    print("cols", sorted(set(idx[:, 3].tolist())))
    for n in range(min(N, 2)):
        print(n, "row-wise bad counts", bad[n].sum(dim=(0, 2)).tolist())
