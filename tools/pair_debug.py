"""Pair-mode (variant +32768) localisation probe (dev tool): error vs torch per variant combo."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2307_08771_b200 import _lib, kernels as K  # noqa: E402


def run(N, H, cs, coff, cin, cout, v):
    dev = "cuda"
    g = torch.Generator().manual_seed(0)
    xfull = torch.randn(N, cs, H, H, generator=g)
    xa = K.act_from_nchw(xfull.to(dev)).view(coff, cin)
    Wt = torch.randn(cout, cin, 1, 1, generator=g) / cin ** 0.5
    lead, cpad = _lib.conv_weight_layout(cin, coff, False, 1, 1)
    wg = K.permute_weights(Wt.to(dev).contiguous(), list(range(cout)), list(range(cin)),
                           layout="gemm", lead=lead, cpad=cpad, out_dtype=torch.bfloat16)
    y = K.empty_act(N, H, H, cout, dev)
    y.buf.fill_(float("nan"))
    K.conv(xa, wg, lead, cpad, cout, 1, 1, 1, 0, y, relu=False, variant=v)
    torch.cuda.synchronize()
    ref = torch.nn.functional.conv2d(xfull[:, coff:coff + cin].to(torch.bfloat16).float().to(dev),
                                     Wt.to(torch.bfloat16).float().to(dev))
    ref = ref.permute(0, 2, 3, 1).reshape(-1, cout)
    out = y.buf[:, :cout].float()
    err = (out - ref).abs()
    bad = (err > 0.05 * ref.abs().max())
    rows = bad.any(1).nonzero().flatten()
    cols = bad.any(0).nonzero().flatten()
    print(f"v={v:6d} maxerr {err.max().item():.3g} bad rows {rows.numel()} [{rows[:4].tolist()}..] "
          f"bad cols {cols.numel()} [{cols[:6].tolist()}..] nan {torch.isnan(out).sum().item()}")
    if rows.numel() and False:
        for j in (1, 2, 5, 33):
            d = (out[:, j:j + 1] - ref).abs().max(0).values
            k = int(d.argmin())
            print(f"   out col {j} closest ref col {k} (maxdiff {d[k].item():.3g}); out/ref[:, j] ratio "
                  f"{(out[:8, j] / ref[:8, j]).tolist()}")
        print("   out[0,:8]", out[0, :8].tolist(), "ref[0,:8]", ref[0, :8].tolist())


for shape in [(2, 16, 256, 0, 256, 128)]:
    print(shape)
    for v in (1 | 4, 1 | 4 | 32768):
        run(*shape, v)
