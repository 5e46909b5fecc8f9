"""Conv kernel microbenchmark + correctness at production sizes (dev tool).

python tools/bench_conv.py [case ...]   -- cases are ResNet-50 layer shapes at batch 256
Each case: checks ub_conv_fwd against torch (bf16-rounded inputs, fp32 math) on
the full output, then times it with CUDA events and prints algorithmic GB/s.
"""

import os
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2307_08771_b200 import _lib, kernels as K  # noqa: E402

# name: (N, H, W, cstride, coff, cin, cout, k, stride, pad, n_gather, res, relu)
VARIANT = int(os.environ.get("UB_VARIANT", "0"))  # ub_conv_desc.variant bits

CASES = {
    "l1_conv3": (256, 56, 56, 32, 0, 32, 256, 1, 1, 0, 0, True, True),
    "l2_conv3_502": (256, 28, 28, 64, 0, 64, 502, 1, 1, 0, 0, True, True),
    "l3_conv3_1016": (256, 14, 14, 128, 0, 128, 1016, 1, 1, 0, 0, True, True),
    "l4_conv1_1024": (256, 7, 7, 1816, 0, 1024, 256, 1, 1, 0, 0, False, True),
    "fc_dense": (256, 1, 1, 1024, 0, 1024, 1000, 1, 1, 0, 0, False, False),
    "b1_l4_conv2_3x3": (1, 7, 7, 256, 0, 256, 256, 3, 1, 1, 0, False, True),
    "b1_l3_conv2_3x3": (1, 14, 14, 128, 0, 128, 128, 3, 1, 1, 0, False, True),
    "l3_conv1_cover": (256, 14, 14, 1016, 0, 1016, 128, 1, 1, 0, 0, False, True),
    "l4_conv2_3x3": (256, 7, 7, 256, 0, 256, 256, 3, 1, 1, 0, False, True),
    "l3_conv2_3x3": (256, 14, 14, 128, 0, 128, 128, 3, 1, 1, 0, False, True),
    "l2_conv2_3x3": (256, 28, 28, 64, 0, 64, 64, 3, 1, 1, 0, False, True),
    "l4_down_cover": (256, 14, 14, 1016, 0, 1016, 1816, 1, 2, 0, 0, False, False),
    "l1_conv1_gather": (256, 56, 56, 240, 0, 237, 64, 1, 1, 0, 128, False, True),
    "l1_conv1_slice": (256, 56, 56, 240, 0, 128, 64, 1, 1, 0, 0, False, True),
    "l1_conv1_dense": (256, 56, 56, 128, 0, 128, 64, 1, 1, 0, 0, False, True),
    "r50_l1_0_conv1": (256, 56, 56, 56, 0, 32, 32, 1, 1, 0, 0, False, True),
    "r50_l2_0_conv1": (256, 56, 56, 240, 70, 128, 64, 1, 1, 0, 0, False, True),
    "r50_l2_3_conv1": (256, 28, 28, 504, 137, 256, 64, 1, 1, 0, 0, False, True),
    "r50_l4_2_conv1": (256, 7, 7, 1816, 530, 1024, 256, 1, 1, 0, 0, False, True),
    "r50_l4_conv3_res": (256, 7, 7, 256, 0, 256, 1816, 1, 1, 0, 0, True, True),
    "r50_l4_0_conv1_cover": (256, 14, 14, 1016, 0, 1016, 256, 1, 1, 0, 0, False, True),
    "r50_l4_0_conv1_dense": (256, 14, 14, 512, 0, 512, 256, 1, 1, 0, 0, False, True),
    "r50_l1_0_down": (256, 56, 56, 56, 17, 32, 237, 1, 1, 0, 0, False, False),
    "l1_conv1_cs248": (256, 56, 56, 248, 0, 128, 64, 1, 1, 0, 0, False, True),
    "l1_conv1_cs256": (256, 56, 56, 256, 0, 128, 64, 1, 1, 0, 0, False, True),
    "l1_conv1_cs256_off64": (256, 56, 56, 256, 64, 128, 64, 1, 1, 0, 0, False, True),
    "l1_conv1_cs288": (256, 56, 56, 288, 0, 128, 64, 1, 1, 0, 0, False, True),
    "l1_conv1_cs320": (256, 56, 56, 320, 0, 128, 64, 1, 1, 0, 0, False, True),
    "l1_conv1_cs512": (256, 56, 56, 512, 0, 128, 64, 1, 1, 0, 0, False, True),
    "l1_conv1_c32": (256, 56, 56, 240, 0, 128, 32, 1, 1, 0, 0, False, True),
    "l1_conv2_3x3": (256, 56, 56, 64, 0, 32, 64, 3, 1, 1, 0, False, True),
    "l2_down_gather_s2": (256, 56, 56, 240, 0, 237, 512, 1, 2, 0, 128, False, False),
    "l3_conv2_3x3s2": (256, 28, 28, 128, 0, 128, 256, 3, 2, 1, 0, False, True),
    "r50_l2_0_conv2_s2": (256, 56, 56, 64, 0, 64, 64, 3, 2, 1, 0, False, True),
    "r50_l3_0_conv2_s2": (256, 28, 28, 128, 0, 128, 128, 3, 2, 1, 0, False, True),
    "r50_l4_0_conv2_s2": (256, 14, 14, 256, 0, 256, 256, 3, 2, 1, 0, False, True),
    "stem_7x7": (256, 224, 224, 8, 0, 2, 64, 7, 2, 3, 0, False, True),
    "l4_conv3": (256, 7, 7, 256, 0, 256, 2048, 1, 1, 0, 0, True, True),
    "l4_down_r18": (4, 14, 14, 232, 66, 128, 390, 1, 2, 0, 0, False, False),
    "l4_down_r18_aligned": (4, 14, 14, 232, 64, 128, 390, 1, 2, 0, 0, False, False),
    "l4_down_r18_c256": (4, 14, 14, 232, 66, 128, 256, 1, 2, 0, 0, False, False),
    "l4_1x1s1_c390": (4, 7, 7, 232, 64, 128, 390, 1, 1, 0, 0, False, False),
    "l4_1x1s1_c416": (4, 7, 7, 232, 64, 128, 416, 1, 1, 0, 0, False, False),
    "l4_1x1s1_c390_big": (64, 7, 7, 232, 64, 128, 390, 1, 1, 0, 0, False, False),
    "l1_conv3_nores": (256, 56, 56, 32, 0, 32, 256, 1, 1, 0, 0, False, True),
    "small_gather_multi": (8, 56, 56, 240, 0, 237, 64, 1, 1, 0, 128, True, True),
    "small_3x3_res_multi": (8, 56, 56, 64, 0, 64, 64, 3, 1, 1, 0, True, True),
    "small_stem_multi": (4, 224, 224, 8, 0, 2, 64, 7, 2, 3, 0, False, True),
    "stem_s2d_4x4": (256, 115, 115, 8, 0, 8, 64, 4, 1, 0, 0, False, True),
    "l1_conv2_c16": (256, 56, 56, 16, 0, 16, 64, 3, 1, 1, 0, False, True),
    # EfficientNetV2-S @ 50 % MBConv expands (1x1, few input channels, wide output)
    "eff_s5_expand": (256, 14, 14, 160, 1, 80, 710, 1, 1, 0, 0, False, True),
    "eff_s5_expand_dense": (256, 14, 14, 80, 0, 80, 710, 1, 1, 0, 0, False, True),
    "eff_s6_expand": (256, 7, 7, 256, 2, 128, 1159, 1, 1, 0, 0, False, True),
    "eff_s4_expand": (256, 14, 14, 128, 0, 64, 387, 1, 1, 0, 0, False, True),
}
ACT = os.environ.get("UB_BENCH_ACT")  # e.g. silu: the epilogue activation instead of ReLU (no check)


def run(name, check=True, iters=20, once=False):
    N, H, W, cs, coff, cin, cout, k, st, pad, ng, use_r, relu = CASES[name]
    dev = "cuda"
    g = torch.Generator(device=dev).manual_seed(0)
    xbuf = torch.randn(N * H * W, cs, device=dev, generator=g).to(torch.bfloat16)
    x = K.Act(xbuf, N, H, W, cs)
    nin = ng if ng else cin
    Wt = (torch.randn(cout, nin, k, k, device=dev, generator=g) / (nin * k * k) ** 0.5).contiguous()
    if ng:
        idx = torch.randperm(cin, device=dev, generator=g)[:ng].sort().values.to(torch.int32)
        xa, lead, cpad = x, *_lib.conv_weight_layout(ng, 0, True, k, k)
    else:
        idx = None
        xa = x.view(coff, cin)
        lead, cpad = _lib.conv_weight_layout(cin, coff, False, k, k)
    wg = K.permute_weights(Wt, list(range(cout)), list(range(nin)), layout="gemm", lead=lead, cpad=cpad,
                           out_dtype=torch.bfloat16)
    Ho = (H + 2 * pad - k) // st + 1
    Wo = (W + 2 * pad - k) // st + 1
    bias = torch.randn(cout, device=dev, generator=g)
    res = K.empty_act(N, Ho, Wo, cout, dev) if use_r else None
    if res is not None:
        res.buf.normal_(generator=g)
    y = K.empty_act(N, Ho, Wo, cout, dev)
    if ACT:
        relu, check = _lib.UB_ACT[ACT], False
    K.conv(xa, wg, lead, cpad, cout, k, k, st, pad, y, gather_idx=idx, bias=bias, residual=res, relu=relu, variant=VARIANT)
    torch.cuda.synchronize()
    if once:
        print(name, "launched once", flush=True)
        return
    err = None
    if check:
        xin = x.to_nchw()
        xin = xin[:, idx.long()] if idx is not None else xin[:, coff:coff + cin]
        ref = torch.nn.functional.conv2d(xin, Wt.to(torch.bfloat16).float(), stride=st, padding=pad)
        ref = ref + bias.view(1, -1, 1, 1)
        if res is not None:
            ref = ref + res.to_nchw()
        if relu:
            ref = ref.clamp_min(0)
        out = y.to_nchw()
        err = float((out - ref).abs().max() / ref.abs().max())
        del ref, xin
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for _ in range(3):
        K.conv(xa, wg, lead, cpad, cout, k, k, st, pad, y, gather_idx=idx, bias=bias, residual=res, relu=relu, variant=VARIANT)
    a.record()
    for _ in range(iters):
        K.conv(xa, wg, lead, cpad, cout, k, k, st, pad, y, gather_idx=idx, bias=bias, residual=res, relu=relu, variant=VARIANT)
    b.record()
    torch.cuda.synchronize()
    us = a.elapsed_time(b) / iters * 1e3
    byts = 2 * (nin * H * W + cout * Ho * Wo * (2 if use_r else 1)) * N + wg.numel() * 2
    flops = 2 * cout * nin * k * k * Ho * Wo * N
    roof = max(byts / 6554.6e9, flops / 1398.9e12) * 1e6
    print(f"{name:22s} err {err if err is None else f'{err:.2e}'}  {us:9.1f} us  {byts/us/1e3:7.1f} GB/s  "
          f"{flops/us/1e6:7.1f} TF/s  roof {roof:7.1f} us  frac {roof/us:.2f}", flush=True)


def run_stem(N=256, cin_idx=(2, 0), iters=10):
    dev = "cuda"
    x = torch.randn(N, 3, 224, 224, device=dev)
    cin = len(cin_idx)
    Wt = torch.randn(64, cin, 7, 7, device=dev) / (cin * 49) ** 0.5
    kpad = _lib.conv_stem_kpad(cin, 7, 7)
    wg = K.permute_weights(Wt.contiguous(), list(range(64)), list(range(cin)), layout="dense", cpad=kpad,
                           out_dtype=torch.bfloat16)
    idx = torch.tensor(cin_idx, dtype=torch.int32, device=dev)
    y = K.empty_act(N, 112, 112, 64, dev)
    for _ in range(3):
        K.conv_stem(x, idx, wg, kpad, 64, 7, 2, 3, y, relu=True)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(iters):
        K.conv_stem(x, idx, wg, kpad, 64, 7, 2, 3, y, relu=True)
    b.record()
    torch.cuda.synchronize()
    us = a.elapsed_time(b) / iters * 1e3
    byts = N * (3 * 224 * 224 * 4 + 64 * 112 * 112 * 2)
    print(f"stem N={N} cin={cin}: {us:.1f} us, {byts/us/1e3:.0f} GB/s (fp32 input read once + bf16 output)", flush=True)


if __name__ == "__main__":
    if "--stem" in sys.argv:
        run_stem(iters=1 if "--once" in sys.argv else 10)
        sys.exit(0)
    torch.backends.cudnn.allow_tf32 = False
    once = "--once" in sys.argv
    names = [a for a in sys.argv[1:] if not a.startswith("--")]
    for n in names or list(CASES):
        run(n, once=once)
