"""Numerics of the sm_100a kernels against plain PyTorch fp32 references.

The conv kernel computes in bf16 x bf16 -> fp32 on tcgen05; the reference is
torch fp32 (TF32 off) on the SAME bf16-rounded inputs and weights, so the only
differences are accumulation order and the final bf16 rounding of the output.
"""

import pytest
import torch

pytestmark = pytest.mark.gpu

from paper_2307_08771_b200 import _lib, kernels as K  # noqa: E402


@pytest.fixture(autouse=True)
def _no_tf32():
    torch.backends.cudnn.allow_tf32 = False
    torch.backends.cuda.matmul.allow_tf32 = False


def _bf(t):
    return t.to(torch.bfloat16).to(torch.float32)


def _rel(a, b):
    return float((a - b).abs().max() / b.abs().max().clamp_min(1e-6))


CASES = [
    # name, N, H, W, cstride, coff, cin, cout, k, stride, pad, gather, bias, res, relu, y_fp32
    ("1x1_aligned", 2, 14, 14, 64, 0, 64, 64, 1, 1, 0, 0, False, False, False, False),
    ("1x1_misaligned_slice", 2, 7, 9, 128, 13, 100, 31, 1, 1, 0, 0, True, False, True, False),
    ("1x1_bk16", 2, 10, 10, 16, 0, 12, 48, 1, 1, 0, 0, True, False, False, False),
    ("3x3_s1", 2, 56, 56, 64, 0, 64, 64, 3, 1, 1, 0, True, False, True, False),
    ("3x3_s2_ntail", 2, 28, 28, 128, 0, 128, 130, 3, 2, 1, 0, False, False, False, False),
    ("1x1_s2_two_ntiles", 2, 28, 28, 256, 0, 256, 512, 1, 2, 0, 0, True, False, False, False),
    ("7x7_s2_stem", 1, 224, 224, 8, 0, 2, 64, 7, 2, 3, 0, True, False, True, False),
    ("gather_res_relu", 2, 14, 14, 256, 0, 256, 64, 1, 1, 0, 100, True, True, True, False),
    ("fc_gather_fp32", 4, 1, 1, 2048, 0, 2048, 1000, 1, 1, 0, 1024, True, False, False, True),
    ("3x3_slice_offset", 3, 14, 14, 96, 40, 48, 72, 3, 1, 1, 0, True, True, True, False),
    ("1x1_large_m", 8, 56, 56, 256, 0, 256, 64, 1, 1, 0, 0, False, False, False, False),
    ("gather_s2_downsample", 2, 28, 28, 240, 0, 237, 128, 1, 2, 0, 128, True, False, False, False),
    ("3x3_s1_misaligned_7x7", 4, 7, 7, 1824, 530, 1024, 40, 3, 1, 1, 0, True, False, True, False),
    ("gather_3x3_s2", 2, 28, 28, 200, 0, 200, 96, 3, 2, 1, 70, True, True, True, False),
    ("gather_3x3_s1", 3, 14, 14, 64, 0, 64, 64, 3, 1, 1, 40, False, False, True, False),
    ("two_ntiles_unaligned_390", 4, 14, 14, 232, 66, 128, 390, 1, 2, 0, 0, True, True, True, False),
    ("three_ntiles_700_gather", 2, 7, 7, 512, 0, 512, 700, 1, 1, 0, 300, True, False, False, False),
    ("1x1_s2_misaligned", 2, 56, 56, 56, 17, 32, 256, 1, 2, 0, 0, True, False, False, False),
    # narrower last A box (16 / 32 channels) for slices ending just past a 64-channel block
    ("1x1_tail16_slice", 2, 14, 14, 240, 70, 128, 64, 1, 1, 0, 0, True, False, True, False),
    ("1x1_tail32_res", 2, 14, 14, 96, 0, 84, 100, 1, 1, 0, 0, True, True, True, False),
    ("1x1_tail16_lead1_two_ntiles", 2, 7, 7, 504, 137, 256, 300, 1, 1, 0, 0, True, False, True, False),
    # packed taps (cin + lead <= 32): several filter taps per 64-wide K-block
    ("packed_3x3_c16", 2, 28, 28, 16, 0, 16, 64, 3, 1, 1, 0, True, False, True, False),
    ("packed_3x3_c24_lead5", 2, 20, 20, 64, 5, 24, 40, 3, 1, 1, 0, True, True, True, False),
    ("packed_3x3_s2_c8", 2, 30, 30, 8, 0, 8, 96, 3, 2, 1, 0, False, False, False, False),
    ("packed_5x5_c3_ragged", 2, 17, 19, 8, 0, 3, 32, 5, 1, 2, 0, True, False, False, False),
    ("packed_4x4_s1_p0_c8", 2, 115, 115, 8, 0, 8, 64, 4, 1, 0, 0, True, False, True, False),
    # halo-tile kernel (stride-1 3x3, cpad 16/32/64): padded widths 64 / 32 / 16 / 8, ragged rows
    ("halo_c32_w56", 2, 56, 56, 32, 0, 32, 32, 3, 1, 1, 0, True, False, True, False),
    ("halo_c64_w28_cout48", 3, 28, 28, 64, 0, 64, 48, 3, 1, 1, 0, True, False, False, False),
    ("halo_c64_w14_slice", 2, 14, 14, 96, 24, 64, 64, 3, 1, 1, 0, True, False, True, False),
    ("halo_c16_w7_cout256", 2, 7, 7, 16, 0, 16, 256, 3, 1, 1, 0, True, False, True, False),
    ("halo_c32_lead_h13_w5", 3, 13, 5, 48, 11, 20, 40, 3, 1, 1, 0, False, False, False, False),
    ("halo_c64_w30_cout16", 2, 17, 30, 64, 0, 64, 16, 3, 1, 1, 0, True, False, True, False),
    # halo with streamed weights (cpad > 64: 64-channel groups x taps through a TMA ring)
    ("halo_c128_w14", 3, 14, 14, 128, 0, 128, 128, 3, 1, 1, 0, True, False, True, False),
    ("halo_c256_w7_cout256", 2, 7, 7, 256, 0, 256, 256, 3, 1, 1, 0, True, False, True, False),
    ("halo_c190_lead_w14_cout100", 3, 14, 14, 256, 37, 190, 100, 3, 1, 1, 0, True, False, False, False),
    ("halo_c128_w28_ragged", 2, 19, 28, 136, 8, 128, 72, 3, 1, 1, 0, False, False, True, False),
    # stacked small images (ipt images per 128-row tile), odd N
    ("halo_c64_w7_stack_n3", 3, 7, 7, 64, 0, 64, 96, 3, 1, 1, 0, True, False, True, False),
    ("halo_c32_h3_w5_stack4_n5", 5, 3, 5, 32, 0, 32, 64, 3, 1, 1, 0, True, False, False, False),
    ("halo_c256_w7_stack_n5", 5, 7, 7, 264, 8, 256, 200, 3, 1, 1, 0, True, False, True, False),
    ("halo_c128_w15_h20_wrap", 2, 20, 15, 128, 0, 128, 64, 3, 1, 1, 0, True, False, True, False),
    ("halo_c32_w31_tma_sw64", 2, 9, 31, 32, 0, 32, 48, 3, 1, 1, 0, True, False, False, False),
    # padded width 128 (one output row per MMA tile): EfficientNetV2's 112-wide 3x3 stages
    ("halo_wp128_c16_w112", 2, 6, 112, 24, 0, 12, 22, 3, 1, 1, 0, True, False, True, False),
    ("halo_wp128_c32_w100_cout96", 2, 5, 100, 32, 0, 24, 96, 3, 1, 1, 0, True, False, False, False),
    ("halo_wp128_c64_w112_slice", 1, 4, 112, 72, 8, 64, 64, 3, 1, 1, 0, True, False, True, False),
    ("halo_wp128_c128_w70", 2, 3, 70, 128, 0, 128, 48, 3, 1, 1, 0, True, False, True, False),
    # stride-2 halo: 2x2 conv over the on-the-fly 2x2-folded input
    ("halo_s2_c64_w56", 2, 56, 56, 64, 0, 64, 64, 3, 2, 1, 0, True, False, True, False),
    ("halo_s2_c128_w28_cout100", 2, 28, 28, 128, 0, 128, 100, 3, 2, 1, 0, True, False, False, False),
    ("halo_s2_c256_w14_stack_n3", 3, 14, 14, 256, 0, 256, 256, 3, 2, 1, 0, True, False, True, False),
    ("halo_s2_c64_h15_w13_odd", 2, 15, 13, 64, 0, 64, 32, 3, 2, 1, 0, False, False, True, False),
    ("halo_s2_c100_slice_w20", 2, 20, 20, 192, 64, 100, 48, 3, 2, 1, 0, True, False, True, False),
]


@pytest.mark.parametrize("case", CASES, ids=[c[0] for c in CASES])
def test_conv_matches_torch(case):
    name, N, H, W, cs, coff, cin, cout, k, st, pad, ng, use_b, use_r, relu, yf = case
    dev = "cuda"
    g = torch.Generator(device="cpu").manual_seed(sum(map(ord, name)))
    xfull = torch.randn(N, cs, H, W, generator=g)
    x = K.act_from_nchw(xfull.to(dev))
    x.C = cs
    Wt = torch.randn(cout, cin if not ng else ng, k, k, generator=g) / (cin * k * k) ** 0.5
    if ng:
        idx = torch.randperm(cin, generator=g)[:ng].to(torch.int32)
        xin = xfull[:, idx.long()]
        xa = x
        idx_dev = idx.to(dev)
        lead, cpad = _lib.conv_weight_layout(ng, 0, True, k, k)
    else:
        xa = x.view(coff, cin)
        xin = xfull[:, coff:coff + cin]
        idx_dev = None
        lead, cpad = _lib.conv_weight_layout(cin, coff, False, k, k)
    nin = Wt.shape[1]
    wg = K.permute_weights(Wt.to(dev).contiguous(), list(range(cout)), list(range(nin)),
                           layout="gemm", lead=lead, cpad=cpad, out_dtype=torch.bfloat16)
    Ho = (H + 2 * pad - k) // st + 1
    Wo = (W + 2 * pad - k) // st + 1
    bias = torch.randn(cout, generator=g).to(dev) if use_b else None
    res = None
    ref = torch.nn.functional.conv2d(_bf(xin).to(dev), _bf(Wt).to(dev), stride=st, padding=pad)
    if use_b:
        ref = ref + bias.view(1, -1, 1, 1)
    if use_r:
        rfull = torch.randn(N, cout + 8, Ho, Wo, generator=g)
        res = K.act_from_nchw(rfull.to(dev)).view(8, cout)
        ref = ref + _bf(rfull[:, 8:8 + cout]).to(dev)
    if relu:
        ref = ref.clamp_min(0)
    if yf:
        y = K.Act(torch.full((N * Ho * Wo, K.pad8(cout)), float("nan"), device=dev), N, Ho, Wo, cout)
    else:
        y = K.empty_act(N, Ho, Wo, cout + 16, dev)
        y.buf.fill_(float("nan"))
        y = y.view(16, cout)
    K.conv(xa, wg, lead, cpad, cout, k, k, st, pad, y, gather_idx=idx_dev, bias=bias, residual=res,
           relu=relu, y_fp32=yf)
    torch.cuda.synchronize()
    out = y.buf[:, y.coff:y.coff + cout].float().reshape(N, Ho, Wo, cout).permute(0, 3, 1, 2)
    assert torch.isfinite(out).all(), f"{name}: non-finite output"
    err = _rel(out, ref)
    assert err < 1e-2, f"{name}: rel err {err}"
    if not yf:  # channels outside the write window stay untouched
        assert torch.isnan(y.buf[:, :16].float()).all()


@pytest.mark.parametrize("N,cin,idx", [(1, 2, [2, 0]), (3, 3, [0, 1, 2]), (2, 1, [1])])
def test_stem_matches_torch(N, cin, idx):
    """Fused stem: fp32 NCHW input, channel GATHER, 7x7/s2 im2col in the producer warps."""
    dev = "cuda"
    g = torch.Generator().manual_seed(N * 10 + cin)
    x = torch.randn(N, 3, 224, 224, generator=g)
    Wt = torch.randn(64, cin, 7, 7, generator=g) / (cin * 49) ** 0.5
    bias = torch.randn(64, generator=g)
    kpad = _lib.conv_stem_kpad(cin, 7, 7)
    wg = K.permute_weights(Wt.to(dev).contiguous(), list(range(64)), list(range(cin)), layout="dense", cpad=kpad,
                           out_dtype=torch.bfloat16)
    y = K.empty_act(N, 112, 112, 64, dev)
    K.conv_stem(x.to(dev), torch.tensor(idx, dtype=torch.int32, device=dev), wg, kpad, 64, 7, 2, 3, y,
                bias=bias.to(dev), relu=True)
    torch.cuda.synchronize()
    ref = torch.nn.functional.conv2d(_bf(x[:, idx]), _bf(Wt), stride=2, padding=3) + bias.view(1, -1, 1, 1)
    ref = ref.clamp_min(0)
    assert _rel(y.to_nchw().cpu(), ref) < 1e-2


@pytest.mark.parametrize("N,H,k,pad,idx,cout", [(2, 224, 7, 3, [2, 0], 64), (3, 224, 7, 3, [1], 32),
                                                (2, 37, 5, 2, [0, 2], 40), (1, 20, 3, 1, [1, 0], 16),
                                                (1, 300, 7, 3, [0, 1], 128), (2, 64, 7, 3, [2, 1], 60)])
def test_stem_s2d_matches_torch(N, H, k, pad, idx, cout):
    """Space-to-depth stem: pack (fp32 NCHW + GATHER -> 2x2-folded rows) + stride-1 tcgen05 conv."""
    dev = "cuda"
    cin = len(idx)
    g = torch.Generator().manual_seed(N * 100 + H + k)
    x = torch.randn(N, 3, H, H, generator=g)
    Wt = torch.randn(cout, cin, k, k, generator=g) / (cin * k * k) ** 0.5
    bias = torch.randn(cout, generator=g)
    wg = K.permute_weights(Wt.to(dev).contiguous(), list(range(cout)), list(range(cin)), layout="s2d",
                           out_dtype=torch.bfloat16)
    Ho = (H + 2 * pad - k) // 2 + 1
    y = K.empty_act(N, Ho, Ho, cout + 8, dev)
    y.buf.fill_(float("nan"))
    y = y.view(8, cout)
    sbuf = K.s2d_buffer(N, H, H, k, pad, dev)
    K.stem_s2d(x.to(dev), torch.tensor(idx, dtype=torch.int32, device=dev), sbuf, wg, cout, k, pad, y,
               bias=bias.to(dev), relu=True)
    torch.cuda.synchronize()
    ref = torch.nn.functional.conv2d(_bf(x[:, idx]), _bf(Wt), stride=2, padding=pad) + bias.view(1, -1, 1, 1)
    ref = ref.clamp_min(0)
    out = y.buf[:, 8:8 + cout].float().reshape(N, Ho, Ho, cout).permute(0, 3, 1, 2).cpu()
    assert torch.isfinite(out).all()
    assert _rel(out, ref) < 1e-2
    assert torch.isnan(y.buf[:, :8].float()).all()


@pytest.mark.parametrize("N,H,k,pad,idx", [(2, 224, 7, 3, [2, 0]), (1, 37, 5, 2, [1]), (2, 20, 3, 1, [0, 1]),
                                            (1, 64, 7, 4, [1, 2])])
def test_stem_s2d_pack_exact(N, H, k, pad, idx):
    """The 2x2 fold is a pure relayout + bf16 rounding: bit-exact against a torch restatement."""
    dev = "cuda"
    cin = len(idx)
    g = torch.Generator().manual_seed(N * 7 + H + k + pad)
    x = torch.randn(N, 3, H, H, generator=g)
    sbuf = K.s2d_buffer(N, H, H, k, pad, dev)
    sbuf.fill_(12345)
    lib = _lib.load()
    xd, idxd = x.to(dev), torch.tensor(idx, dtype=torch.int32, device=dev)  # alive until the kernel ran
    _lib.check(lib.ub_stem_s2d_pack(K._p(xd), N, 3, H, H, K._p(idxd), cin, k, pad, K._p(sbuf), K._stream()))
    torch.cuda.synchronize()
    Hs, Ws = _lib.stem_s2d_geometry(N, H, H, k, pad)[:2]
    xp = torch.zeros(N, cin, 2 * Hs + 2, 2 * Ws + 2)
    xp[:, :, pad:pad + H, pad:pad + H] = x[:, idx]
    xp = xp[:, :, :2 * Hs, :2 * Ws].to(torch.bfloat16)
    # S[n][Y][X][(py * 2 + px) * cin + c] = x[n][idx[c]][2Y + py - pad][2X + px - pad]
    ref = xp.reshape(N, cin, Hs, 2, Ws, 2).permute(0, 2, 4, 3, 5, 1).reshape(N, Hs, Ws, 4 * cin)
    full = torch.zeros(N, Hs, Ws, 8, dtype=torch.bfloat16)
    full[..., :4 * cin] = ref
    got = sbuf.view(torch.bfloat16)[:N * Hs * Ws * 8].reshape(N, Hs, Ws, 8).cpu()
    bad = (got.view(torch.int16) != full.view(torch.int16)).nonzero()
    assert bad.numel() == 0, (bad[:8].tolist(), got[tuple(bad[0])].item(), full[tuple(bad[0])].item())


@pytest.mark.parametrize("N,H,idx,cout", [(3, 224, [2, 0], 64), (5, 64, [1], 60), (2, 100, [0, 2], 32),
                                         (3, 224, [2, 0], 32), (2, 224, [1], 24), (4, 112, [0, 2], 16),
                                         (37, 224, [2, 0], 32)])
def test_stem_s2d_maxpool_matches_torch(N, H, idx, cout):
    """Stem with the 3x3/s2/p1 max pool fused into its epilogue (bands of pooled rows,
    halo tiles, row hand-over ring) == conv -> bias -> ReLU -> max_pool2d.  cout <= 32 with an
    even pooled height takes the four-conv-rows-per-MMA (quad) form; the fused-pack launch
    (always the pair form) must agree with it bit for bit."""
    dev = "cuda"
    k, pad = 7, 3
    cin = len(idx)
    g = torch.Generator().manual_seed(N * 1000 + H + cout)
    x = torch.randn(N, 3, H, H, generator=g)
    Wt = torch.randn(cout, cin, k, k, generator=g) / (cin * k * k) ** 0.5
    bias = torch.randn(cout, generator=g)
    wg = K.permute_weights(Wt.to(dev).contiguous(), list(range(cout)), list(range(cin)), layout="s2d",
                           out_dtype=torch.bfloat16)
    Ho = (H + 2 * pad - k) // 2 + 1
    Hp = Ho // 2
    y = K.empty_act(N, Hp, Hp, cout + 8, dev)
    y.buf.fill_(float("nan"))
    y = y.view(8, cout)
    sbuf = K.s2d_buffer(N, H, H, k, pad, dev)
    xd, idxd = x.to(dev), torch.tensor(idx, dtype=torch.int32, device=dev)
    K.stem_s2d_maxpool(xd, idxd, sbuf, wg, cout, k, pad, y, bias=bias.to(dev), relu=True)
    # the fused-pack form (one launch, no S buffer) is bit-identical
    y_f = K.empty_act(N, Hp, Hp, cout + 8, dev)
    y_f.buf.fill_(float("nan"))
    y_f = y_f.view(8, cout)
    K.stem_maxpool(xd, idxd, wg, cout, k, pad, y_f, bias=bias.to(dev), relu=True)
    torch.cuda.synchronize()
    assert torch.equal(y_f.buf.view(torch.int16), y.buf.view(torch.int16))
    torch.cuda.synchronize()
    conv = torch.nn.functional.conv2d(_bf(x[:, idx]), _bf(Wt), stride=2, padding=pad) + bias.view(1, -1, 1, 1)
    ref = torch.nn.functional.max_pool2d(_bf(conv.clamp_min(0)), 3, 2, 1)
    out = y.buf[:, 8:8 + cout].float().reshape(N, Hp, Hp, cout).permute(0, 3, 1, 2).cpu()
    assert torch.isfinite(out).all()
    assert _rel(out, ref) < 1e-2
    assert torch.isnan(y.buf[:, :8].float()).all()


def test_permute_weights_bit_exact():
    dev = "cuda"
    g = torch.Generator().manual_seed(0)
    W = torch.randn(40, 24, 3, 3, generator=g, dtype=torch.float64)
    rows = [3, 1, 0, 39, 7, -1, 12]
    cols = [5, 2, 23, -1, 0]
    out = K.permute_weights(W.to(dev), rows, cols, out_dtype=torch.float64)
    ref = torch.zeros(len(rows), len(cols), 3, 3, dtype=torch.float64)
    for i, r in enumerate(rows):
        for j, c in enumerate(cols):
            if r >= 0 and c >= 0:
                ref[i, j] = W[r, c]
    assert torch.equal(out.cpu(), ref)


@pytest.mark.parametrize("rows", [False, True])
@pytest.mark.parametrize("N,H,W,cs,coff,idx,stride", [
    (2, 9, 9, 40, 0, [5, 3, -1, 39, 0, 17, 18], 1),
    (3, 14, 14, 64, 8, [1, 2, 3, 50, 7, 9, 11, 13, 40, 41], 2),
    (2, 7, 5, 1024, 16, list(range(0, 1000, 3)), 2),
    (2, 6, 6, 136, 3, [130, 2, -1, 77, 4, 5, 6, 100, 99], 1),   # window crosses 8-channel blocks, odd offset
    (1, 3, 3, 2048, 0, list(range(2047, -1, -1)), 1),           # full reversed row
    (2, 5, 5, 64, 57, [-1, -1, 6], 1),                           # one kept channel at the row's end
])
def test_channel_gather_2d(N, H, W, cs, coff, idx, stride, rows):
    """Gather + stride subsample into a compact buffer: bit-exact, zero-padded to pad8(n)."""
    dev = "cuda"
    g = torch.Generator().manual_seed(N + H + len(idx))
    x = torch.randn(N, cs, H, W, generator=g)
    xa = K.act_from_nchw(x.to(dev)).view(coff, cs - coff)
    idx_t = torch.tensor(idx, dtype=torch.int32)
    Ho, Wo = (H - 1) // stride + 1, (W - 1) // stride + 1
    y = K.empty_act(N, Ho, Wo, len(idx), dev)
    y.buf.fill_(float("nan"))
    if rows:
        K.gather_rows(xa, idx_t.to(dev), K.gather_window(idx), stride, y)
    else:
        K.channel_gather_2d(xa, idx_t.to(dev), stride, y)
    torch.cuda.synchronize()
    ref = torch.zeros(N, K.pad8(len(idx)), Ho, Wo)
    for i, j in enumerate(idx):
        if j >= 0:
            ref[:, i] = _bf(x[:, coff + j, ::stride, ::stride])
    got = y.buf.float().reshape(N, Ho, Wo, -1).permute(0, 3, 1, 2).cpu()
    assert torch.equal(got, ref)


def test_channel_gather_and_pools():
    dev = "cuda"
    g = torch.Generator().manual_seed(1)
    x = torch.randn(2, 40, 9, 9, generator=g)
    xa = K.act_from_nchw(x.to(dev))
    idx = torch.tensor([5, 3, -1, 39, 0, 17, 18], dtype=torch.int32)
    y = K.empty_act(2, 9, 9, len(idx), dev)
    K.channel_gather(xa, idx.to(dev), y)
    ref = torch.zeros(2, len(idx), 9, 9)
    for i, j in enumerate(idx.tolist()):
        if j >= 0:
            ref[:, i] = _bf(x[:, j])
    torch.cuda.synchronize()
    assert torch.equal(y.to_nchw().cpu(), ref)

    yp = K.empty_act(2, 5, 5, 40, dev)
    K.maxpool(xa, 3, 2, 1, yp)
    refp = torch.nn.functional.max_pool2d(_bf(x), 3, 2, 1)
    assert torch.equal(yp.to_nchw().cpu(), refp)

    ya = K.empty_act(2, 1, 1, 40, dev)
    K.avgpool_global(xa, ya)
    refa = _bf(x).mean(dim=(2, 3))
    assert _rel(ya.to_nchw().cpu().reshape(2, 40), refa) < 1e-2


@pytest.mark.parametrize("N,H,cin,cout,res,variant,kind", [
    (2, 14, 64, 237, True, 0, "random"), (3, 7, 128, 1016, True, 65, "random"), (2, 9, 32, 40, False, 0, "random"),
    (2, 14, 128, 1016, True, 0, "lo_halves"), (2, 56, 32, 237, True, 0, "hi_halves"),
    (2, 14, 128, 1016, True, 2, "random"), (1, 5, 64, 130, False, 1, "all")])
def test_conv_dual_store(N, H, cin, cout, res, variant, kind):
    """Compacted second store (ub_conv_desc.y2): per 64-channel group the kept channels land in
    consecutive columns from an 8-aligned base, the group's pad columns are zero; bit-exact
    copies of y; columns past the layout untouched; y unchanged by the second store."""
    dev = "cuda"
    g = torch.Generator().manual_seed(cout + N)
    x = K.act_from_nchw(torch.randn(N, cin, H, H, generator=g).to(dev))
    Wt = torch.randn(cout, cin, 1, 1, generator=g) / cin ** 0.5
    lead, cpad = _lib.conv_weight_layout(cin, 0, False, 1, 1)
    wg = K.permute_weights(Wt.to(dev).contiguous(), list(range(cout)), list(range(cin)), layout="gemm", lead=lead,
                           cpad=cpad, out_dtype=torch.bfloat16)
    bias = torch.randn(cout, generator=g).to(dev)
    r = K.act_from_nchw(torch.randn(N, cout, H, H, generator=g).to(dev)) if res else None
    if kind == "random":
        kept = sorted(torch.randperm(cout, generator=g)[:cout // 2 + 3].tolist())
    elif kind == "lo_halves":  # every lane keeps exactly one of (j, j + 32): only the low halves
        kept = [c for c in range(cout) if (c // 32) % 2 == 0 and c % 3]
    elif kind == "hi_halves":
        kept = [c for c in range(cout) if (c // 32) % 2 == 1]
    else:
        kept = list(range(cout))
    m, cols, width = [-1] * cout, [], 0
    for grp in range(0, cout, 64):
        ks = [c for c in kept if grp <= c < grp + 64]
        for k, c in enumerate(ks):
            m[c] = width + k
        cols += [width + k for k in range(len(ks))]
        width += K.pad8(len(ks))
    y = K.empty_act(N, H, H, cout, dev)
    y2 = K.empty_act(N, H, H, width + 8, dev)
    y2.buf.fill_(float("nan"))
    K.conv(x, wg, lead, cpad, cout, 1, 1, 1, 0, y, bias=bias, residual=r, relu=True, variant=variant, y2=y2,
           y2_map=torch.tensor(m, dtype=torch.int32, device=dev))
    yref = K.empty_act(N, H, H, cout, dev)
    K.conv(x, wg, lead, cpad, cout, 1, 1, 1, 0, yref, bias=bias, residual=r, relu=True, variant=variant)
    torch.cuda.synchronize()
    assert torch.equal(y.buf[:, :cout], yref.buf[:, :cout])
    assert torch.equal(y2.buf[:, cols].view(torch.int16), y.buf[:, kept].view(torch.int16))
    pad = sorted(set(range(width)) - set(cols))
    if pad:
        assert (y2.buf[:, pad].float() == 0).all()
    assert torch.isnan(y2.buf[:, width:].float()).all()


@pytest.mark.parametrize("HW,C", [(49, 1816), (81, 44), (5, 64)])
def test_avgpool_global_sequential_sum(HW, C):
    """Global average pool == fp32 sum in pixel order, / HW, rounded to bf16 (both the 8-channel
    vector kernel (C % 8 == 0) and the scalar one)."""
    import numpy as np
    dev = "cuda"
    g = torch.Generator().manual_seed(HW + C)
    x = torch.randn(2, C, 1, HW, generator=g)
    xa = K.act_from_nchw(x.to(dev))
    ya = K.empty_act(2, 1, 1, C, dev)
    K.avgpool_global(xa, ya)
    torch.cuda.synchronize()
    xb = _bf(x).numpy().astype(np.float32)
    s = np.zeros((2, C), dtype=np.float32)
    for p in range(HW):
        s = s + xb[:, :, 0, p]
    ref = torch.from_numpy(s / np.float32(HW)).to(torch.bfloat16).float()
    assert torch.equal(ya.to_nchw().cpu().reshape(2, C), ref)


@pytest.mark.parametrize("H,C,coff,k,st,pd", [(112, 64, 0, 3, 2, 1), (57, 48, 16, 3, 2, 1), (20, 24, 8, 2, 2, 0),
                                             (30, 60, 0, 3, 2, 1)])
def test_maxpool_rows_matches_torch(H, C, coff, k, st, pd):
    """Row-staged max pool (bit-exact: max of bf16 values); C = 60 is the ragged-tail case."""
    dev = "cuda"
    g = torch.Generator().manual_seed(H + C)
    ragged = C % 8 != 0
    x = torch.randn(3, C + coff + (0 if ragged else 8), H, H + 3, generator=g)
    xa = K.act_from_nchw(x.to(dev)).view(coff, C)
    Ho = (H + 2 * pd - k) // st + 1
    Wo = (H + 3 + 2 * pd - k) // st + 1
    yp = K.empty_act(3, Ho, Wo, C if ragged else C + 8, dev)
    yp = yp if ragged else yp.view(8, C)
    K.maxpool(xa, k, st, pd, yp)
    torch.cuda.synchronize()
    refp = torch.nn.functional.max_pool2d(_bf(x[:, coff:coff + C]), k, st, pd)
    assert torch.equal(yp.to_nchw().cpu(), refp)


def test_stage_input_gathers_channels():
    dev = "cuda"
    x = torch.randn(2, 3, 8, 8)
    y = K.empty_act(2, 8, 8, 2, dev, cstride=8)
    K.stage_input(x.to(dev), y, torch.tensor([2, 0], dtype=torch.int32, device=dev))
    torch.cuda.synchronize()
    got = y.buf.float().cpu().reshape(2, 8, 8, 8)
    assert torch.equal(got[..., 0], _bf(x[:, 2]))
    assert torch.equal(got[..., 1], _bf(x[:, 0]))
    assert (got[..., 2:] == 0).all()


@pytest.mark.parametrize("HW,C,coff,cs,N", [(49, 1816, 0, 1816, 3), (49, 64, 8, 80, 3), (3, 4096, 0, 4096, 3),
                                            (81, 40, 0, 40, 3), (49, 1816, 0, 1816, 80), (130, 64, 8, 80, 150)])
def test_avgpool_gather_matches_pool_then_gather(HW, C, coff, cs, N):
    """ub_avgpool_gather == global pool (fp32, / HW, bf16) followed by the GATHER (-1 -> 0),
    compacted, in both forms (N = 3: phased small-batch kernel; N = 80 / 150: the large one;
    HW = 130 > 56 takes the phased loop twice); checked against an fp64 host sum rounded to bf16 (the kernel's pixel-phase
    partial sums may differ from a sequential fp32 sum by one bf16 ulp)."""
    import numpy as np
    dev = "cuda"
    g = torch.Generator().manual_seed(HW * 7 + C)
    xw = torch.randn(N, cs, 1, HW, generator=g)
    xa = K.act_from_nchw(xw.to(dev)).view(coff, C)
    perm = torch.randperm(C, generator=g)[: max(4, C // 2)].sort().values.tolist()
    idx = perm[:3] + [-1] + perm[3:]
    idx_dev = torch.tensor(idx, dtype=torch.int32, device=dev)
    ya = K.empty_act(N, 1, 1, len(idx), dev)
    K.avgpool_gather(xa, idx_dev, ya)
    torch.cuda.synchronize()
    xb = _bf(xw).numpy().astype(np.float64)[:, coff:coff + C, 0, :]
    pooled = (xb.sum(axis=2) / HW).astype(np.float32)
    ref = np.zeros((N, len(idx)), dtype=np.float32)
    for j, c in enumerate(idx):
        if c >= 0:
            ref[:, j] = pooled[:, c]
    ref = torch.from_numpy(ref).to(torch.bfloat16).float()
    got = ya.to_nchw().cpu().reshape(N, len(idx))
    assert (got[:, 3] == 0).all()
    assert torch.allclose(got, ref, rtol=8e-3, atol=1e-6)


PAIR_CASES = [
    # name, N, H, W, cstride, coff, cin, cout, variant extra
    ("fc_1000_m2", 256, 1, 1, 1024, 0, 1024, 1000, 0),
    ("cover_odd_mtiles", 3, 14, 14, 1016, 0, 1016, 128, 0),
    ("slice_tail16_cout64", 4, 14, 14, 240, 70, 128, 64, 0),
    ("slice_lead2_two_ntiles", 8, 7, 7, 1816, 530, 1024, 256, 8192),
    ("single_pair_short", 1, 15, 15, 64, 0, 64, 96, 0),
]


@pytest.mark.parametrize("case", PAIR_CASES, ids=[c[0] for c in PAIR_CASES])
def test_conv_pair_mode_bit_exact(case):
    """Variant +32768 (two M tiles per streamed weight box, four TMEM accumulators) gives the
    same bits as the default schedule (same k-block order per tile) and matches torch."""
    name, N, H, W, cs, coff, cin, cout, extra = case
    dev = "cuda"
    g = torch.Generator(device="cpu").manual_seed(sum(map(ord, name)))
    xfull = torch.randn(N, cs, H, W, generator=g)
    x = K.act_from_nchw(xfull.to(dev))
    xa = x.view(coff, cin)
    Wt = torch.randn(cout, cin, 1, 1, generator=g) / cin ** 0.5
    lead, cpad = _lib.conv_weight_layout(cin, coff, False, 1, 1)
    wg = K.permute_weights(Wt.to(dev).contiguous(), list(range(cout)), list(range(cin)),
                           layout="gemm", lead=lead, cpad=cpad, out_dtype=torch.bfloat16)
    bias = torch.randn(cout, generator=g).to(dev)
    outs = []
    for v in (1 | 4 | extra, 1 | 4 | 32768 | extra):
        y = K.empty_act(N, H, W, cout, dev)
        y.buf.fill_(float("nan"))
        K.conv(xa, wg, lead, cpad, cout, 1, 1, 1, 0, y, bias=bias, relu=True, variant=v)
        torch.cuda.synchronize()
        outs.append(y.buf[:, :cout].clone())
    ref = torch.nn.functional.conv2d(_bf(xfull[:, coff:coff + cin]).to(dev), _bf(Wt).to(dev))
    ref = (ref + bias.view(1, -1, 1, 1)).clamp_min(0)
    errs = [_rel(o.float().reshape(N, H, W, cout).permute(0, 3, 1, 2), ref) for o in outs]
    assert max(errs) < 1e-2, (name, errs)
    assert torch.equal(outs[0].view(torch.int16), outs[1].view(torch.int16)), name


@pytest.mark.parametrize("N,cout", [(4, 1000), (256, 1000), (2, 70)])
def test_conv_fp32_classifier_32_channel_tiles_bit_exact(N, cout):
    """Variant +65536 (32-channel N tiles for an fp32 output): same bits as the 64-channel
    tiling (same k-block order per output), no write outside each tile's own columns."""
    dev = "cuda"
    g = torch.Generator().manual_seed(N + cout)
    cin = 1024
    x = K.act_from_nchw(torch.randn(N, cin, 1, 1, generator=g).to(dev))
    Wt = torch.randn(cout, cin, 1, 1, generator=g) / cin ** 0.5
    lead, cpad = _lib.conv_weight_layout(cin, 0, False, 1, 1)
    wg = K.permute_weights(Wt.to(dev).contiguous(), list(range(cout)), list(range(cin)),
                           layout="gemm", lead=lead, cpad=cpad, out_dtype=torch.bfloat16)
    bias = torch.randn(cout, generator=g).to(dev)
    outs = []
    for v in (0, 65536):
        y = K.Act(torch.full((N, K.pad8(cout)), float("nan"), device=dev), N, 1, 1, cout)
        K.conv(x, wg, lead, cpad, cout, 1, 1, 1, 0, y, bias=bias, y_fp32=True, variant=v)
        torch.cuda.synchronize()
        outs.append(y.buf.clone())
    assert torch.equal(outs[0][:, :cout], outs[1][:, :cout])
    assert torch.isnan(outs[1][:, cout:]).all()
    ref = x.to_nchw().reshape(N, cin).to(dev) @ _bf(Wt).reshape(cout, cin).to(dev).T + bias
    assert _rel(outs[1][:, :cout], ref) < 1e-2


@pytest.mark.parametrize("layout,kk,cin,lead", [("gemm", 1, 100, 5), ("gemm", 3, 64, 0), ("gemm", 3, 24, 3),
                                                 ("s2d", 7, 2, 0), ("dense", 7, 3, 0)])
def test_production_bf16_layouts_bit_exact_vs_fp32_oihw(layout, kk, cin, lead):
    """The production weight operands (bf16, BN scale folded into the rows, K-major GEMM /
    space-to-depth / dense im2col layouts) are bit-identical to the fp32 OIHW result of the
    same plan maps, scaled in fp32 and rounded once to bf16."""
    dev = "cuda"
    g = torch.Generator().manual_seed(kk * 100 + cin)
    O, I = 48, cin + 7
    W = torch.randn(O, I, kk, kk, generator=g)
    rows = [5, 0, 47, -1, 12, 3, 30, 31]
    cols = list(range(I - 1, I - 1 - cin, -1))
    cols[1] = -1
    scale = (0.5 + torch.rand(len(rows), generator=g)).to(dev)
    Wd = W.to(dev).contiguous()
    oihw = K.permute_weights(Wd, rows, cols, out_dtype=torch.float32)
    ref = (oihw * scale.view(-1, 1, 1, 1)).to(torch.bfloat16)  # one fp32 product, one RN to bf16
    if layout == "gemm":
        lead_, cpad = _lib.conv_weight_layout(cin, lead, False, kk, kk)
        got = K.permute_weights(Wd, rows, cols, row_scale=scale, layout="gemm", lead=lead_, cpad=cpad,
                                out_dtype=torch.bfloat16)
        assert got.shape == (len(rows), kk * kk, cpad)
        want = torch.zeros(len(rows), kk * kk, cpad, dtype=torch.bfloat16, device=dev)
        want[:, :, lead_:lead_ + cin] = ref.permute(0, 2, 3, 1).reshape(len(rows), kk * kk, cin)
    elif layout == "s2d":
        got = K.permute_weights(Wd, rows, cols, row_scale=scale, layout="s2d", out_dtype=torch.bfloat16)
        kq = (kk + 1) // 2
        want = torch.zeros(len(rows), kq, kq, 2, 2, 2, dtype=torch.bfloat16, device=dev)  # [o][dy][dx][py][px][c]
        for dy in range(kq):
            for dx in range(kq):
                for py in range(2):
                    for px in range(2):
                        r, s = 2 * dy + py, 2 * dx + px
                        if r < kk and s < kk:
                            want[:, dy, dx, py, px, :cin] = ref[:, :, r, s]
        want = want.reshape(len(rows), kq * kq * 8)
    else:
        kpad = _lib.conv_stem_kpad(cin, kk, kk)
        got = K.permute_weights(Wd, rows, cols, row_scale=scale, layout="dense", cpad=kpad, out_dtype=torch.bfloat16)
        want = torch.zeros(len(rows), kpad, dtype=torch.bfloat16, device=dev)
        want[:, :kk * kk * cin] = ref.permute(0, 2, 3, 1).reshape(len(rows), -1)
    torch.cuda.synchronize()
    assert torch.equal(got.view(torch.int16), want.view(torch.int16))


@pytest.mark.parametrize("pool2,affine,relu,stride", [(False, True, True, 1), (True, True, True, 1),
                                                      (True, False, False, 1), (False, True, False, 2)])
def test_gather_rows_prologue_and_pool(pool2, affine, relu, stride):
    """ub_gather_rows_ex: gather through a column map + the reader's BN/ReLU prologue
    (+ the 2x2 average pool moved in front of a 1x1 conv) vs torch fp32 on the bf16 input."""
    dev = "cuda"
    g = torch.Generator().manual_seed(int(pool2) * 10 + int(affine) + stride)
    N, C, H, W, cs, coff = 2, 150, 10, 12, 168, 8
    x = torch.randn(N, cs, H, W, generator=g)
    xa = K.act_from_nchw(x.to(dev))
    idx = [3, 140, -1, 7, 8, 9, 77, 31, 0, 149, 60]
    sc = 0.5 + torch.rand(len(idx), generator=g)
    sh = torch.randn(len(idx), generator=g)
    Ho, Wo = (H // 2, W // 2) if pool2 else ((H - 1) // stride + 1, (W - 1) // stride + 1)
    y = K.empty_act(N, Ho, Wo, len(idx), dev)
    y.buf.fill_(float("nan"))
    xv = xa.view(coff, C)
    K.gather_rows_ex(xv, torch.tensor(idx, dtype=torch.int32, device=dev), K.gather_window(idx), stride, y,
                     pool2=pool2, scale=sc.to(dev) if affine else None, shift=sh.to(dev) if affine else None,
                     relu=relu)
    torch.cuda.synchronize()
    xs = _bf(x)[:, coff:coff + C]
    ref = torch.zeros(N, K.pad8(len(idx)), H, W)
    for i, j in enumerate(idx):
        if j >= 0:
            v = xs[:, j]
            if affine:
                v = sc[i] * v + sh[i]
            if relu:
                v = v.clamp_min(0)
            ref[:, i] = v
    ref = torch.nn.functional.avg_pool2d(ref, 2, 2) if pool2 else ref[:, :, ::stride, ::stride]
    got = y.buf.float().reshape(N, Ho, Wo, -1).permute(0, 3, 1, 2).cpu()
    assert torch.isfinite(got).all()
    assert (got - ref).abs().max() <= 1e-2 * ref.abs().max() + 1e-6
    assert (got[:, len(idx):] == 0).all()


@pytest.mark.parametrize("act", ["none", "relu", "relu6", "hardswish", "hardsigmoid", "silu", "sigmoid"])
@pytest.mark.parametrize("aligned", [True, False])
def test_eltwise(act, aligned):
    """ub_eltwise: y = act(a * scale + shift + b) * gate, vector (16-byte) and scalar paths."""
    dev = "cuda"
    g = torch.Generator().manual_seed(len(act) + int(aligned))
    N, C, H, W = 3, 37, 5, 6
    coff = 8 if aligned else 3
    a = K.act_from_nchw(torch.randn(N, C + 16, H, W, generator=g).to(dev) * 3).view(coff, C)
    b = K.act_from_nchw(torch.randn(N, C + 8, H, W, generator=g).to(dev)).view(8 if aligned else 1, C)
    gate = K.act_from_nchw(torch.rand(N, C, 1, 1, generator=g).to(dev))
    sc, sh = torch.randn(C, generator=g), torch.randn(C, generator=g)
    y = K.empty_act(N, H, W, C, dev)
    K.eltwise(a, y, sc.to(dev), sh.to(dev), b, act, gate)
    torch.cuda.synchronize()
    fns = {"none": lambda v: v, "relu": torch.relu, "relu6": lambda v: v.clamp(0, 6),
           "hardswish": torch.nn.functional.hardswish, "hardsigmoid": torch.nn.functional.hardsigmoid,
           "silu": torch.nn.functional.silu, "sigmoid": torch.sigmoid}
    ref = fns[act](a.to_nchw().cpu() * sc.view(1, -1, 1, 1) + sh.view(1, -1, 1, 1) + b.to_nchw().cpu())
    ref = ref * gate.to_nchw().cpu()
    assert _rel(y.to_nchw().cpu(), ref) < 1e-2


@pytest.mark.parametrize("N,HW,C,act", [(3, 49, 1159, "none"), (2, 196, 710, "silu"), (1, 9, 13, "none"),
                                        (5, 3, 64, "hardswish")])
def test_eltwise_gate_only(N, HW, C, act):
    """The squeeze-excitation `mul` (gate only: ub_eltwise's dedicated gate kernel), output at
    a channel offset of a wider row; bit-exact against the same bf16 arithmetic in torch."""
    dev = "cuda"
    g = torch.Generator().manual_seed(N * HW + C)
    cs = (C + 7) // 8 * 8 + 16
    a = K.act_from_nchw(torch.randn(N, cs, HW, 1, generator=g).to(dev)).view(8, C)
    gate = K.act_from_nchw(torch.rand(N, C, 1, 1, generator=g).to(dev))
    yb = K.empty_act(N, HW, 1, cs, dev)
    yb.buf.fill_(7.0)
    y = yb.view(16, C)
    K.eltwise(a, y, None, None, None, act, gate)
    torch.cuda.synchronize()
    fns = {"none": lambda v: v, "silu": torch.nn.functional.silu, "hardswish": torch.nn.functional.hardswish}
    ref = fns[act](a.to_nchw().cpu()) * gate.to_nchw().cpu()
    got = y.to_nchw().cpu()
    assert _rel(got, ref) < 1e-2
    if act == "none":
        assert torch.equal(got, ref.to(torch.bfloat16).float())
    full = yb.buf.float().cpu()
    assert (full[:, :16] == 7.0).all() and (full[:, 16 + C:] == 7.0).all()  # neighbours untouched


@pytest.mark.parametrize("N,HW,C,act", [(2, 49, 1159, "none"), (3, 196, 24, "relu"), (1, 9, 13, "silu")])
def test_eltwise_add_only(N, HW, C, act):
    """A residual ADD no epilogue absorbed (ub_eltwise's add kernel): y = act(a + b) at channel
    offsets of wider rows; bit-exact against the same fp32 sum rounded to bf16."""
    dev = "cuda"
    g = torch.Generator().manual_seed(N * HW * 7 + C)
    cs = (C + 7) // 8 * 8 + 16
    a = K.act_from_nchw(torch.randn(N, cs, HW, 1, generator=g).to(dev)).view(8, C)
    b = K.act_from_nchw(torch.randn(N, cs, HW, 1, generator=g).to(dev)).view(16, C)
    yb = K.empty_act(N, HW, 1, cs, dev)
    yb.buf.fill_(7.0)
    y = yb.view(8, C)
    K.eltwise(a, y, None, None, b, act)
    torch.cuda.synchronize()
    fns = {"none": lambda v: v, "relu": torch.relu, "silu": torch.nn.functional.silu}
    ref = fns[act](a.to_nchw().cpu() + b.to_nchw().cpu())
    got = y.to_nchw().cpu()
    assert _rel(got, ref) < 1e-2
    if act != "silu":
        assert torch.equal(got, ref.to(torch.bfloat16).float())
    full = yb.buf.float().cpu()
    assert (full[:, :8] == 7.0).all() and (full[:, 8 + C:] == 7.0).all()


def test_avgpool2d():
    dev = "cuda"
    x = torch.randn(2, 45, 13, 14, generator=torch.Generator().manual_seed(3))
    xa = K.act_from_nchw(x.to(dev))
    for k, s, p in ((2, 2, 0), (3, 1, 1), (3, 2, 1)):
        Ho, Wo = (13 + 2 * p - k) // s + 1, (14 + 2 * p - k) // s + 1
        y = K.empty_act(2, Ho, Wo, 45, dev)
        K.avgpool2d(xa, k, s, p, y)
        torch.cuda.synchronize()
        ref = torch.nn.functional.avg_pool2d(_bf(x), k, s, p)
        assert _rel(y.to_nchw().cpu(), ref) < 1e-2


@pytest.mark.parametrize("k,stride,act,C", [(3, 1, "relu", 16), (3, 2, "hardswish", 72), (5, 1, "hardswish", 96),
                                             (5, 2, "silu", 40), (3, 1, "none", 13)])
def test_dwconv(k, stride, act, C):
    """ub_dwconv (depthwise conv + folded BN + activation) vs torch fp32 on bf16 inputs."""
    dev = "cuda"
    g = torch.Generator().manual_seed(k * 10 + stride + C)
    N, H, W = 2, 17, 14
    x = torch.randn(N, C, H, W, generator=g)
    w = torch.randn(C, 1, k, k, generator=g) / k
    b = torch.randn(C, generator=g)
    xa = K.act_from_nchw(x.to(dev))
    pad = k // 2
    Ho, Wo = (H + 2 * pad - k) // stride + 1, (W + 2 * pad - k) // stride + 1
    y = K.empty_act(N, Ho, Wo, C, dev)
    wt = torch.zeros(k * k, K.pad8(C))
    wt[:, :C] = w.reshape(C, k * k).t()
    K.dwconv(xa, wt.to(dev), b.to(dev), k, stride, pad, act, y)
    torch.cuda.synchronize()
    fns = {"none": lambda v: v, "relu": torch.relu, "hardswish": torch.nn.functional.hardswish,
           "silu": torch.nn.functional.silu}
    ref = fns[act](torch.nn.functional.conv2d(_bf(x), w, b, stride=stride, padding=pad, groups=C))
    assert _rel(y.to_nchw().cpu(), ref) < 1e-2


@pytest.mark.parametrize("act", ["hardswish", "silu", "hardsigmoid"])
def test_conv_epilogue_activations(act):
    """Conv epilogues apply UB_ACT_* activations (TMA-store and halo paths)."""
    dev = "cuda"
    g = torch.Generator().manual_seed(len(act))
    fns = {"hardswish": torch.nn.functional.hardswish, "silu": torch.nn.functional.silu,
           "hardsigmoid": torch.nn.functional.hardsigmoid}
    for k, cin, cout in ((1, 64, 96), (3, 64, 64)):
        x = torch.randn(2, cin, 14, 14, generator=g)
        Wt = torch.randn(cout, cin, k, k, generator=g) / (cin * k * k) ** 0.5
        bias = torch.randn(cout, generator=g)
        xa = K.act_from_nchw(x.to(dev))
        lead, cpad = _lib.conv_weight_layout(cin, 0, False, k, k)
        wg = K.permute_weights(Wt.to(dev).contiguous(), list(range(cout)), list(range(cin)), layout="gemm",
                               lead=lead, cpad=cpad, out_dtype=torch.bfloat16)
        y = K.empty_act(2, 14, 14, cout, dev)
        K.conv(xa, wg, lead, cpad, cout, k, k, 1, k // 2, y, bias=bias.to(dev), relu=_lib.UB_ACT[act])
        torch.cuda.synchronize()
        ref = fns[act](torch.nn.functional.conv2d(_bf(x), _bf(Wt), bias, padding=k // 2))
        assert _rel(y.to_nchw().cpu(), ref) < 1e-2, (k, act)


@pytest.mark.parametrize("act,cin,cout", [("silu", 80, 710), ("hardswish", 64, 320), ("relu", 128, 512),
                                          ("none", 96, 256), ("silu", 40, 130)])
def test_conv_1x1_four_epilogue_groups(act, cin, cout):
    """TMA-fed 1x1 without residual and N tiles >= 128 channels: the four-group epilogue
    (producer warps 16-23 drain too, one output slot per warp) vs torch fp32."""
    dev = "cuda"
    g = torch.Generator().manual_seed(cin * 7 + cout)
    N, H = 6, 14
    x = torch.randn(N, cin, H, H, generator=g)
    Wt = torch.randn(cout, cin, 1, 1, generator=g) / cin ** 0.5
    bias = torch.randn(cout, generator=g)
    xa = K.act_from_nchw(x.to(dev))
    lead, cpad = _lib.conv_weight_layout(cin, 0, False, 1, 1)
    wg = K.permute_weights(Wt.to(dev).contiguous(), list(range(cout)), list(range(cin)), layout="gemm",
                           lead=lead, cpad=cpad, out_dtype=torch.bfloat16)
    y = K.empty_act(N, H, H, cout, dev)
    K.conv(xa, wg, lead, cpad, cout, 1, 1, 1, 0, y, bias=bias.to(dev), relu=_lib.UB_ACT[act])
    torch.cuda.synchronize()
    fns = {"none": lambda v: v, "relu": torch.relu, "silu": torch.nn.functional.silu,
           "hardswish": torch.nn.functional.hardswish}
    ref = fns[act](torch.nn.functional.conv2d(_bf(x), _bf(Wt), bias))
    assert _rel(y.to_nchw().cpu(), ref) < 1e-2


@pytest.mark.parametrize("M,KK,O,fp32,act", [(1, 72, 425, False, "hardsigmoid"), (4, 2048, 1000, True, "none"),
                                             (16, 37, 9, False, "relu"), (3, 512, 1000, True, "none")])
def test_linear_small(M, KK, O, fp32, act):
    """ub_linear_small (CHANNEL_MIX over <= 16 rows on CUDA cores) through a gather with a
    zero-filled entry, vs torch fp32 on the bf16 operands."""
    dev = "cuda"
    g = torch.Generator().manual_seed(M * 1000 + KK)
    src_w = KK + 20
    x = torch.randn(M, src_w, 1, 1, generator=g)
    xa = K.act_from_nchw(x.to(dev))
    perm = torch.randperm(src_w, generator=g)[:KK].tolist()
    perm[min(3, KK - 1)] = -1
    W = torch.randn(O, KK, generator=g) / KK ** 0.5
    b = torch.randn(O, generator=g)
    wd = torch.zeros(O, (KK + 7) // 8 * 8)
    wd[:, :KK] = W
    y = K.empty_act(M, 1, 1, O, dev) if not fp32 else None
    if fp32:
        y = K.Act(torch.zeros(M, (O + 3) // 4 * 4, device=dev), M, 1, 1, O, 0)
    xcol = torch.tensor([xa.coff + p if p >= 0 else -1 for p in perm], dtype=torch.int32, device=dev)
    K.linear_small(xa, xcol, wd.to(torch.bfloat16).to(dev), O, y, bias=b.to(dev), act=_lib.UB_ACT[act], y_fp32=fp32)
    torch.cuda.synchronize()
    xin = torch.stack([_bf(x[:, p, 0, 0]) if p >= 0 else torch.zeros(M) for p in perm], dim=1)
    fns = {"none": lambda v: v, "relu": torch.relu, "hardsigmoid": torch.nn.functional.hardsigmoid}
    ref = fns[act](xin @ _bf(W).t() + b)
    got = y.buf[:, :O].float().cpu()
    assert _rel(got, ref) < 1e-2


@pytest.mark.parametrize("N,H,C", [(1, 56, 12), (2, 28, 433), (1, 7, 1024)])
def test_avgpool_split(N, H, C):
    dev = "cuda"
    x = torch.randn(N, C, H, H, generator=torch.Generator().manual_seed(C))
    xa = K.act_from_nchw(x.to(dev))
    y = K.empty_act(N, 1, 1, C, dev)
    K.avgpool_split(xa, y)
    torch.cuda.synchronize()
    assert _rel(y.to_nchw().cpu(), _bf(x).mean(dim=(2, 3), keepdim=True)) < 1e-2


@pytest.mark.parametrize("cin,k,s,cout,act,H,W", [(3, 3, 2, 24, "silu", 37, 45), (2, 3, 2, 16, "hardswish", 37, 45),
                                                   (3, 7, 2, 70, "relu", 37, 45), (1, 5, 1, 40, "none", 37, 45),
                                                   (3, 3, 2, 22, "silu", 37, 45), (2, 3, 2, 13, "relu", 37, 45),
                                                   (3, 3, 1, 7, "none", 37, 45),
                                                   # 16-byte-multiple widths
                                                   (3, 3, 2, 24, "silu", 67, 64), (2, 3, 2, 16, "hardswish", 40, 36),
                                                   (3, 7, 2, 70, "relu", 33, 52), (1, 3, 1, 9, "none", 21, 20)])
def test_conv_direct(cin, k, s, cout, act, H, W):
    """ub_conv_direct (few-channel stem on CUDA cores, INPUT GATHER applied) vs torch fp32."""
    dev = "cuda"
    g = torch.Generator().manual_seed(cin * 100 + k * 10 + cout)
    N, C = 2, 3
    x = torch.randn(N, C, H, W, generator=g)
    idx = [2, 0, 1][:cin]
    Wt = torch.randn(cout, cin, k, k, generator=g) / (cin * k * k) ** 0.5
    b = torch.randn(cout, generator=g)
    pad = k // 2
    Ho, Wo = (H + 2 * pad - k) // s + 1, (W + 2 * pad - k) // s + 1
    wd = torch.zeros(k * k, cin, _lib.load().ub_conv_direct_wcols(cout))
    wd[:, :, :cout] = Wt.permute(2, 3, 1, 0).reshape(k * k, cin, cout)
    y = K.empty_act(N, Ho, Wo, cout, dev)
    K.conv_direct(x.to(dev), torch.tensor(idx, dtype=torch.int32, device=dev), wd.to(dev), b.to(dev), cout, k, s, pad,
                  _lib.UB_ACT[act], y)
    torch.cuda.synchronize()
    fns = {"none": lambda v: v, "relu": torch.relu, "hardswish": torch.nn.functional.hardswish,
           "silu": torch.nn.functional.silu}
    ref = fns[act](torch.nn.functional.conv2d(x[:, idx], Wt, b, stride=s, padding=pad))
    assert _rel(y.to_nchw().cpu(), ref) < 1e-2


@pytest.mark.parametrize("N,H,C,C1,C2,acts", [(1, 56, 16, 8, 16, ("relu", "hardsigmoid")),
                                              (3, 14, 730, 48, 730, ("silu", "sigmoid")),
                                              (2, 7, 576, 144, 570, ("relu", "hardsigmoid"))])
def test_se_gate(N, H, C, C1, C2, acts):
    """ub_se_gate (pool + fc1 + fc2 in one launch) vs torch fp32 on the bf16 operands."""
    dev = "cuda"
    g = torch.Generator().manual_seed(C + C1)
    x = torch.randn(N, C, H, H, generator=g)
    W1 = torch.randn(C1, C, generator=g) / C ** 0.5
    W2 = torch.randn(C2, C1, generator=g) / C1 ** 0.5
    b1, b2 = torch.randn(C1, generator=g), torch.randn(C2, generator=g)

    def pack(W):
        t = torch.zeros(W.shape[0], (W.shape[1] + 7) // 8 * 8, dtype=torch.bfloat16)
        t[:, :W.shape[1]] = W.to(torch.bfloat16)
        return t.to(dev)

    xa = K.act_from_nchw(x.to(dev))
    gate = K.empty_act(N, 1, 1, C2, dev)
    K.se_gate(xa, pack(W1), C1, b1.to(dev), _lib.UB_ACT[acts[0]], pack(W2), C2, b2.to(dev), _lib.UB_ACT[acts[1]],
              gate)
    torch.cuda.synchronize()
    fns = {"relu": torch.relu, "silu": torch.nn.functional.silu, "sigmoid": torch.sigmoid,
           "hardsigmoid": torch.nn.functional.hardsigmoid}
    pooled = _bf(x).mean(dim=(2, 3))
    h = fns[acts[0]](pooled @ _bf(W1).t() + b1)
    ref = fns[acts[1]](h @ _bf(W2).t() + b2)
    assert _rel(gate.to_nchw().cpu().reshape(N, C2), ref) < 1e-2


@pytest.mark.parametrize("N,H,stride,C", [(3, 14, 1, 730), (3, 28, 2, 192), (3, 7, 1, 13), (3, 17, 1, 96),
                                          (45, 7, 1, 1159), (32, 14, 1, 100)])
def test_dwconv_fused_se_pool(N, H, stride, C):
    """ub_dwconv_pool's per-tile channel sums == the sums of its own stored output, and
    ub_se_gate_parts over them == ub_se_gate re-reading the tensor (fp32 order only; N >= 32
    takes the several-images-per-CTA gate kernel, N = 45 a ragged last image group)."""
    dev = "cuda"
    g = torch.Generator().manual_seed(H * 100 + C)
    k = 3
    x = torch.randn(N, C, H, H, generator=g)
    w = torch.randn(C, 1, k, k, generator=g) / k
    b = torch.randn(C, generator=g)
    xa = K.act_from_nchw(x.to(dev))
    Ho = (H + 2 - k) // stride + 1
    nparts = K.dwconv_pool_parts(k, stride, Ho, Ho)
    assert nparts == ((Ho + 7) // 8) ** 2
    y = K.empty_act(N, Ho, Ho, C, dev)
    y0 = K.empty_act(N, Ho, Ho, C, dev)
    wt = torch.zeros(k * k, K.pad8(C))
    wt[:, :C] = w.reshape(C, k * k).t()
    part = torch.full((N * nparts, K.pad8(C)), float("nan"), device=dev)
    K.dwconv(xa, wt.to(dev), b.to(dev), k, stride, 1, "silu", y, part)
    K.dwconv(xa, wt.to(dev), b.to(dev), k, stride, 1, "silu", y0)
    torch.cuda.synchronize()
    out = y.to_nchw().float()
    assert torch.equal(out, y0.to_nchw().float())  # the fused pool leaves the output unchanged
    sums = part.view(N, nparts, -1).sum(1)[:, :C]
    assert torch.allclose(sums, out.sum(dim=(2, 3)), rtol=1e-5, atol=1e-3)
    C1, C2 = 24, C
    W1 = torch.randn(C1, C, generator=g) / C ** 0.5
    W2 = torch.randn(C2, C1, generator=g) / C1 ** 0.5

    def pack(W):
        t = torch.zeros(W.shape[0], (W.shape[1] + 7) // 8 * 8, dtype=torch.bfloat16)
        t[:, :W.shape[1]] = W.to(torch.bfloat16)
        return t.to(dev)

    g1, g2 = K.empty_act(N, 1, 1, C2, dev), K.empty_act(N, 1, 1, C2, dev)
    args = (pack(W1), C1, None, _lib.UB_ACT["silu"], pack(W2), C2, None, _lib.UB_ACT["sigmoid"])
    K.se_gate(y, *args, g1)
    K.se_gate(y, *args, g2, part, nparts)
    torch.cuda.synchronize()
    assert (g1.to_nchw().float() - g2.to_nchw().float()).abs().max().item() <= 2 ** -8


@pytest.mark.parametrize("width,n,affine,stride", [(1016, 496, True, 1), (600, 300, False, 1), (2040, 1500, True, 1),
                                                   (1016, 508, False, 2), (2040, 1020, False, 2)])
def test_gather_rows_wide(width, n, affine, stride):
    """ub_gather_rows_ex with more than 256 gathered channels (the lane-interleaved form)."""
    dev = "cuda"
    g = torch.Generator().manual_seed(width + n)
    N, H, cs = 2, 5, (width + 7) // 8 * 8
    x = torch.randn(N, cs, H, H, generator=g)
    xa = K.act_from_nchw(x.to(dev))
    idx = sorted(torch.randperm(width, generator=g)[:n].tolist())
    idx[5] = -1
    sc, sh = 0.5 + torch.rand(n, generator=g), torch.randn(n, generator=g)
    Ho = (H - 1) // stride + 1
    y = K.empty_act(N, Ho, Ho, n, dev)
    K.gather_rows_ex(xa, torch.tensor(idx, dtype=torch.int32, device=dev), K.gather_window(idx), stride, y,
                     scale=sc.to(dev) if affine else None, shift=sh.to(dev) if affine else None, relu=affine)
    torch.cuda.synchronize()
    ref = torch.zeros(N, n, Ho, Ho)
    for i, j in enumerate(idx):
        if j >= 0:
            v = _bf(x[:, j, ::stride, ::stride])
            ref[:, i] = (sc[i] * v + sh[i]).clamp_min(0) if affine else v
    got = y.to_nchw().cpu()
    assert (got - ref).abs().max() <= 1e-2 * ref.abs().max()
