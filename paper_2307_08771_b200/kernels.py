"""Torch-tensor wrappers over the C ABI (device memory + current stream).

PyTorch is plumbing here: tensors provide device allocations and the CUDA
stream; all arithmetic happens in libupscale_b200.so.  Every wrapper raises
if the library is missing -- there is no eager fallback.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import torch

from . import _lib

_DT = {torch.float32: _lib.UB_F32, torch.float64: _lib.UB_F64, torch.bfloat16: _lib.UB_BF16}


def _p(t):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def _stream():
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def _dev_i32(seq, device) -> torch.Tensor:
    return torch.as_tensor(list(seq), dtype=torch.int32).to(device)


@dataclass
class Act:
    """An NHWC bf16 activation view: `buf` is [N*H*W, cstride]; the logical
    tensor is channels [coff, coff + C) (a SLICE view needs no copy).

    `cmap` (optional): logical channel i lives in physical column coff + cmap[i].  A
    zero-copy CONCAT whose bands start on 16-byte boundaries (each producer stores at an
    8-aligned channel offset) is such a view; cmap is None when the layout is dense."""

    buf: torch.Tensor
    N: int
    H: int
    W: int
    C: int
    coff: int = 0
    cmap: tuple | None = None

    @property
    def cstride(self) -> int:
        return self.buf.shape[-1]

    @property
    def npix(self) -> int:
        return self.N * self.H * self.W

    @property
    def width(self) -> int:
        """Physical columns spanned from coff."""
        return self.C if self.cmap is None else (self.cmap[-1] + 1 if self.cmap else 0)

    def phys(self, i: int) -> int:
        """Physical column (relative to coff) of logical channel i (-1 stays -1)."""
        if i < 0 or self.cmap is None:
            return i
        return self.cmap[i]

    def view(self, start: int, length: int) -> "Act":
        if self.cmap is None:
            return Act(self.buf, self.N, self.H, self.W, length, self.coff + start)
        sub = self.cmap[start:start + length]
        if all(b - a == 1 for a, b in zip(sub, sub[1:])):  # contiguous inside one band
            return Act(self.buf, self.N, self.H, self.W, length, self.coff + sub[0])
        return Act(self.buf, self.N, self.H, self.W, length, self.coff, tuple(sub))

    def to_nchw(self, dtype=torch.float32) -> torch.Tensor:
        cols = [self.coff + self.phys(i) for i in range(self.C)]
        t = self.buf[:, cols].reshape(self.N, self.H, self.W, self.C)
        return t.permute(0, 3, 1, 2).to(dtype)


def pad8(c: int) -> int:
    return (c + 7) // 8 * 8


def empty_act(N, H, W, C, device, cstride=None) -> Act:
    cs = cstride or pad8(C)
    return Act(torch.empty((N * H * W, cs), dtype=torch.bfloat16, device=device), N, H, W, C, 0)


def act_from_nchw(x: torch.Tensor, cstride=None) -> Act:
    N, C, H, W = x.shape
    a = empty_act(N, H, W, C, x.device, cstride)
    a.buf.zero_()
    a.buf[:, :C] = x.permute(0, 2, 3, 1).reshape(N * H * W, C).to(torch.bfloat16)
    return a


# --------------------------------------------------------------------------- export
def permute_weights(W: torch.Tensor, rows, cols, row_scale: torch.Tensor | None = None,
                    layout: str = "oihw", lead: int = 0, cpad: int = 0,
                    out_dtype=torch.float32, rows_dev=None, cols_dev=None) -> torch.Tensor:
    """apply_plan weight math (planner.py:661-673, 755-767) on a 4-D tensor."""
    assert W.is_cuda and W.dim() == 4 and W.is_contiguous()
    O, I, kh, kw = W.shape
    r = rows_dev if rows_dev is not None else _dev_i32(rows, W.device)
    c = cols_dev if cols_dev is not None else _dev_i32(cols, W.device)
    nr, nc = r.numel(), c.numel()
    if layout == "oihw":
        out = torch.empty((nr, nc, kh, kw), dtype=out_dtype, device=W.device)
        lay = _lib.UB_LAYOUT_OIHW
    elif layout == "dense":
        out = torch.empty((nr, cpad), dtype=out_dtype, device=W.device)
        lay = _lib.UB_LAYOUT_GEMM_DENSE
    elif layout == "s2d":  # [rows][kq][kq][8] (ub_conv_s2d)
        kq = (kw + 1) // 2
        out = torch.empty((nr, kq * kq * 8), dtype=out_dtype, device=W.device)
        lay = _lib.UB_LAYOUT_S2D
    else:
        out = torch.empty((nr, kh * kw, cpad), dtype=out_dtype, device=W.device)
        lay = _lib.UB_LAYOUT_GEMM
    if row_scale is not None:
        row_scale = row_scale.to(device=W.device, dtype=torch.float32).contiguous()
    _lib.call("ub_permute_weights", _p(W), _DT[W.dtype], O, I, kh, kw, _p(r), nr, _p(c), nc,
              _p(row_scale), lay, lead, cpad, _p(out), _DT[out_dtype], _stream())
    return out


def permute_vector(v: torch.Tensor, idx) -> torch.Tensor:
    """planner.py:731-733: v[perm] for per-channel vectors."""
    i = _dev_i32(idx, v.device)
    out = torch.empty(i.numel(), dtype=v.dtype, device=v.device)
    _lib.call("ub_permute_vector", _p(v), _DT[v.dtype], _p(i), i.numel(), _p(out), _stream())
    return out


# --------------------------------------------------------------------------- inference
def channel_gather(x: Act, idx_dev: torch.Tensor, y: Act) -> None:
    """Baseline-export copy: a reference GATHER node (interp.py:75-77) as index_select."""
    _lib.call("ub_channel_gather", _p(x.buf), x.cstride, x.coff, _p(idx_dev), idx_dev.numel(),
              x.npix, _p(y.buf), y.cstride, y.coff, _stream())


def channel_gather_2d(x: Act, idx_dev: torch.Tensor, stride: int, y: Act) -> None:
    """Gather channels idx of every stride-th pixel of x into the compact y (the "copy" read
    plan of a strided / gathered 1x1 conv)."""
    _lib.call("ub_channel_gather_2d", _p(x.buf), x.cstride, x.coff, _p(idx_dev), idx_dev.numel(), x.N, x.H, x.W,
              stride, _p(y.buf), y.cstride, y.coff, _stream())


def gather_rows(x: Act, idx_dev: torch.Tensor, window: tuple[int, int], stride: int, y: Act) -> None:
    """ub_gather_rows: the channels idx (all within window = (lo, hi)) of every stride-th
    pixel of x into the compact y; the source rows are staged through shared memory."""
    lo, hi = window
    _lib.call("ub_gather_rows", _p(x.buf), x.cstride, x.coff, lo, hi, _p(idx_dev), idx_dev.numel(), x.N, x.H, x.W,
              stride, _p(y.buf), y.cstride, y.coff, _stream())


def gather_rows_ex(x: Act, idx_dev: torch.Tensor, window: tuple[int, int], stride: int, y: Act,
                   pool2: bool = False, scale: torch.Tensor | None = None, shift: torch.Tensor | None = None,
                   relu: bool = False) -> None:
    """ub_gather_rows_ex: gather + the reader's BN/ReLU prologue (+ a 2x2 average pool)."""
    lo, hi = window
    _lib.call("ub_gather_rows_ex", _p(x.buf), x.cstride, x.coff, lo, hi, _p(idx_dev), idx_dev.numel(), x.N, x.H,
              x.W, stride, int(pool2), _p(scale), _p(shift), int(relu), _p(y.buf), y.cstride, y.coff, _stream())


def gather_window(idx) -> tuple[int, int]:
    kept = [int(i) for i in idx if i >= 0]
    return (min(kept), max(kept)) if kept else (0, 0)


def conv(x: Act, w: torch.Tensor, lead: int, cpad: int, cout: int, kh: int, kw: int, stride: int, pad: int,
         y: Act, gather_idx: torch.Tensor | None = None, bias: torch.Tensor | None = None,
         residual: Act | None = None, relu: bool = False, y_fp32: bool = False, variant: int = 0,
         y2: Act | None = None, y2_map: torch.Tensor | None = None) -> None:
    """One conv (ub_conv_fwd).  y2 / y2_map: compacted second store of the output channels c
    with y2_map[c] >= 0 into column y2_map[c] of y2 (the producer side of a later GATHER)."""
    Ho = (x.H + 2 * pad - kh) // stride + 1
    Wo = (x.W + 2 * pad - kw) // stride + 1
    assert y.N == x.N and y.H == Ho and y.W == Wo, "output geometry mismatch"
    d = _lib.ConvDesc()
    d.N, d.H, d.W = x.N, x.H, x.W
    d.cin = gather_idx.numel() if gather_idx is not None else x.C
    d.cout = cout
    d.kh, d.kw, d.stride, d.pad, d.Ho, d.Wo = kh, kw, stride, pad, Ho, Wo
    d.x, d.x_cstride, d.x_coff = x.buf.data_ptr(), x.cstride, x.coff
    d.gather_idx = gather_idx.data_ptr() if gather_idx is not None else None
    d.w, d.w_lead, d.w_cpad = w.data_ptr(), lead, cpad
    d.bias = bias.data_ptr() if bias is not None else None
    if residual is not None:
        d.residual, d.res_cstride, d.res_coff = residual.buf.data_ptr(), residual.cstride, residual.coff
    d.relu = int(relu)  # UB_ACT_* code (True / 1 = ReLU)
    d.y, d.y_cstride, d.y_coff = y.buf.data_ptr(), y.cstride, y.coff
    d.y_dtype = _lib.UB_F32 if y_fp32 else _lib.UB_BF16
    d.variant = variant
    if y2 is not None:
        assert y2.coff == 0 and y2_map is not None and y2_map.numel() == cout
        d.y2, d.y2_cstride, d.y2_map = y2.buf.data_ptr(), y2.cstride, y2_map.data_ptr()
    _lib.check(_lib.load().ub_conv_fwd(ctypes.byref(d), _stream()))


def conv_stem(x_nchw: torch.Tensor, idx_dev: torch.Tensor, w: torch.Tensor, kpad: int, cout: int, k: int,
              stride: int, pad: int, y: Act, bias: torch.Tensor | None = None, relu: bool = False) -> None:
    """Fused stem: im2col straight from the fp32 NCHW model input with the INPUT
    node's GATHER (idx_dev) applied on the fly; w is UB_LAYOUT_GEMM_DENSE."""
    N, C, H, W = x_nchw.shape
    Ho = (H + 2 * pad - k) // stride + 1
    Wo = (W + 2 * pad - k) // stride + 1
    assert y.N == N and y.H == Ho and y.W == Wo, "output geometry mismatch"
    d = _lib.ConvDesc()
    d.N, d.H, d.W = N, H, W
    d.cin = idx_dev.numel()
    d.cout = cout
    d.kh, d.kw, d.stride, d.pad, d.Ho, d.Wo = k, k, stride, pad, Ho, Wo
    d.x, d.x_cstride, d.x_coff = x_nchw.data_ptr(), 0, 0
    d.gather_idx = idx_dev.data_ptr()
    d.w, d.w_lead, d.w_cpad = w.data_ptr(), 0, kpad
    d.bias = bias.data_ptr() if bias is not None else None
    d.relu = int(relu)
    d.y, d.y_cstride, d.y_coff = y.buf.data_ptr(), y.cstride, y.coff
    d.y_dtype = _lib.UB_BF16
    d.x_nchw_f32, d.x_channels = 1, C
    _lib.check(_lib.load().ub_conv_fwd(ctypes.byref(d), _stream()))


def s2d_buffer(N: int, H: int, W: int, k: int, pad: int, device) -> torch.Tensor:
    """Zeroed staging buffer of the space-to-depth stem (bf16 rows of 8)."""
    _, _, nbytes = _lib.stem_s2d_geometry(N, H, W, k, pad)
    return torch.zeros(nbytes // 2, dtype=torch.bfloat16, device=device)


def stem_s2d(x_nchw: torch.Tensor, idx_dev: torch.Tensor, s_buf: torch.Tensor, w: torch.Tensor, cout: int, k: int,
             pad: int, y: Act, bias: torch.Tensor | None = None, relu: bool = False) -> None:
    """Stride-2 stem as pack (fp32 NCHW + GATHER -> 2x2-folded bf16) + stride-1 tcgen05 conv;
    w is UB_LAYOUT_S2D."""
    N, C, H, W = x_nchw.shape
    lib = _lib.load()
    _lib.check(lib.ub_stem_s2d_pack(_p(x_nchw), N, C, H, W, _p(idx_dev), idx_dev.numel(), k, pad, _p(s_buf),
                                    _stream()))
    _lib.check(lib.ub_conv_s2d(_p(s_buf), N, H, W, k, pad, _p(w), cout, _p(bias), int(relu), _p(y.buf), y.cstride,
                               y.coff, _stream()))


def stem_s2d_maxpool(x_nchw: torch.Tensor, idx_dev: torch.Tensor, s_buf: torch.Tensor, w: torch.Tensor, cout: int,
                     k: int, pad: int, y: Act, bias: torch.Tensor | None = None, relu: bool = False,
                     pool=(3, 2, 1)) -> None:
    """stem_s2d with the following 3x3/s2 max pool fused into the epilogue; y is the pooled
    output."""
    N, C, H, W = x_nchw.shape
    lib = _lib.load()
    _lib.check(lib.ub_stem_s2d_pack(_p(x_nchw), N, C, H, W, _p(idx_dev), idx_dev.numel(), k, pad, _p(s_buf),
                                    _stream()))
    _lib.check(lib.ub_conv_s2d_maxpool(_p(s_buf), N, H, W, k, pad, _p(w), cout, _p(bias), int(relu), *pool,
                                       _p(y.buf), y.cstride, y.coff, _stream()))


def stem_maxpool(x_nchw: torch.Tensor, idx_dev: torch.Tensor, w: torch.Tensor, cout: int, k: int, pad: int, y: Act,
                 bias: torch.Tensor | None = None, relu: bool = False, pool=(3, 2, 1)) -> None:
    """stem_s2d_maxpool with the pack fused into the kernel's producer (one launch, no S)."""
    N, C, H, W = x_nchw.shape
    _lib.check(_lib.load().ub_stem_maxpool(_p(x_nchw), N, C, H, W, _p(idx_dev), idx_dev.numel(), k, pad, _p(w), cout,
                                           _p(bias), int(relu), *pool, _p(y.buf), y.cstride, y.coff, _stream()))


def h2d_input_channels(host: torch.Tensor, dev: torch.Tensor, channels) -> int:
    """Pinned host NCHW fp32 -> device NCHW fp32, only `channels` (the INPUT GATHER's
    kept planes; the others are left untouched). Returns the bytes copied."""
    assert host.is_pinned() and host.is_contiguous() and dev.is_contiguous() and host.shape == dev.shape
    N, C, H, W = host.shape
    ch = (ctypes.c_int32 * len(channels))(*channels)
    nbytes = ctypes.c_longlong()
    _lib.call("ub_h2d_input_channels", _p(host), N, C, H * W, ch, len(channels), _p(dev), ctypes.byref(nbytes),
              _stream())
    return nbytes.value


def stage_input(x: torch.Tensor, y: Act, idx_dev: torch.Tensor | None = None) -> None:
    N, C, H, W = x.shape
    n = idx_dev.numel() if idx_dev is not None else C
    _lib.call("ub_stage_input", _p(x), N, C, H, W, _p(idx_dev), n, _p(y.buf), y.cstride, _stream())


def maxpool(x: Act, k: int, stride: int, pad: int, y: Act) -> None:
    _lib.call("ub_maxpool2d", _p(x.buf), x.N, x.H, x.W, x.C, x.cstride, x.coff, k, stride, pad,
              y.H, y.W, _p(y.buf), y.cstride, y.coff, _stream())


def avgpool_global(x: Act, y: Act) -> None:
    _lib.call("ub_avgpool_global", _p(x.buf), x.N, x.H * x.W, x.C, x.cstride, x.coff,
              _p(y.buf), y.cstride, y.coff, _stream())


def avgpool_gather(x: Act, idx_dev: torch.Tensor, y: Act) -> None:
    _lib.call("ub_avgpool_gather", _p(x.buf), x.N, x.H * x.W, x.C, x.cstride, x.coff, _p(idx_dev), idx_dev.numel(),
              _p(y.buf), y.cstride, y.coff, _stream())


def eltwise(a: Act, y: Act, scale=None, shift=None, b: Act | None = None, act: str = "none",
            gate: Act | None = None) -> None:
    """ub_eltwise: y = act(a * scale + shift + b) * gate (gate: per-image [N, 1, 1, C])."""
    d = _lib.EltwiseDesc()
    d.N, d.HW, d.C = a.N, a.H * a.W, a.C
    d.a, d.a_cstride, d.a_coff = a.buf.data_ptr(), a.cstride, a.coff
    d.scale = scale.data_ptr() if scale is not None else None
    d.shift = shift.data_ptr() if shift is not None else None
    if b is not None:
        d.b, d.b_cstride, d.b_coff = b.buf.data_ptr(), b.cstride, b.coff
    d.act = _lib.UB_ACT[act]
    if gate is not None:
        assert gate.H * gate.W == 1 and gate.N == a.N
        d.gate, d.gate_cstride, d.gate_coff = gate.buf.data_ptr(), gate.cstride, gate.coff
    d.y, d.y_cstride, d.y_coff = y.buf.data_ptr(), y.cstride, y.coff
    _lib.check(_lib.load().ub_eltwise(ctypes.byref(d), _stream()))


def dwconv(x: Act, w: torch.Tensor, bias: torch.Tensor | None, k: int, stride: int, pad: int, act: str,
           y: Act, part: torch.Tensor | None = None) -> None:
    """ub_dwconv: depthwise k x k conv, w fp32 [k*k, pad8(C)] (BN folded), fused activation.
    part (fp32 [N * dwconv_pool_parts(..), pad8(C)]): also write the per-tile channel sums of
    the output (ub_dwconv_pool, the fused SE pool)."""
    if part is None:
        _lib.call("ub_dwconv", _p(x.buf), x.N, x.H, x.W, x.C, x.cstride, x.coff, _p(w), _p(bias), k, stride, pad,
                  _lib.UB_ACT[act], y.H, y.W, _p(y.buf), y.cstride, y.coff, _stream())
    else:
        assert part.dtype == torch.float32 and part.shape == (x.N * dwconv_pool_parts(k, stride, y.H, y.W), pad8(y.C))
        _lib.call("ub_dwconv_pool", _p(x.buf), x.N, x.H, x.W, x.C, x.cstride, x.coff, _p(w), _p(bias), k, stride, pad,
                  _lib.UB_ACT[act], y.H, y.W, _p(y.buf), y.cstride, y.coff, _p(part), _stream())


def dwconv_pool_parts(k: int, stride: int, Ho: int, Wo: int) -> int:
    """Pool partials per image ub_dwconv_pool writes for this shape (0: no fused pool)."""
    return _lib.load().ub_dwconv_pool_parts(k, stride, Ho, Wo)


def avgpool_split(x: Act, y: Act) -> None:
    _lib.call("ub_avgpool_split", _p(x.buf), x.N, x.H * x.W, x.C, x.cstride, x.coff, _p(y.buf), y.cstride, y.coff,
              _stream())


def linear_small(x: Act, xcol_dev: torch.Tensor, w: torch.Tensor, O: int, y: Act, bias=None, act: int = 0,
                 y_fp32: bool = False) -> None:
    """ub_linear_small: CHANNEL_MIX over M = N*H*W <= 16 rows; xcol_dev = element offsets of
    the K input columns inside a row (SLICE / GATHER / column map); w bf16 [O][pad8(K)]."""
    assert w.dim() == 2 and w.shape[0] >= O
    _lib.call("ub_linear_small", _p(x.buf), x.npix, x.cstride, _p(xcol_dev), xcol_dev.numel(), _p(w), w.shape[1], O,
              _p(bias), act, _p(y.buf), _lib.UB_F32 if y_fp32 else _lib.UB_BF16, y.cstride, y.coff, _stream())


def conv_direct(x_nchw: torch.Tensor, idx_dev: torch.Tensor, w: torch.Tensor, bias, cout: int, k: int, stride: int,
                pad: int, act: int, y: Act) -> None:
    """ub_conv_direct: few-channel stem on CUDA cores; w fp32 [k*k, cin, ub_conv_direct_wcols(cout)]."""
    N, C, H, W = x_nchw.shape
    _lib.call("ub_conv_direct", _p(x_nchw), N, C, H, W, _p(idx_dev), idx_dev.numel(), _p(w), _p(bias), cout, k, stride,
              pad, act, _p(y.buf), y.cstride, y.coff, _stream())


def se_gate(x: Act, w1: torch.Tensor, C1: int, b1, act1: int, w2: torch.Tensor, C2: int, b2, act2: int,
            gate: Act, part: torch.Tensor | None = None, nparts: int = 0) -> None:
    """ub_se_gate: pool + fc1 + fc2 of a squeeze-excitation block; w1 [C1, ldw1], w2 [C2, ldw2] bf16.
    part/nparts: pool from ub_dwconv_pool's per-tile partial sums instead of re-reading x."""
    if part is None:
        _lib.call("ub_se_gate", _p(x.buf), x.N, x.H * x.W, x.C, x.cstride, x.coff, _p(w1), w1.shape[1], C1, _p(b1),
                  act1, _p(w2), w2.shape[1], C2, _p(b2), act2, _p(gate.buf), gate.cstride, gate.coff, _stream())
    else:
        _lib.call("ub_se_gate_parts", _p(x.buf), x.N, x.H * x.W, x.C, x.cstride, x.coff, _p(w1), w1.shape[1], C1,
                  _p(b1), act1, _p(w2), w2.shape[1], C2, _p(b2), act2, _p(gate.buf), gate.cstride, gate.coff,
                  _p(part), nparts, _stream())


def avgpool2d(x: Act, k: int, stride: int, pad: int, y: Act) -> None:
    _lib.call("ub_avgpool2d", _p(x.buf), x.N, x.H, x.W, x.C, x.cstride, x.coff, k, stride, pad, y.H, y.W,
              _p(y.buf), y.cstride, y.coff, _stream())


def affine_add_relu(a: Act, y: Act, scale=None, shift=None, b: Act | None = None, relu=False) -> None:
    _lib.call("ub_affine_add_relu", _p(a.buf), a.cstride, a.coff, _p(scale), _p(shift),
              _p(b.buf) if b is not None else None, b.cstride if b else 0, b.coff if b else 0,
              int(relu), a.npix, a.C, _p(y.buf), y.cstride, y.coff, _stream())
