"""ctypes binding of the C ABI in include/upscale_b200.h.

The product path has no fallback: if `libupscale_b200.so` is missing or fails
to load, every GPU entry point raises `ExtensionMissingError`.
"""

from __future__ import annotations

import ctypes
import threading
from pathlib import Path

LIB_PATH = Path(__file__).resolve().parent / "libupscale_b200.so"

UB_OK = 0
UB_EINVAL = -1
UB_EUNSUPPORTED = -2
UB_ECUDA = -3

UB_F32, UB_F64, UB_BF16 = 0, 1, 2
UB_LAYOUT_OIHW, UB_LAYOUT_GEMM, UB_LAYOUT_GEMM_DENSE, UB_LAYOUT_S2D = 0, 1, 2, 3

c_int, c_ll, c_vp = ctypes.c_int, ctypes.c_longlong, ctypes.c_void_p


class ExtensionMissingError(RuntimeError):
    """The sm_100a library is not built / not loadable (no CPU fallback exists)."""


class UBError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"[ub status {code}] {msg}")
        self.code = code


class ConvDesc(ctypes.Structure):
    _fields_ = [
        ("N", c_int), ("H", c_int), ("W", c_int),
        ("cin", c_int), ("cout", c_int),
        ("kh", c_int), ("kw", c_int), ("stride", c_int), ("pad", c_int),
        ("Ho", c_int), ("Wo", c_int),
        ("x", c_vp), ("x_cstride", c_int), ("x_coff", c_int),
        ("gather_idx", c_vp),
        ("w", c_vp), ("w_lead", c_int), ("w_cpad", c_int),
        ("bias", c_vp),
        ("residual", c_vp), ("res_cstride", c_int), ("res_coff", c_int),
        ("relu", c_int),
        ("y", c_vp), ("y_cstride", c_int), ("y_coff", c_int),
        ("y_dtype", c_int),
        ("x_nchw_f32", c_int), ("x_channels", c_int),
        ("variant", c_int),
        ("y2", c_vp), ("y2_cstride", c_int), ("y2_map", c_vp),
    ]


UB_ACT = {"none": 0, "relu": 1, "relu6": 2, "hardswish": 3, "hardsigmoid": 4, "silu": 5, "sigmoid": 6}


class EltwiseDesc(ctypes.Structure):
    _fields_ = [
        ("N", c_int), ("HW", c_int), ("C", c_int),
        ("a", c_vp), ("a_cstride", c_int), ("a_coff", c_int),
        ("scale", c_vp), ("shift", c_vp),
        ("b", c_vp), ("b_cstride", c_int), ("b_coff", c_int),
        ("act", c_int),
        ("gate", c_vp), ("gate_cstride", c_int), ("gate_coff", c_int),
        ("y", c_vp), ("y_cstride", c_int), ("y_coff", c_int),
    ]


# name -> (restype, argtypes); must match include/upscale_b200.h exactly.
SIGNATURES = {
    "ub_last_error": (ctypes.c_char_p, []),
    "ub_abi_version": (c_int, []),
    "ub_launch_count": (c_ll, []),
    "ub_reset_launch_count": (None, []),
    "ub_permute_weights": (c_int, [c_vp, c_int, c_int, c_int, c_int, c_int, c_vp, c_int, c_vp, c_int,
                                   c_vp, c_int, c_int, c_int, c_vp, c_int, c_vp]),
    "ub_permute_vector": (c_int, [c_vp, c_int, c_vp, c_int, c_vp, c_vp]),
    "ub_index_faults": (c_int, [ctypes.POINTER(ctypes.c_ulonglong)]),
    "ub_channel_gather": (c_int, [c_vp, c_int, c_int, c_vp, c_int, c_ll, c_vp, c_int, c_int, c_vp]),
    "ub_channel_gather_2d": (c_int, [c_vp, c_int, c_int, c_vp, c_int, c_int, c_int, c_int, c_int, c_vp, c_int, c_int,
                                     c_vp]),
    "ub_gather_rows": (c_int, [c_vp, c_int, c_int, c_int, c_int, c_vp, c_int, c_int, c_int, c_int, c_int, c_vp,
                               c_int, c_int, c_vp]),
    "ub_gather_rows_ex": (c_int, [c_vp, c_int, c_int, c_int, c_int, c_vp, c_int, c_int, c_int, c_int, c_int, c_int,
                                  c_vp, c_vp, c_int, c_vp, c_int, c_int, c_vp]),
    "ub_eltwise": (c_int, [ctypes.POINTER(EltwiseDesc), c_vp]),
    "ub_avgpool2d": (c_int, [c_vp, c_int, c_int, c_int, c_int, c_int, c_int, c_int, c_int, c_int, c_int, c_int, c_vp,
                             c_int, c_int, c_vp]),
    "ub_dwconv": (c_int, [c_vp, c_int, c_int, c_int, c_int, c_int, c_int, c_vp, c_vp, c_int, c_int, c_int, c_int,
                          c_int, c_int, c_vp, c_int, c_int, c_vp]),
    "ub_dwconv_pool_parts": (c_int, [c_int, c_int, c_int, c_int]),
    "ub_dwconv_pool": (c_int, [c_vp, c_int, c_int, c_int, c_int, c_int, c_int, c_vp, c_vp, c_int, c_int, c_int, c_int,
                               c_int, c_int, c_vp, c_int, c_int, c_vp, c_vp]),
    "ub_avgpool_split": (c_int, [c_vp, c_int, c_int, c_int, c_int, c_int, c_vp, c_int, c_int, c_vp]),
    "ub_linear_small": (c_int, [c_vp, c_int, c_int, c_vp, c_int, c_vp, c_int, c_int, c_vp, c_int, c_vp, c_int, c_int,
                                c_int, c_vp]),
    "ub_conv_direct_wcols": (c_int, [c_int]),
    "ub_conv_direct": (c_int, [c_vp, c_int, c_int, c_int, c_int, c_vp, c_int, c_vp, c_vp, c_int, c_int, c_int, c_int,
                               c_int, c_vp, c_int, c_int, c_vp]),
    "ub_se_gate": (c_int, [c_vp, c_int, c_int, c_int, c_int, c_int, c_vp, c_int, c_int, c_vp, c_int, c_vp, c_int,
                           c_int, c_vp, c_int, c_vp, c_int, c_int, c_vp]),
    "ub_se_gate_parts": (c_int, [c_vp, c_int, c_int, c_int, c_int, c_int, c_vp, c_int, c_int, c_vp, c_int, c_vp, c_int,
                                 c_int, c_vp, c_int, c_vp, c_int, c_int, c_vp, c_int, c_vp]),
    "ub_conv_weight_layout": (c_int, [c_int, c_int, c_int, ctypes.POINTER(c_int), ctypes.POINTER(c_int)]),
    "ub_conv_weight_layout2": (c_int, [c_int, c_int, c_int, c_int, c_int, ctypes.POINTER(c_int),
                                       ctypes.POINTER(c_int)]),
    "ub_conv_fwd": (c_int, [ctypes.POINTER(ConvDesc), c_vp]),
    "ub_conv_stem_kpad": (c_int, [c_int, c_int, c_int]),
    "ub_stem_s2d_geometry": (c_int, [c_int, c_int, c_int, c_int, c_int, ctypes.POINTER(c_int),
                                     ctypes.POINTER(c_int), ctypes.POINTER(c_ll)]),
    "ub_stem_s2d_pack": (c_int, [c_vp, c_int, c_int, c_int, c_int, c_vp, c_int, c_int, c_int, c_vp, c_vp]),
    "ub_conv_s2d": (c_int, [c_vp, c_int, c_int, c_int, c_int, c_int, c_vp, c_int, c_vp, c_int, c_vp, c_int,
                            c_int, c_vp]),
    "ub_conv_s2d_maxpool": (c_int, [c_vp, c_int, c_int, c_int, c_int, c_int, c_vp, c_int, c_vp, c_int, c_int,
                                    c_int, c_int, c_vp, c_int, c_int, c_vp]),
    "ub_stem_maxpool": (c_int, [c_vp, c_int, c_int, c_int, c_int, c_vp, c_int, c_int, c_int, c_vp, c_int, c_vp, c_int,
                                c_int, c_int, c_int, c_vp, c_int, c_int, c_vp]),
    "ub_h2d_input_channels": (c_int, [c_vp, c_int, c_int, c_int, ctypes.POINTER(ctypes.c_int32), c_int, c_vp,
                                      ctypes.POINTER(c_ll), c_vp]),
    "ub_plan_order_segment": (c_int, [c_int, c_vp, c_vp, c_int, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp]),
    "ub_stage_input": (c_int, [c_vp, c_int, c_int, c_int, c_int, c_vp, c_int, c_vp, c_int, c_vp]),
    "ub_maxpool2d": (c_int, [c_vp, c_int, c_int, c_int, c_int, c_int, c_int, c_int, c_int, c_int,
                             c_int, c_int, c_vp, c_int, c_int, c_vp]),
    "ub_avgpool_global": (c_int, [c_vp, c_int, c_int, c_int, c_int, c_int, c_vp, c_int, c_int, c_vp]),
    "ub_avgpool_gather": (c_int, [c_vp, c_int, c_int, c_int, c_int, c_int, c_vp, c_int, c_vp, c_int, c_int,
                                  c_vp]),
    "ub_affine_add_relu": (c_int, [c_vp, c_int, c_int, c_vp, c_vp, c_vp, c_int, c_int, c_int, c_ll,
                                   c_int, c_vp, c_int, c_int, c_vp]),
}

_lock = threading.Lock()
_lib = None


def load() -> ctypes.CDLL:
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not LIB_PATH.exists():
            raise ExtensionMissingError(
                f"{LIB_PATH} not built; run `python -m paper_2307_08771_b200.build` "
                "(or __graft_entry__.build()). There is no CPU fallback.")
        try:
            lib = ctypes.CDLL(str(LIB_PATH))
        except OSError as exc:
            raise ExtensionMissingError(f"cannot load {LIB_PATH}: {exc}") from exc
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
        return lib


def check(rc: int) -> None:
    if rc != UB_OK:
        msg = load().ub_last_error().decode(errors="replace")
        raise UBError(rc, msg)


def call(name: str, *args) -> None:
    check(getattr(load(), name)(*args))


def index_faults() -> int:
    """Plan indices the permute kernel found outside the source tensor since the last
    call (synchronising; export time only)."""
    n = ctypes.c_ulonglong()
    check(load().ub_index_faults(ctypes.byref(n)))
    return int(n.value)


def num_sms_hint() -> int:
    """SM count of the current device (148 on B200) for host-side launch heuristics."""
    try:
        import torch

        if torch.cuda.is_available():
            return torch.cuda.get_device_properties(torch.cuda.current_device()).multi_processor_count
    except Exception:
        pass
    return 148


def launch_count() -> int:
    return int(load().ub_launch_count())


def reset_launch_count() -> None:
    load().ub_reset_launch_count()


def conv_stem_kpad(cin: int, kh: int, kw: int) -> int:
    return int(load().ub_conv_stem_kpad(cin, kh, kw))


def stem_s2d_geometry(N: int, H: int, W: int, k: int, pad: int) -> tuple[int, int, int]:
    """(Hs, Ws, bytes) of the space-to-depth stem input buffer."""
    hs, ws, nb = c_int(), c_int(), c_ll()
    check(load().ub_stem_s2d_geometry(N, H, W, k, pad, ctypes.byref(hs), ctypes.byref(ws), ctypes.byref(nb)))
    return hs.value, ws.value, nb.value


def conv_weight_layout(cin: int, coff: int, gather: bool, kh: int = 1, kw: int = 1) -> tuple[int, int]:
    lead, cpad = c_int(), c_int()
    check(load().ub_conv_weight_layout2(cin, coff, int(gather), kh, kw, ctypes.byref(lead), ctypes.byref(cpad)))
    return lead.value, cpad.value
