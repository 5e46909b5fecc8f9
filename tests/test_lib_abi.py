"""The C-ABI library loads (no GPU needed) and exports every entry point that
include/upscale_b200.h declares, with the ctypes binding covering all of them."""

import re
import subprocess
from pathlib import Path

import pytest

from paper_2307_08771_b200 import _lib

ROOT = Path(__file__).resolve().parents[1]
HEADER = ROOT / "include" / "upscale_b200.h"


def declared_functions():
    text = re.sub(r"/\*.*?\*/", "", HEADER.read_text(), flags=re.S)
    return sorted(set(re.findall(r"\b(ub_[a-z0-9_]+)\s*\(", text)))


@pytest.fixture(scope="module")
def lib():
    if not _lib.LIB_PATH.exists():
        from paper_2307_08771_b200 import build

        build.build()
    return _lib.load()


def test_header_declares_the_hot_path():
    fns = declared_functions()
    for name in ("ub_permute_weights", "ub_permute_vector", "ub_channel_gather", "ub_conv_fwd",
                 "ub_conv_weight_layout", "ub_conv_stem_kpad", "ub_last_error"):
        assert name in fns


def test_library_exports_every_declared_symbol(lib):
    out = subprocess.run(["nm", "-D", "--defined-only", str(_lib.LIB_PATH)], capture_output=True, text=True).stdout
    exported = set(re.findall(r"\bT (ub_[a-z0-9_]+)$", out, flags=re.M))
    missing = [f for f in declared_functions() if f not in exported]
    assert not missing, missing
    assert set(_lib.SIGNATURES) == set(declared_functions())


def test_abi_version_and_host_only_helpers(lib):
    assert lib.ub_abi_version() == 7
    assert _lib.conv_weight_layout(100, 13, False) == (5, 128)   # misaligned slice: lead 5, 105 -> 128
    assert _lib.conv_weight_layout(12, 0, False) == (0, 16)      # BK 16
    assert _lib.conv_weight_layout(32, 0, False) == (0, 32)      # BK 32
    assert _lib.conv_weight_layout(128, 7, True) == (0, 128)     # gather: no lead
    assert _lib.conv_weight_layout(16, 0, False, 3, 3) == (0, 16)   # packed taps: 4 per K-block
    assert _lib.conv_weight_layout(24, 5, False, 3, 3) == (5, 32)   # 29 -> 32: 2 taps per K-block
    assert _lib.conv_weight_layout(2, 0, False, 7, 7) == (0, 8)
    assert _lib.conv_weight_layout(48, 0, False, 3, 3) == (0, 64)   # too wide to pack
    assert _lib.conv_weight_layout(16, 0, True, 3, 3) == (0, 64)    # gather reads never pack
    assert _lib.conv_stem_kpad(2, 7, 7) == 128
    with pytest.raises(_lib.UBError):
        _lib.conv_weight_layout(0, 0, False)


def test_sm100a_code_is_in_the_library(lib):
    sass = subprocess.run(["cuobjdump", "-sass", str(_lib.LIB_PATH)], capture_output=True, text=True).stdout
    if not sass:
        pytest.skip("cuobjdump unavailable")
    assert "UTCHMMA" in sass       # tcgen05.mma
    assert "UTMASTG" in sass       # TMA bulk tensor store
    assert "LDGSTS" in sass        # cp.async producers
    assert "LDTM" in sass and "STTM" in sass  # tcgen05.ld / tcgen05.st


def test_argument_errors_fail_loudly_without_touching_the_device(lib):
    """Bad arguments come back as negative status + ub_last_error text (raised as UBError by
    the binding) before any CUDA call, so this runs without a GPU."""
    import ctypes

    with pytest.raises(_lib.UBError, match="ub_avgpool_gather: bad arguments"):
        _lib.call("ub_avgpool_gather", ctypes.c_void_p(16), 2, 49, 64, 64, 0, None, 8,
                  ctypes.c_void_p(16), 8, 0, None)
    with pytest.raises(_lib.UBError, match="multiples of 8"):
        _lib.call("ub_avgpool_gather", ctypes.c_void_p(16), 2, 49, 60, 64, 0, ctypes.c_void_p(16), 8,
                  ctypes.c_void_p(16), 8, 0, None)
    with pytest.raises(_lib.UBError, match="ub_avgpool_global"):
        _lib.call("ub_avgpool_global", None, 2, 49, 64, 64, 0, ctypes.c_void_p(16), 64, 0, None)
    assert lib.ub_last_error()
