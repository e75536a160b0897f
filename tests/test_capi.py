"""C-ABI surface checks that need no GPU: the library loads and exports every
symbol include/ns2b.h declares, and the Python binding covers all of them."""

from __future__ import annotations

import ctypes
import re
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
HEADER = ROOT / "include" / "ns2b.h"
LIB = ROOT / "paper_2212_05231_b200" / "libns2b.so"


def header_symbols():
    txt = HEADER.read_text()
    return sorted(set(re.findall(r"NS2B_API[^;(]*?\b(ns2b_\w+)\s*\(", txt)))


@pytest.fixture(scope="module")
def lib():
    if not LIB.exists():
        from paper_2212_05231_b200 import build

        build.build()
    return ctypes.CDLL(str(LIB))


def test_header_declares_entry_points():
    syms = header_symbols()
    assert len(syms) >= 20
    for s in ("ns2b_march_count", "ns2b_field_forward", "ns2b_field_backward", "ns2b_composite",
              "ns2b_adam_multi", "ns2b_interp_full", "ns2b_scatter_second"):
        assert s in syms


def test_library_exports_every_header_symbol(lib):
    for s in header_symbols():
        assert hasattr(lib, s), f"{s} declared in ns2b.h but not exported"


def test_abi_version_and_error_plumbing(lib):
    lib.ns2b_abi_version.restype = ctypes.c_int
    assert lib.ns2b_abi_version() == 1
    lib.ns2b_last_error.restype = ctypes.c_char_p
    assert isinstance(lib.ns2b_last_error(), bytes)


def test_binding_covers_header():
    from paper_2212_05231_b200 import _lib

    assert set(header_symbols()) == set(_lib.exported_symbols())


def test_invalid_args_fail_loudly_without_touching_device(lib):
    """Argument validation happens before any CUDA call: a bad level count returns
    NS2B_EINVAL with a 'shape error' message."""
    from paper_2212_05231_b200 import _lib

    f = _lib.FieldT()
    f.num_levels = 17
    f.features_per_level = 2
    f.hidden_width = 64
    fn = lib.ns2b_field_sdf
    fn.argtypes = [ctypes.POINTER(_lib.FieldT), ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p,
                   ctypes.c_void_p]
    rc = fn(ctypes.byref(f), None, 0, None, None)
    assert rc == -1
    lib.ns2b_last_error.restype = ctypes.c_char_p
    assert lib.ns2b_last_error().startswith(b"shape error")


def test_product_requires_cuda_no_fallback():
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2212_05231_b200 import _lib

    with pytest.raises(RuntimeError, match="no CPU fallback"):
        _lib.device()
