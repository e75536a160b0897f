"""ctypes binding of libns2b.so (include/ns2b.h).

The library is loaded from the package directory (built in-tree by build.py).
There is no fallback: if the library or a CUDA device is missing, every product
entry point raises.  Status codes map to the reference's exception types
(`relu_mlp.ShapeError` / `ValueError` for bad shapes, RuntimeError for CUDA).
"""

from __future__ import annotations

import ctypes
import os
from pathlib import Path

import torch

_PKG = Path(__file__).resolve().parent
LIB_PATH = _PKG / "libns2b.so"

P = ctypes.c_void_p
I64 = ctypes.c_int64
I32 = ctypes.c_int32
F64 = ctypes.c_double
SZ = ctypes.c_size_t

NS2B_EINVAL = -1
NS2B_ECUDA = -2
NS2B_EUNSUPPORTED = -3
MAX_LEVELS = 16


class ShapeError(ValueError):
    """Mirrors `hashsdf.relu_mlp.ShapeError` (`relu_mlp.py:29-30`)."""


class FieldT(ctypes.Structure):
    _fields_ = [
        ("num_levels", I32), ("table_size", I32), ("features_per_level", I32), ("n_active", I32),
        ("resolutions", I32 * MAX_LEVELS),
        ("aabb_min", ctypes.c_float * 3), ("aabb_extent", ctypes.c_float * 3),
        ("inv_extent", ctypes.c_float * 3), ("hidden_width", I32),
        ("tables", P), ("sdf_w", P), ("color_w", P),
    ]


class OccT(ctypes.Structure):
    _fields_ = [("resolution", I32), ("lo", F64 * 3), ("hi", F64 * 3), ("step_size", F64),
                ("bits", P)]


_SIGS = {
    "ns2b_last_error": (ctypes.c_char_p, []),
    "ns2b_abi_version": (ctypes.c_int, []),
    "ns2b_launch_count": (ctypes.c_uint64, []),
    "ns2b_interp_features": (ctypes.c_int, [P, I64, P, I64, I64, I64, P, I64, P, P]),
    "ns2b_interp_full": (ctypes.c_int, [P, I64, P, I64, I64, I64, P, I64, P, P, P, P, P, P, P]),
    "ns2b_hessian_contract": (ctypes.c_int, [P, I64, P, I64, I64, I64, P, I64, P, P, P, P]),
    "ns2b_scatter_first": (ctypes.c_int, [P, I64, I64, I64, P, P, P, I64, I64, P]),
    "ns2b_scatter_second": (ctypes.c_int, [P, I64, I64, I64, P, P, P, I64, I64, P]),
    "ns2b_adam_step_f32": (ctypes.c_int, [P, P, P, P, I64, I64, F64, F64, F64, F64, P]),
    "ns2b_adam_step_f64": (ctypes.c_int, [P, P, P, P, I64, I64, F64, F64, F64, F64, P]),
    "ns2b_march_count": (ctypes.c_int, [P, P, I64, ctypes.POINTER(OccT), P, P]),
    "ns2b_scan_offsets": (ctypes.c_int, [P, I64, P, P, ctypes.POINTER(SZ), P]),
    "ns2b_march_fill": (ctypes.c_int, [P, P, I64, ctypes.POINTER(OccT), P, P, P, P, P, P]),
    "ns2b_march_count_masked": (ctypes.c_int, [P, P, I64, ctypes.POINTER(OccT), P, P, P]),
    "ns2b_march_fill_masked": (ctypes.c_int, [P, P, I64, ctypes.POINTER(OccT), P, P, P, P, P, P, P]),
    "ns2b_field_forward": (ctypes.c_int, [ctypes.POINTER(FieldT), P, P, P, P, I64, P, P, P, P, P,
                                          P, P]),
    "ns2b_field_workspace_bytes": (ctypes.c_int, [I64, ctypes.POINTER(SZ)]),
    "ns2b_field_gather": (ctypes.c_int, [ctypes.POINTER(FieldT), P, P, P, P, I64, P, P]),
    "ns2b_field_mlp_forward": (ctypes.c_int, [ctypes.POINTER(FieldT), P, P, P, P, I64, P, P, P, P, P,
                                              P, P]),
    "ns2b_field_mlp_forward_eik": (ctypes.c_int, [ctypes.POINTER(FieldT), P, P, P, P, I64, P, P, P, P, P,
                                                  F64, P, P, P]),
    "ns2b_field_forward_fused_eik": (ctypes.c_int, [ctypes.POINTER(FieldT), P, P, P, P, I64, P, P, P, P, P,
                                                    F64, P, P, P]),
    "ns2b_field_mlp_backward": (ctypes.c_int, [ctypes.POINTER(FieldT), P, P, P, P, I64, P, P, P, F64,
                                               P, P, P, P, P]),
    "ns2b_field_scatter": (ctypes.c_int, [ctypes.POINTER(FieldT), P, P, I64, P, P, P]),
    "ns2b_field_backward_inputs": (ctypes.c_int, [ctypes.POINTER(FieldT), P, I64, P, P, P, F64, P, P, P, P,
                                                  P, P, P]),
    "ns2b_occupancy_from_sdf": (ctypes.c_int, [P, I64, F64, F64, F64, P, P, P]),
    "ns2b_field_sdf": (ctypes.c_int, [ctypes.POINTER(FieldT), P, I64, P, P]),
    "ns2b_occupancy_update": (ctypes.c_int, [ctypes.POINTER(FieldT), ctypes.POINTER(OccT), F64,
                                             F64, P, P, P]),
    "ns2b_composite": (ctypes.c_int, [P, I64, P, P, F64, P, F64, F64, P, P, P, P, P, P, P, P, P]),
    "ns2b_composite_backward": (ctypes.c_int, [P, I64, P, P, F64, P, P, P, P, P, P, P, P]),
    "ns2b_field_backward": (ctypes.c_int, [ctypes.POINTER(FieldT), P, P, P, P, I64, P, P, P, F64,
                                           P, P, P, P, P, P]),
    "ns2b_check_finite": (ctypes.c_int, [P, P, P, I32, P, P]),
    "ns2b_adam_multi": (ctypes.c_int, [P, P, P, P, P, P, P, P, I32, F64, F64, F64, P, P]),
    "ns2b_adam_scalar_f64": (ctypes.c_int, [P, P, F64, P, P, I64, F64, F64, F64, F64, P, P, I32,
                                            P]),
    "ns2b_bench_l2_read": (ctypes.c_int, [P, I64, I32, P, P]),
    "ns2b_bench_red": (ctypes.c_int, [P, I64, I64, ctypes.c_uint32, P]),
    "ns2b_bench_gather": (ctypes.c_int, [P, I64, I64, ctypes.c_uint32, P, P]),
    "ns2b_bench_red_coalesced": (ctypes.c_int, [P, I64, I64, ctypes.c_uint32, P]),
    "ns2b_bench_umma": (ctypes.c_int, [I32, I32, I32, P, P]),
    "ns2b_rays_from_picks": (ctypes.c_int, [P, I64, I64, P, P, P, I32, I32, P, P, P, P, P, P]),
    "ns2b_selftest_umma": (ctypes.c_int, [P, P, P, I32, P]),
}

_lib = None


def lib():
    """Load libns2b.so (raises if it was not built or there is no CUDA device)."""
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise RuntimeError(f"libns2b.so not built ({LIB_PATH}); run "
                               "`python -m paper_2212_05231_b200.build` (no CPU fallback)")
        lb = ctypes.CDLL(str(LIB_PATH))
        for name, (res, args) in _SIGS.items():
            fn = getattr(lb, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lb
    return _lib


def exported_symbols():
    return list(_SIGS)


def require_cuda():
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2212_05231_b200 needs a CUDA device (sm_100a); "
                           "there is no CPU fallback")


def check(rc: int, what: str = ""):
    if rc == 0:
        return
    msg = lib().ns2b_last_error().decode(errors="replace")
    if rc == NS2B_EINVAL:
        if msg.startswith("shape error"):
            raise ShapeError(msg)
        raise ValueError(msg)
    if rc == NS2B_EUNSUPPORTED:
        raise NotImplementedError(msg)
    raise RuntimeError(f"{what}: {msg}")


def call(name: str, *args):
    check(getattr(lib(), name)(*args), name)


def ptr(t):
    """Device pointer of a torch tensor (or None -> NULL)."""
    if t is None:
        return None
    return ctypes.c_void_p(t.data_ptr())


def stream_ptr(stream=None):
    s = stream if stream is not None else torch.cuda.current_stream()
    return ctypes.c_void_p(s.cuda_stream)


def field_workspace(capacity, device, cache=None):
    """Device workspace tensor for `capacity` samples (reused from `cache` if large enough)."""
    n = ctypes.c_size_t(0)
    call("ns2b_field_workspace_bytes", int(max(capacity, 1)), ctypes.byref(n))
    if cache is not None and cache.numel() >= n.value:
        return cache
    return torch.empty(int(n.value), dtype=torch.uint8, device=device)


def launch_count() -> int:
    return int(lib().ns2b_launch_count())


def i64_array(vals):
    return (I64 * len(vals))(*[int(v) for v in vals])


def f64_array(vals):
    return (F64 * len(vals))(*[float(v) for v in vals])


def device():
    require_cuda()
    return torch.device("cuda", torch.cuda.current_device())


def env_flag(name, default="0"):
    return os.environ.get(name, default) not in ("", "0", "false", "False")
