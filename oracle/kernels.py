"""ctypes front for oracle/csrc/hashgrid_oracle.c (TEST INFRASTRUCTURE ONLY).

Same call signatures as the reference's numba kernels (`hashsdf/_kernels.py:40-218`):
gathers return new arrays, scatters/Adam mutate their first argument in place.
"""

from __future__ import annotations

import ctypes
import os
import subprocess
from pathlib import Path

import numpy as np

_HERE = Path(__file__).resolve().parent
_SRC = _HERE / "csrc" / "hashgrid_oracle.c"
_LIB_PATH = _HERE / "_build" / "libns2b_oracle.so"
_lib = None

_P = ctypes.c_void_p
_I = ctypes.c_int64
_D = ctypes.c_double


def build(force: bool = False) -> Path:
    """Compile the C restatement with gcc (no FMA contraction, OpenMP gathers)."""
    if _LIB_PATH.exists() and not force and _LIB_PATH.stat().st_mtime >= _SRC.stat().st_mtime:
        return _LIB_PATH
    _LIB_PATH.parent.mkdir(parents=True, exist_ok=True)
    tmp = _LIB_PATH.with_suffix(f".{os.getpid()}.tmp.so")
    cmd = ["gcc", "-O2", "-fPIC", "-shared", "-ffp-contract=off", "-fno-fast-math",
           "-fopenmp", "-o", str(tmp), str(_SRC), "-lm"]
    subprocess.run(cmd, check=True)
    os.replace(tmp, _LIB_PATH)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        _lib = ctypes.CDLL(str(build()))
        _lib.orc_interp_features.argtypes = [_P, _I, _P, _I, _I, _I, _P, _I, _P, ctypes.c_int]
        _lib.orc_interp_full.argtypes = [_P, _I, _P, _I, _I, _I, _P, _I, _P, _P, _P, _P, _P, _P,
                                         ctypes.c_int]
        _lib.orc_scatter_first.argtypes = [_P, _I, _I, _I, _P, _P, _P, _I, _I]
        _lib.orc_scatter_second.argtypes = [_P, _I, _I, _I, _P, _P, _P, _I, _I]
        _lib.orc_hessian_contract.argtypes = [_P, _I, _P, _I, _I, _I, _P, _I, _P, _P, _P,
                                              ctypes.c_int]
        _lib.orc_adam_step_f32.argtypes = [_P, _P, _P, _P, _I, _I, _D, _D, _D, _D]
        _lib.orc_adam_step_f64.argtypes = [_P, _P, _P, _P, _I, _I, _D, _D, _D, _D]
    return _lib


NUM_THREADS = int(os.environ.get("NS2B_ORACLE_THREADS", "1"))


def _ptr(a):
    return a.ctypes.data


def _c(a, dtype):
    return np.ascontiguousarray(a, dtype=dtype)


def interp_features(xn, tables, resolutions, n_active):
    """`_kernels.interp_features` (`hashsdf/_kernels.py:40-64`)."""
    xn = _c(xn, np.float32)
    tables = _c(tables, np.float32)
    res = _c(resolutions, np.int64)
    nlev, tsize, nfeat = tables.shape
    out = np.zeros((xn.shape[0], nlev * nfeat), np.float32)
    lib().orc_interp_features(_ptr(xn), xn.shape[0], _ptr(tables), nlev, tsize, nfeat,
                              _ptr(res), int(n_active), _ptr(out), NUM_THREADS)
    return out


def interp_full(xn, tables, resolutions, n_active, inv_extent):
    """`_kernels.interp_full` (`hashsdf/_kernels.py:67-119`)."""
    xn = _c(xn, np.float32)
    tables = _c(tables, np.float32)
    res = _c(resolutions, np.int64)
    inv = _c(inv_extent, np.float32)
    npts = xn.shape[0]
    nlev, tsize, nfeat = tables.shape
    feats = np.zeros((npts, nlev * nfeat), np.float32)
    jac = np.zeros((npts, nlev * nfeat, 3), np.float32)
    cidx = np.zeros((npts, nlev, 8), np.int64)
    cw = np.zeros((npts, nlev, 8), np.float32)
    cdw = np.zeros((npts, nlev, 8, 3), np.float32)
    lib().orc_interp_full(_ptr(xn), npts, _ptr(tables), nlev, tsize, nfeat, _ptr(res),
                          int(n_active), _ptr(inv), _ptr(feats), _ptr(jac), _ptr(cidx),
                          _ptr(cw), _ptr(cdw), NUM_THREADS)
    return feats, jac, cidx, cw, cdw


def hessian_contract(xn, tables, resolutions, n_active, inv_extent, coeff):
    """`_kernels.hessian_contract` (`hashsdf/_kernels.py:159-206`): (P, 3, 3)."""
    xn = _c(xn, np.float32)
    tables = _c(tables, np.float32)
    res = _c(resolutions, np.int64)
    inv = _c(inv_extent, np.float32)
    coeff = _c(coeff, np.float32)
    nlev, tsize, nfeat = tables.shape
    if coeff.shape != (xn.shape[0], nlev * nfeat):
        raise ValueError("coeff must be (P, L*F)")
    out = np.zeros((xn.shape[0], 3, 3), np.float32)
    lib().orc_hessian_contract(_ptr(xn), xn.shape[0], _ptr(tables), nlev, tsize, nfeat, _ptr(res),
                               int(n_active), _ptr(inv), _ptr(coeff), _ptr(out), NUM_THREADS)
    return out


def _check_inplace(a, dtype):
    if a.dtype != dtype or not a.flags.c_contiguous:
        raise TypeError("in-place buffer must be a C-contiguous %s array" % np.dtype(dtype).name)


def scatter_first(grad, cidx, cw, dl_dfeat, n_active):
    """`_kernels.scatter_first` (`hashsdf/_kernels.py:122-133`), in place on grad."""
    _check_inplace(grad, np.float32)
    cidx = _c(cidx, np.int64)
    cw = _c(cw, np.float32)
    d = _c(dl_dfeat, np.float32)
    nlev, tsize, nfeat = grad.shape
    lib().orc_scatter_first(_ptr(grad), nlev, tsize, nfeat, _ptr(cidx), _ptr(cw), _ptr(d),
                            cidx.shape[0], int(n_active))


def scatter_second(grad, cidx, cdw, u, n_active):
    """`_kernels.scatter_second` (`hashsdf/_kernels.py:136-156`), in place on grad."""
    _check_inplace(grad, np.float32)
    cidx = _c(cidx, np.int64)
    cdw = _c(cdw, np.float32)
    u = _c(u, np.float32)
    nlev, tsize, nfeat = grad.shape
    lib().orc_scatter_second(_ptr(grad), nlev, tsize, nfeat, _ptr(cidx), _ptr(cdw), _ptr(u),
                             cidx.shape[0], int(n_active))


def adam_step(param, grad, m, v, t, lr, beta1, beta2, eps):
    """`_kernels.adam_step` (`hashsdf/_kernels.py:209-218`) on flat views, in place."""
    if param.dtype == np.float64:
        fn, dt = lib().orc_adam_step_f64, np.float64
    else:
        fn, dt = lib().orc_adam_step_f32, np.float32
    for a in (param, m, v):
        _check_inplace(a, dt)
    g = _c(grad, dt)
    fn(_ptr(param), _ptr(g), _ptr(m), _ptr(v), param.shape[0], int(t), float(lr), float(beta1),
       float(beta2), float(eps))
