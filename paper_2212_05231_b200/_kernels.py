"""Drop-in for `hashsdf._kernels` (`_kernels.py:40-218`, incl. hessian_contract :159-206) backed by libns2b on the GPU.

Same signatures and semantics: numpy arrays in; `interp_*` return new numpy arrays,
`scatter_*` and `adam_step` mutate their first argument in place.  Each call copies
its inputs to the device, runs the sm_100a kernel, and copies results back, so an
unmodified numpy training loop can run on B200 kernels by monkey-patching this
module in (tests/test_gpu_parity.py does exactly that with the oracle's loop).
"""

from __future__ import annotations

import numpy as np
import torch

from . import _lib

PRIME_X = np.uint32(1)
PRIME_Y = np.uint32(2654435761)
PRIME_Z = np.uint32(805459861)


def _dev(a, dtype):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=dtype)).to(_lib.device())


def interp_features(xn, tables, resolutions, n_active):
    xd = _dev(xn, np.float32)
    td = _dev(tables, np.float32)
    rd = _dev(resolutions, np.int64)
    nlev, tsize, nfeat = tables.shape
    out = torch.empty((xd.shape[0], nlev * nfeat), dtype=torch.float32, device=xd.device)
    _lib.call("ns2b_interp_features", _lib.ptr(xd), xd.shape[0], _lib.ptr(td), nlev, tsize, nfeat,
              _lib.ptr(rd), int(n_active), _lib.ptr(out), _lib.stream_ptr())
    return out.cpu().numpy()


def interp_full(xn, tables, resolutions, n_active, inv_extent):
    xd = _dev(xn, np.float32)
    td = _dev(tables, np.float32)
    rd = _dev(resolutions, np.int64)
    inv = _dev(inv_extent, np.float32)
    P = xd.shape[0]
    nlev, tsize, nfeat = tables.shape
    kw = dict(device=xd.device)
    feats = torch.empty((P, nlev * nfeat), dtype=torch.float32, **kw)
    jac = torch.empty((P, nlev * nfeat, 3), dtype=torch.float32, **kw)
    cidx = torch.empty((P, nlev, 8), dtype=torch.int64, **kw)
    cw = torch.empty((P, nlev, 8), dtype=torch.float32, **kw)
    cdw = torch.empty((P, nlev, 8, 3), dtype=torch.float32, **kw)
    _lib.call("ns2b_interp_full", _lib.ptr(xd), P, _lib.ptr(td), nlev, tsize, nfeat, _lib.ptr(rd),
              int(n_active), _lib.ptr(inv), _lib.ptr(feats), _lib.ptr(jac), _lib.ptr(cidx),
              _lib.ptr(cw), _lib.ptr(cdw), _lib.stream_ptr())
    return tuple(t.cpu().numpy() for t in (feats, jac, cidx, cw, cdw))


def hessian_contract(xn, tables, resolutions, n_active, inv_extent, coeff):
    xd = _dev(xn, np.float32)
    td = _dev(tables, np.float32)
    rd = _dev(resolutions, np.int64)
    inv = _dev(inv_extent, np.float32)
    cf = _dev(coeff, np.float32)
    nlev, tsize, nfeat = tables.shape
    out = torch.empty((xd.shape[0], 3, 3), dtype=torch.float32, device=xd.device)
    _lib.call("ns2b_hessian_contract", _lib.ptr(xd), xd.shape[0], _lib.ptr(td), nlev, tsize, nfeat,
              _lib.ptr(rd), int(n_active), _lib.ptr(inv), _lib.ptr(cf), _lib.ptr(out),
              _lib.stream_ptr())
    return out.cpu().numpy()


def _scatter(name, grad, cidx, w, d, n_active):
    g = _dev(grad, np.float32)
    nlev, tsize, nfeat = grad.shape
    # keep every device temporary referenced until the kernel has been enqueued and
    # the result copied back (a dropped tensor's block can be reused by the next
    # allocation on the stream)
    ci, wd, dd = _dev(cidx, np.int64), _dev(w, np.float32), _dev(d, np.float32)
    _lib.call(name, _lib.ptr(g), nlev, tsize, nfeat, _lib.ptr(ci), _lib.ptr(wd), _lib.ptr(dd),
              cidx.shape[0], int(n_active), _lib.stream_ptr())
    grad[...] = g.cpu().numpy()


def scatter_first(grad, cidx, cw, dl_dfeat, n_active):
    _scatter("ns2b_scatter_first", grad, cidx, cw, dl_dfeat, n_active)


def scatter_second(grad, cidx, cdw, u, n_active):
    _scatter("ns2b_scatter_second", grad, cidx, cdw, u, n_active)


def adam_step(param, grad, m, v, t, lr, beta1, beta2, eps):
    dt = np.float64 if param.dtype == np.float64 else np.float32
    fn = "ns2b_adam_step_f64" if dt == np.float64 else "ns2b_adam_step_f32"
    pd, gd, md, vd = (_dev(a, dt) for a in (param, grad, m, v))
    _lib.call(fn, _lib.ptr(pd), _lib.ptr(gd), _lib.ptr(md), _lib.ptr(vd), param.shape[0], int(t),
              float(lr), float(beta1), float(beta2), float(eps), _lib.stream_ptr())
    param[...] = pd.cpu().numpy()
    m[...] = md.cpu().numpy()
    v[...] = vd.cpu().numpy()
