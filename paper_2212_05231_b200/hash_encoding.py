"""Multi-resolution hash-grid encoding on B200 (API of `hashsdf/hash_encoding.py`).

Tables live in device memory as (L, T, 2) fp32; every function here takes and
returns torch CUDA tensors (numpy inputs are uploaded).  The gathers/scatters run
in libns2b (`ns2b_interp_full`, `ns2b_scatter_first/second`); the fused training
step does not use these array-level entry points at all (it recomputes corner
records inside the field kernels), but they keep the reference's module API and
its kernel-level seam usable from Python.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _lib

DEFAULT_AABB = ((-1.0, -1.0, -1.0), (1.0, 1.0, 1.0))
PRIMES = (1, 2654435761, 805459861)  # _kernels.py:15-17


def level_resolutions(num_levels, min_resolution, max_resolution):
    """round(min * b**i), ends pinned (`hash_encoding.py:31-45`)."""
    if num_levels < 2:
        raise ValueError("need at least 2 levels")
    if not min_resolution < max_resolution:
        raise ValueError("min_resolution must be below max_resolution")
    growth = np.exp((np.log(max_resolution) - np.log(min_resolution)) / (num_levels - 1))
    res = [int(round(min_resolution * growth**i)) for i in range(num_levels)]
    res[0], res[-1] = int(min_resolution), int(max_resolution)
    return res


class MultiResHashGrid:
    """L levels of (T, 2) fp32 tables on the GPU (`hash_encoding.py:48-109`).

    ``tables`` is a CUDA tensor; when the grid belongs to SdfFieldParams it is a view
    into the flat parameter buffer.  Initialisation draws from the numpy generator
    exactly like the reference (so seeded runs match it) and uploads once.
    """

    def __init__(self, num_levels=14, min_resolution=16, max_resolution=2048,
                 features_per_level=2, table_size=2**19, aabb=DEFAULT_AABB, dtype=np.float32,
                 rng=None, tables=None):
        if int(features_per_level) != 2:
            raise _lib.ShapeError("shape error: features_per_level must be 2")
        if np.dtype(dtype) != np.float32:
            raise NotImplementedError("device tables are fp32")
        self.num_levels = int(num_levels)
        self.features_per_level = 2
        self.table_size = int(table_size)
        self.resolutions = np.asarray(
            level_resolutions(num_levels, min_resolution, max_resolution), np.int64)
        lo = np.asarray(aabb[0], np.float64)
        hi = np.asarray(aabb[1], np.float64)
        if not np.all(hi > lo):
            raise ValueError("aabb must have positive extent on each axis")
        self.aabb_min, self.aabb_extent = lo, hi - lo
        self.dtype = np.dtype(np.float32)
        shape = (self.num_levels, self.table_size, 2)
        if tables is not None:
            self.tables = tables
        else:
            dev = _lib.device()
            if rng is None:
                self.tables = torch.zeros(shape, dtype=torch.float32, device=dev)
            else:
                host = rng.uniform(-1e-4, 1e-4, size=shape).astype(np.float32)
                self.tables = torch.from_numpy(host).to(dev)
        self._res_dev = None

    @property
    def encoding_dim(self):
        return 3 + self.num_levels * self.features_per_level

    def level_is_dense(self, level):
        n = int(self.resolutions[level])
        return (n + 1) ** 3 <= self.table_size

    def feature_slice(self, level):
        return slice(3 + 2 * level, 3 + 2 * (level + 1))

    def normalize(self, x):
        """fp32 (x - lo)/extent clipped to [0,1] (`hash_encoding.py:102-106`)."""
        x = as_device(x, torch.float32)
        lo = torch.tensor(self.aabb_min.astype(np.float32), device=x.device)
        ext = torch.tensor(self.aabb_extent.astype(np.float32), device=x.device)
        return ((x - lo) / ext).clamp_(0.0, 1.0)

    def zero_gradient(self):
        return torch.zeros_like(self.tables)

    def resolutions_device(self):
        if self._res_dev is None or self._res_dev.device != self.tables.device:
            self._res_dev = torch.from_numpy(self.resolutions).to(self.tables.device)
        return self._res_dev

    def inv_extent_f32(self):
        return (1.0 / self.aabb_extent).astype(np.float32)


@dataclass
class CornerRecords:
    """(P, L, 8) rows, weights and (P, L, 8, 3) weight gradients (device)."""

    indices: torch.Tensor
    weights: torch.Tensor
    weight_gradients: torch.Tensor
    active_levels: int


@dataclass
class EncodedPoint:
    e: torch.Tensor
    jacobian: torch.Tensor | None
    corner_records: CornerRecords | None


_NP = {torch.float32: np.float32, torch.float64: np.float64, torch.int64: np.int64,
       torch.int32: np.int32, torch.uint8: np.uint8}


def as_device(x, dtype):
    """Tensor on the current CUDA device with the given dtype (numpy is uploaded)."""
    if isinstance(x, torch.Tensor):
        t = x.to(device=_lib.device(), dtype=dtype)
    else:
        host = np.ascontiguousarray(np.asarray(x), dtype=_NP[dtype])
        t = torch.from_numpy(host).to(_lib.device())
    return t.contiguous()


def active_level_count(grid, max_level):
    """`hash_encoding.py:132-138`."""
    return int(np.clip(np.floor(max_level), 0, grid.num_levels))


def hash_index(cell, level, grid):
    """Host-side row of an integer vertex (`hash_encoding.py:141-160`), including the
    reference helper's 32-bit masking of each product."""
    c = [int(v) for v in np.asarray(cell, np.int64)]
    n = int(grid.resolutions[level])
    if min(c) < 0 or max(c) > n:
        raise ValueError("cell out of bounds")
    if grid.level_is_dense(level):
        return c[0] + (n + 1) * (c[1] + (n + 1) * c[2])
    h = 0
    for v, p in zip(c, PRIMES):
        h ^= (v * p) & 0xFFFFFFFF
    return h % grid.table_size


def _batch(x):
    if isinstance(x, torch.Tensor):
        return x[None, :] if x.dim() == 1 else x
    x = np.asarray(x)
    return x[None, :] if x.ndim == 1 else x


def encode(grid, x, max_level, need_jacobian=False):
    """`hash_encoding.py:170-201` on the GPU."""
    xb = as_device(_batch(x), torch.float32)
    if not bool(torch.isfinite(xb).all()):
        raise ValueError("invalid position")
    xn = grid.normalize(xb)
    na = active_level_count(grid, max_level)
    npts = xb.shape[0]
    L, T = grid.num_levels, grid.table_size
    st = _lib.stream_ptr()
    feats = torch.empty((npts, 2 * L), dtype=torch.float32, device=xb.device)
    if not need_jacobian:
        _lib.call("ns2b_interp_features", _lib.ptr(xn), npts, _lib.ptr(grid.tables), L, T, 2,
                  _lib.ptr(grid.resolutions_device()), na, _lib.ptr(feats), st)
        return EncodedPoint(torch.cat([xb, feats], dim=1), None, None)
    inv = torch.from_numpy(grid.inv_extent_f32()).to(xb.device)
    jf = torch.empty((npts, 2 * L, 3), dtype=torch.float32, device=xb.device)
    cidx = torch.empty((npts, L, 8), dtype=torch.int64, device=xb.device)
    cw = torch.empty((npts, L, 8), dtype=torch.float32, device=xb.device)
    cdw = torch.empty((npts, L, 8, 3), dtype=torch.float32, device=xb.device)
    _lib.call("ns2b_interp_full", _lib.ptr(xn), npts, _lib.ptr(grid.tables), L, T, 2,
              _lib.ptr(grid.resolutions_device()), na, _lib.ptr(inv), _lib.ptr(feats),
              _lib.ptr(jf), _lib.ptr(cidx), _lib.ptr(cw), _lib.ptr(cdw), st)
    jac = torch.zeros((npts, grid.encoding_dim, 3), dtype=torch.float32, device=xb.device)
    jac[:, 0, 0] = 1.0
    jac[:, 1, 1] = 1.0
    jac[:, 2, 2] = 1.0
    jac[:, 3:, :] = jf
    return EncodedPoint(torch.cat([xb, feats], dim=1), jac, CornerRecords(cidx, cw, cdw, na))


def encode_features_only(grid, x, max_level):
    """`hash_encoding.py:204-211`."""
    return encode(grid, x, max_level, need_jacobian=False).e[:, 3:]


def encode_jacobian(grid, x, max_level):
    return encode(grid, x, max_level, need_jacobian=True).jacobian


def backward_first(grid, point, dl_de, out=None):
    """`hash_encoding.py:224-237`: out += scatter of the feature cotangent."""
    rec = point.corner_records
    if rec is None:
        raise ValueError("stale sample: encode was called without caches")
    out = grid.zero_gradient() if out is None else out
    d = as_device(dl_de, torch.float32)[:, 3:].contiguous()
    _lib.call("ns2b_scatter_first", _lib.ptr(out), grid.num_levels, grid.table_size, 2,
              _lib.ptr(rec.indices), _lib.ptr(rec.weights), _lib.ptr(d), rec.indices.shape[0],
              rec.active_levels, _lib.stream_ptr())
    return out


def backward_second(grid, point, u, out=None):
    """`hash_encoding.py:257-272`: out += Eq. 9 scatter of the jacobian cotangent."""
    rec = point.corner_records
    if rec is None:
        raise ValueError("stale sample: encode was called without caches")
    out = grid.zero_gradient() if out is None else out
    uu = as_device(u, torch.float32)[:, 3:, :].contiguous()
    _lib.call("ns2b_scatter_second", _lib.ptr(out), grid.num_levels, grid.table_size, 2,
              _lib.ptr(rec.indices), _lib.ptr(rec.weight_gradients), _lib.ptr(uu),
              rec.indices.shape[0], rec.active_levels, _lib.stream_ptr())
    return out


def hessian_contract(grid, x, max_level, coeff):
    """`hash_encoding.py:240-254` on the GPU: (P, 3, 3) fp32, the interpolation
    curvature sum_a coeff[p, a] d2 e_a / dx dx (coeff (P, L*F), feature rows only)."""
    xb = as_device(_batch(x), torch.float32)
    xn = grid.normalize(xb)
    npts = xb.shape[0]
    L = grid.num_levels
    cf = as_device(coeff, torch.float32).reshape(npts, 2 * L).contiguous()
    inv = torch.from_numpy(grid.inv_extent_f32()).to(xb.device)
    out = torch.empty((npts, 3, 3), dtype=torch.float32, device=xb.device)
    _lib.call("ns2b_hessian_contract", _lib.ptr(xn), npts, _lib.ptr(grid.tables), L, grid.table_size,
              2, _lib.ptr(grid.resolutions_device()), active_level_count(grid, max_level),
              _lib.ptr(inv), _lib.ptr(cf), _lib.ptr(out), _lib.stream_ptr())
    return out
