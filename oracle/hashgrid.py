"""Oracle: multi-resolution hash grid (TEST INFRASTRUCTURE ONLY).

Restates `hashsdf/hash_encoding.py`.  The per-point loops live in
oracle/csrc/hashgrid_oracle.c (restating `hashsdf/_kernels.py`).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import kernels

DEFAULT_AABB = ((-1.0, -1.0, -1.0), (1.0, 1.0, 1.0))
HASH_PRIMES = (1, 2654435761, 805459861)  # _kernels.py:15-17


def level_resolutions(num_levels, min_resolution, max_resolution):
    """Geometric level resolutions, ends pinned (`hash_encoding.py:31-45`)."""
    if num_levels < 2:
        raise ValueError("need at least 2 levels")
    if not min_resolution < max_resolution:
        raise ValueError("min_resolution must be below max_resolution")
    b = np.exp((np.log(max_resolution) - np.log(min_resolution)) / (num_levels - 1))
    out = [int(round(min_resolution * b**i)) for i in range(num_levels)]
    out[0], out[-1] = int(min_resolution), int(max_resolution)
    return out


class HashGrid:
    """Tables (L, T, F) over an aabb (`hash_encoding.py:48-109`)."""

    def __init__(self, num_levels=14, min_resolution=16, max_resolution=2048,
                 features_per_level=2, table_size=2**19, aabb=DEFAULT_AABB,
                 dtype=np.float32, rng=None):
        self.num_levels = int(num_levels)
        self.features_per_level = int(features_per_level)
        self.table_size = int(table_size)
        self.resolutions = np.asarray(
            level_resolutions(num_levels, min_resolution, max_resolution), np.int64)
        lo = np.asarray(aabb[0], np.float64)
        hi = np.asarray(aabb[1], np.float64)
        if not np.all(hi > lo):
            raise ValueError("aabb must have positive extent on each axis")
        self.aabb_min, self.aabb_extent = lo, hi - lo
        self.dtype = np.dtype(dtype)
        shape = (self.num_levels, self.table_size, self.features_per_level)
        if rng is None:
            self.tables = np.zeros(shape, self.dtype)
        else:
            self.tables = rng.uniform(-1e-4, 1e-4, size=shape).astype(self.dtype)

    @property
    def encoding_dim(self):
        return 3 + self.num_levels * self.features_per_level

    def level_is_dense(self, level):
        n = int(self.resolutions[level])
        return (n + 1) ** 3 <= self.table_size

    def normalize(self, x):
        """fp32 (x - lo) / extent clipped to [0,1] (`hash_encoding.py:102-106`)."""
        x = np.asarray(x, self.dtype)
        lo = self.aabb_min.astype(self.dtype)
        ext = self.aabb_extent.astype(self.dtype)
        return np.clip((x - lo) / ext, 0.0, 1.0)

    def zero_gradient(self):
        return np.zeros_like(self.tables)


@dataclass
class Corners:
    """Per (point, level, corner) rows / weights / weight gradients
    (`hash_encoding.py:112-120`)."""

    indices: np.ndarray
    weights: np.ndarray
    weight_gradients: np.ndarray
    active_levels: int


@dataclass
class Encoded:
    e: np.ndarray
    jacobian: np.ndarray | None
    corner_records: Corners | None


def active_level_count(grid, max_level):
    """`hash_encoding.py:132-138`: floor(max_level) clipped to [0, L]."""
    return int(np.clip(np.floor(max_level), 0, grid.num_levels))


def hash_index(cell, level, grid):
    """Host-side row lookup (`hash_encoding.py:141-160`).  Note: this Python helper
    masks each product to 32 bits before the xor, unlike the kernel (which keeps
    64-bit products); both agree whenever T is a power of two."""
    c = [int(v) for v in np.asarray(cell, np.int64)]
    n = int(grid.resolutions[level])
    if min(c) < 0 or max(c) > n:
        raise ValueError("cell out of bounds")
    if grid.level_is_dense(level):
        return c[0] + (n + 1) * (c[1] + (n + 1) * c[2])
    m32 = 0xFFFFFFFF
    h = 0
    for v, prime in zip(c, HASH_PRIMES):
        h ^= (v * prime) & m32
    return h % grid.table_size


def _batch(x):
    x = np.asarray(x)
    return x[None, :] if x.ndim == 1 else x


def encode(grid, x, max_level, need_jacobian=False):
    """`hash_encoding.py:170-201`: e = [x, level features]; optional jacobian
    (rows 0..2 identity) and corner records."""
    xb = _batch(x)
    if not np.all(np.isfinite(xb)):
        raise ValueError("invalid position")
    xb = np.ascontiguousarray(xb, grid.dtype)
    xn = grid.normalize(xb)
    n_active = active_level_count(grid, max_level)
    if not need_jacobian:
        feats = kernels.interp_features(xn, grid.tables, grid.resolutions, n_active)
        return Encoded(np.concatenate([xb, feats], axis=1), None, None)
    inv_extent = np.ascontiguousarray(1.0 / grid.aabb_extent, grid.dtype)
    feats, jf, cidx, cw, cdw = kernels.interp_full(xn, grid.tables, grid.resolutions,
                                                   n_active, inv_extent)
    npts = xb.shape[0]
    jac = np.zeros((npts, grid.encoding_dim, 3), grid.dtype)
    jac[:, 0:3, :] = np.eye(3, dtype=grid.dtype)
    jac[:, 3:, :] = jf
    return Encoded(np.concatenate([xb, feats], axis=1), jac,
                   Corners(cidx, cw, cdw, n_active))


def encode_features_only(grid, x, max_level):
    """`hash_encoding.py:204-211`."""
    xb = np.ascontiguousarray(_batch(x), grid.dtype)
    return kernels.interp_features(grid.normalize(xb), grid.tables, grid.resolutions,
                                   active_level_count(grid, max_level))


def backward_first(grid, point, dl_de, out=None):
    """`hash_encoding.py:224-237`: scatter the feature slice of dL/de."""
    rec = point.corner_records
    if rec is None:
        raise ValueError("stale sample: encode was called without caches")
    out = grid.zero_gradient() if out is None else out
    kernels.scatter_first(out, rec.indices, rec.weights,
                          np.ascontiguousarray(dl_de[:, 3:], grid.dtype), rec.active_levels)
    return out


def backward_second(grid, point, u, out=None):
    """`hash_encoding.py:257-272`: Eq. 9 scatter of the jacobian cotangent."""
    rec = point.corner_records
    if rec is None:
        raise ValueError("stale sample: encode was called without caches")
    out = grid.zero_gradient() if out is None else out
    kernels.scatter_second(out, rec.indices, rec.weight_gradients,
                           np.ascontiguousarray(u[:, 3:, :], grid.dtype), rec.active_levels)
    return out


def hessian_contract(grid, x, max_level, coeff):
    """`hash_encoding.py:240-254`: sum_a coeff[p,a] d2 e_a / dx dx, (P, 3, 3)."""
    xb = np.ascontiguousarray(_batch(x), grid.dtype)
    xn = grid.normalize(xb)
    inv_extent = np.ascontiguousarray(1.0 / grid.aabb_extent, grid.dtype)
    return kernels.hessian_contract(xn, grid.tables, grid.resolutions,
                                    active_level_count(grid, max_level), inv_extent, coeff)
