"""The neural field on B200 (API of `hashsdf/field.py`).

All learnable state lives in ONE flat fp32 device buffer
    [ H1 (w, E+1) | H2 (16, w) | C1 (w, 25) | C2 (w, w) | C3 (3, w) | pad | tables (L, T, 2) ]
so the gradient all-reduce and the fused multi-group Adam each touch one contiguous
range (MLPs first, then the active table levels).  `grid.tables`, `sdf_net.layers`
and `color_net.layers` are views into it; `sharpness_log` is a separate fp64 device
scalar (`field.py:78`).

`eval_field` / `field_backward` call the libns2b field kernels (csrc/field_tc.cu):
the forward (gather + tcgen05 MLP forward) writes d, g, n, c per sample and leaves
its staged operand tiles in the cache's workspace; the backward (tcgen05 MLP
backward + table scatter) reads them back and accumulates all parameter gradients,
including the Eq. 9 table path and the Theorem-1 SDF path.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from . import hash_encoding as enc
from .hash_encoding import as_device
from .relu_mlp import MlpWeights, ShapeError

GEO_FEATURE_DIM = 15
COLOR_IN_DIM = 3 + 3 + 3 + 1 + GEO_FEATURE_DIM


@dataclass
class FieldConfig:
    """`field.py:49-58`."""

    num_levels: int = 14
    min_resolution: int = 16
    max_resolution: int = 2048
    features_per_level: int = 2
    table_size: int = 2**19
    hidden_width: int = 64
    aabb: tuple = enc.DEFAULT_AABB
    dtype: type = np.float32


class ParamLayout:
    """Offsets (in floats) of every parameter block inside the flat buffer."""

    def __init__(self, num_levels, table_size, width=64):
        self.L, self.T, self.w = int(num_levels), int(table_size), int(width)
        self.E = 3 + 2 * self.L
        w = self.w
        self.sdf_shapes = [(w, self.E + 1), (1 + GEO_FEATURE_DIM, w)]
        self.color_shapes = [(w, COLOR_IN_DIM), (w, w), (3, w)]
        off = 0
        self.sdf_offs = []
        for s in self.sdf_shapes:
            self.sdf_offs.append(off)
            off += s[0] * s[1]
        self.color_offs = []
        for s in self.color_shapes:
            self.color_offs.append(off)
            off += s[0] * s[1]
        self.mlp_floats = off
        self.tables_off = (off + 63) // 64 * 64
        self.table_floats = self.L * self.T * 2
        self.total = self.tables_off + self.table_floats

    def views(self, flat):
        sdf = [flat[o:o + a * b].view(a, b) for o, (a, b) in zip(self.sdf_offs, self.sdf_shapes)]
        col = [flat[o:o + a * b].view(a, b) for o, (a, b) in zip(self.color_offs, self.color_shapes)]
        tab = flat[self.tables_off:self.tables_off + self.table_floats].view(self.L, self.T, 2)
        return sdf, col, tab

    def active_end(self, n_active):
        """End of the [MLP | tables[:n_active]] prefix that receives gradients."""
        return self.tables_off + int(n_active) * self.T * 2


class SdfFieldParams:
    """Ω (tables), Θ (SDF net), Υ (colour net) and s_log on the GPU
    (`field.py:61-116`)."""

    def __init__(self, grid, sdf_net, color_net, sharpness_log):
        enc_dim = grid.encoding_dim
        if sdf_net.in_dim != enc_dim + 1:
            raise ShapeError("shape error: sdf net input must be encoding dim + 1")
        if sdf_net.out_dim != 1 + GEO_FEATURE_DIM:
            raise ShapeError("shape error: sdf net must output 16 values")
        if color_net.in_dim != COLOR_IN_DIM or color_net.out_dim != 3:
            raise ShapeError("shape error: color net must map 25 -> 3")
        if sdf_net.depth != 2 or color_net.depth != 3:
            raise NotImplementedError("kernels implement the paper's 1-layer SDF / 2-layer colour nets")
        width = sdf_net.layers[0].shape[0]
        if width != 64 or any(h.shape[0] != 64 for h in color_net.layers[:-1]):
            raise NotImplementedError("kernels are built for hidden width 64")
        self.layout = ParamLayout(grid.num_levels, grid.table_size, width)
        dev = _lib.device()
        self.flat = torch.zeros(self.layout.total, dtype=torch.float32, device=dev)
        sdf_v, col_v, tab_v = self.layout.views(self.flat)
        for dst, src in zip(sdf_v, sdf_net.layers):
            dst.copy_(src)
        for dst, src in zip(col_v, color_net.layers):
            dst.copy_(src)
        tab_v.copy_(grid.tables)
        grid.tables = tab_v
        sdf_net.layers = sdf_v
        color_net.layers = col_v
        self.grid, self.sdf_net, self.color_net = grid, sdf_net, color_net
        slog = np.asarray(sharpness_log, np.float64).reshape(1)
        self.sharpness_log = torch.from_numpy(slog.copy()).to(dev)
        self._slog_host = float(slog[0])

    @classmethod
    def create(cls, config=None, rng=None, sharpness=20.0):
        """Seeded init with the reference's rng draw order (`field.py:80-99`)."""
        cfg = config or FieldConfig()
        rng = rng or np.random.default_rng(0)
        grid = enc.MultiResHashGrid(cfg.num_levels, cfg.min_resolution, cfg.max_resolution,
                                    cfg.features_per_level, cfg.table_size, cfg.aabb, cfg.dtype,
                                    rng)
        w = cfg.hidden_width
        sdf = MlpWeights.random_host([grid.encoding_dim + 1, w, 1 + GEO_FEATURE_DIM], rng)
        col = MlpWeights.random_host([COLOR_IN_DIM, w, w, 3], rng)
        return cls(grid, MlpWeights(sdf), MlpWeights(col), np.log(sharpness))

    @property
    def sharpness(self):
        return float(np.exp(self._slog_host))

    @property
    def dtype(self):
        return np.dtype(np.float32)

    def refresh_host_mirror(self, slog_value=None):
        """Update the host copy of s_log (after a device-side Adam step)."""
        if slog_value is None:
            slog_value = float(self.sharpness_log.item())
        self._slog_host = float(slog_value)

    def copy(self):
        grid = enc.MultiResHashGrid(self.grid.num_levels, int(self.grid.resolutions[0]),
                                    int(self.grid.resolutions[-1]), 2, self.grid.table_size,
                                    (tuple(self.grid.aabb_min),
                                     tuple(self.grid.aabb_min + self.grid.aabb_extent)),
                                    tables=self.grid.tables.clone())
        grid.resolutions = self.grid.resolutions.copy()
        out = SdfFieldParams(grid, self.sdf_net.copy(), self.color_net.copy(),
                             np.array([self._slog_host]))
        out.sharpness_log.copy_(self.sharpness_log)
        return out

    def field_struct(self, n_active):
        """ns2b_field_t describing this field with `n_active` leading levels."""
        g = self.grid
        f = _lib.FieldT()
        f.num_levels = g.num_levels
        f.table_size = g.table_size
        f.features_per_level = 2
        f.n_active = int(n_active)
        for i, r in enumerate(g.resolutions):
            f.resolutions[i] = int(r)
        lo = g.aabb_min.astype(np.float32)
        ext = g.aabb_extent.astype(np.float32)
        inv = g.inv_extent_f32()
        for k in range(3):
            f.aabb_min[k] = float(lo[k])
            f.aabb_extent[k] = float(ext[k])
            f.inv_extent[k] = float(inv[k])
        f.hidden_width = self.layout.w
        f.tables = ctypes.c_void_p(self.grid.tables.data_ptr())
        f.sdf_w = ctypes.c_void_p(self.sdf_net.layers[0].data_ptr())
        f.color_w = ctypes.c_void_p(self.color_net.layers[0].data_ptr())
        return f


def fibonacci_directions(n):
    """`field.py:119-125`."""
    k = np.arange(n) + 0.5
    polar = np.arccos(1 - 2 * k / n)
    azim = np.pi * (1 + 5**0.5) * k
    return np.stack([np.cos(azim) * np.sin(polar), np.sin(azim) * np.sin(polar), np.cos(polar)],
                    axis=1)


def sal_geometry_init(params, radius=0.5, rng=None):
    """Sphere-like SDF init (`field.py:128-165`): drawn on the host with the
    reference's rng order, uploaded into the flat buffer."""
    rng = rng or np.random.default_rng(0)
    grid, sdf = params.grid, params.sdf_net
    shape = tuple(grid.tables.shape)
    grid.tables.copy_(torch.from_numpy(rng.uniform(-1e-4, 1e-4, size=shape).astype(np.float32)))
    width = sdf.layers[0].shape[0]
    e = grid.encoding_dim
    pairs = (width - 2) // 2
    dirs = fibonacci_directions(pairs)
    h1 = np.zeros((width, e + 1))
    h1[0:2 * pairs:2, 0:3] = dirs
    h1[1:2 * pairs:2, 0:3] = -dirs
    h1[width - 2, e] = 1.0
    h1[:, 3:e] = rng.standard_normal((width, e - 3)) * np.sqrt(2.0 / e)
    sdf.layers[0].copy_(torch.from_numpy(h1.astype(np.float32)))
    h2 = rng.standard_normal(tuple(sdf.layers[1].shape)) * 0.1
    h2[0, :] = 0.0
    h2[0, :2 * pairs] = 2.0 / pairs
    h2[0, width - 2] = -radius
    sdf.layers[1].copy_(torch.from_numpy(h2.astype(np.float32)))
    for h in params.color_net.layers:
        w = rng.standard_normal(tuple(h.shape)) * np.sqrt(2.0 / h.shape[1])
        h.copy_(torch.from_numpy(w.astype(np.float32)))
    return params


@dataclass
class FieldCache:
    """Device-side handle for field_backward (`field.py:168-191`).  Only positions,
    view directions and the level cutoff are needed: the backward recomputes the
    encoding, activations and masks per sample."""

    x: torch.Tensor
    max_level: float
    n_active: int
    ray_ids: torch.Tensor
    dirs: torch.Tensor          # fp64 (m, 3) indexed by ray_ids
    count: torch.Tensor         # device int32 [P]
    sdf: torch.Tensor
    normals: torch.Tensor
    colors: torch.Tensor | None = None
    geo: torch.Tensor | None = None
    has_color: bool = True
    workspace: torch.Tensor | None = None  # gather results the backward reuses

    @property
    def d(self):
        return self.sdf

    @property
    def g(self):
        return self.geo

    @property
    def sdf_out(self):
        return torch.cat([self.sdf[:, None], self.geo], dim=1)

    @property
    def view_dirs(self):
        return self.dirs[self.ray_ids.long()].float()


@dataclass
class FieldGrads:
    tables: torch.Tensor
    sdf_layers: list
    color_layers: list
    flat: torch.Tensor | None = None
    dl_dx: torch.Tensor | None = None
    dl_dv: torch.Tensor | None = None


def new_grads(params):
    flat = torch.zeros_like(params.flat)
    sdf, col, tab = params.layout.views(flat)
    return FieldGrads(tab, sdf, col, flat)


def eval_field(params, x, view_dirs=None, max_level=None, need_color=True):
    """Forward over a batch (`field.py:208-244`); returns a FieldCache."""
    if max_level is None:
        max_level = params.grid.num_levels
    xb = as_device(x, torch.float32).reshape(-1, 3).contiguous()
    if not bool(torch.isfinite(xb).all()):
        raise ValueError("invalid position")
    npts = xb.shape[0]
    if need_color:
        if view_dirs is None:
            raise ValueError("view_dirs required for color evaluation")
        v = as_device(view_dirs, torch.float64).reshape(-1, 3).contiguous()
    else:
        v = torch.zeros((npts, 3), dtype=torch.float64, device=xb.device)
    ray_ids = torch.arange(npts, dtype=torch.int32, device=xb.device)
    count = torch.tensor([npts], dtype=torch.int32, device=xb.device)
    na = enc.active_level_count(params.grid, max_level)
    sdf = torch.empty(npts, dtype=torch.float32, device=xb.device)
    colors = torch.empty((npts, 3), dtype=torch.float32, device=xb.device)
    normals = torch.empty((npts, 3), dtype=torch.float32, device=xb.device)
    geo = torch.empty((npts, GEO_FEATURE_DIM), dtype=torch.float32, device=xb.device)
    f = params.field_struct(na)
    ws = _lib.field_workspace(npts, xb.device)
    _lib.call("ns2b_field_forward", ctypes.byref(f), _lib.ptr(xb), _lib.ptr(ray_ids), _lib.ptr(v),
              _lib.ptr(count), npts, _lib.ptr(sdf), _lib.ptr(colors), _lib.ptr(normals),
              _lib.ptr(geo), None, _lib.ptr(ws), _lib.stream_ptr())
    return FieldCache(xb, max_level, na, ray_ids, v, count, sdf, normals,
                      colors if need_color else None, geo, need_color, ws)


def eval_sdf(params, x, max_level=None):
    c = eval_field(params, x, max_level=max_level, need_color=False)
    return c.d, c.g, c


def eval_normal(params, x, max_level=None):
    return eval_field(params, x, max_level=max_level, need_color=False).normals


def field_sdf_only(params, positions, max_level):
    """Lean SDF query (`renderer.py:131-142`)."""
    xb = as_device(positions, torch.float32).reshape(-1, 3).contiguous()
    out = torch.empty(xb.shape[0], dtype=torch.float32, device=xb.device)
    f = params.field_struct(enc.active_level_count(params.grid, max_level))
    _lib.call("ns2b_field_sdf", ctypes.byref(f), _lib.ptr(xb), xb.shape[0], _lib.ptr(out),
              _lib.stream_ptr())
    return out


def sigmoid(z):
    """Stable logistic (`field.py:40-46`) on host arrays or device tensors."""
    if isinstance(z, torch.Tensor):
        return torch.sigmoid(z)
    z = np.asarray(z)
    out = np.empty_like(z)
    pos = z >= 0
    out[pos] = 1.0 / (1.0 + np.exp(-z[pos]))
    ez = np.exp(z[~pos])
    out[~pos] = ez / (1.0 + ez)
    return out


def eval_color(params, cache, view_dirs):
    """Colour of an evaluated batch for new view directions (`field.py:258-269`).  The
    colour net is fused into the field forward kernel, so this re-runs the forward at the
    cached positions and level cutoff with the new directions and refreshes the cache
    (the SDF outputs are unchanged, so field_backward sees a consistent cache)."""
    fresh = eval_field(params, cache.x, view_dirs, cache.max_level, need_color=True)
    for k in ("ray_ids", "dirs", "count", "sdf", "normals", "colors", "geo", "has_color", "workspace"):
        setattr(cache, k, getattr(fresh, k))
    return cache.colors


def field_backward(params, cache, dl_dc=None, dl_dd=None, dl_dn=None, need_input_grads=False,
                   grads=None):
    """Parameter gradients from per-sample cotangents (`field.py:272-350`).

    Accumulates into `grads` (a FieldGrads from new_grads) when given.  With
    `need_input_grads` also sets grads.dl_dx / grads.dl_dv (P,3) fp32, the position
    and view-direction cotangents of the transform optimiser (`field.py:332-349`:
    the tcgen05 backward leaves the colour-input and de_aug position cotangents in the
    workspace, `field_input_levels_kernel` adds de.J and the encoding curvature)."""
    if cache is None or cache.x is None:
        raise ValueError("stale sample")
    if dl_dc is not None and not cache.has_color:
        raise ValueError("stale sample")
    npts = cache.x.shape[0]
    dev = cache.x.device

    def _cot(a, shape):
        if a is None:
            return torch.zeros(shape, dtype=torch.float32, device=dev)
        return as_device(a, torch.float32).reshape(shape).contiguous()

    gc = _cot(dl_dc, (npts, 3))
    gd = _cot(dl_dd, (npts,))
    gn = None if dl_dn is None else _cot(dl_dn, (npts, 3))
    grads = new_grads(params) if grads is None else grads
    f = params.field_struct(cache.n_active)
    if not need_input_grads:
        _lib.call("ns2b_field_backward", ctypes.byref(f), _lib.ptr(cache.x), _lib.ptr(cache.ray_ids),
                  _lib.ptr(cache.dirs), _lib.ptr(cache.count), npts, _lib.ptr(gc), _lib.ptr(gd),
                  _lib.ptr(gn), 0.0, None, _lib.ptr(grads.sdf_layers[0]),
                  _lib.ptr(grads.color_layers[0]), _lib.ptr(grads.tables), _lib.ptr(cache.workspace),
                  _lib.stream_ptr())
        return grads
    grads.dl_dx = torch.empty((npts, 3), dtype=torch.float32, device=dev)
    grads.dl_dv = torch.empty((npts, 3), dtype=torch.float32, device=dev)
    _lib.call("ns2b_field_backward_inputs", ctypes.byref(f), _lib.ptr(cache.count), npts, _lib.ptr(gc),
              _lib.ptr(gd), _lib.ptr(gn), 0.0, None, _lib.ptr(grads.sdf_layers[0]),
              _lib.ptr(grads.color_layers[0]), _lib.ptr(grads.dl_dx), _lib.ptr(grads.dl_dv),
              _lib.ptr(cache.workspace), _lib.stream_ptr())
    _lib.call("ns2b_field_scatter", ctypes.byref(f), _lib.ptr(cache.x), _lib.ptr(cache.count), npts,
              _lib.ptr(grads.tables), _lib.ptr(cache.workspace), _lib.stream_ptr())
    return grads
