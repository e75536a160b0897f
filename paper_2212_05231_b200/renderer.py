"""Occupancy marching + NeuS volume rendering on B200 (API of `hashsdf/renderer.py`).

Device kernels (libns2b): `ns2b_march_count(_masked)` / `ns2b_scan_offsets` / `ns2b_march_fill(_masked)`
(K1, fp64, bit-exact sample sets), `ns2b_field_forward` (K2), `ns2b_composite`
(K3: per-ray alpha / transmittance / weights / colour, optionally fused with the
Huber loss and the compositing backward) and `ns2b_composite_backward` (K4).

Samples are stored ray-major; per-interval quantities (alpha, weight, T before)
are kept per *sample* (the interval's first sample) so every kernel indexes one
contiguous per-ray range.  `RenderRecords.interval_first / alphas / weights`
reproduce the reference's per-interval views on demand.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from . import field as fieldmod
from . import hash_encoding as enc
from .hash_encoding import as_device

ALPHA_MAX = 1.0 - 1e-7         # renderer.py:28
LOGISTIC_CLAMP = 80.0          # renderer.py:29
MAX_SAMPLES_PER_RAY = 512      # renderer.py:30
STEP_DIVISOR = 512             # renderer.py:31
EMA_DECAY = 0.95               # renderer.py:32


# ------------------------------------------------------------ host helpers --
def sdf_transforms(sharpness, f):
    """(Phi_s, phi_s) host helper (`renderer.py:35-49`); the kernels inline it."""
    z = np.clip(sharpness * np.asarray(f, np.float64), -LOGISTIC_CLAMP, LOGISTIC_CLAMP)
    cdf = np.where(z >= 0, 1.0 / (1.0 + np.exp(-np.abs(z))),
                   np.exp(-np.abs(z)) / (1.0 + np.exp(-np.abs(z))))
    return cdf, sharpness * cdf * (1.0 - cdf)


def alpha(f_i, f_next, sharpness):
    """`renderer.py:52-56` host helper."""
    a, _ = sdf_transforms(sharpness, f_i)
    b, _ = sdf_transforms(sharpness, f_next)
    return np.clip((a - b) / a, 0.0, ALPHA_MAX)


def composite(alphas, colors):
    """`renderer.py:59-69` host helper for one ray."""
    a = np.asarray(alphas, np.float64)
    c = np.asarray(colors, np.float64)
    trans = np.concatenate([[1.0], np.cumprod(1.0 - a)])
    w = trans[:-1] * a
    return w @ c.reshape(len(a), -1), w, float(trans[-1])


# ---------------------------------------------------------------- occupancy --
class OccupancyGrid:
    """Coarse G^3 grid of occupied cells (`renderer.py:72-105`); ema (fp64) and bits
    (uint8) live on the device, [x][y][z] order."""

    def __init__(self, resolution=128, aabb=((-1.0, -1.0, -1.0), (1.0, 1.0, 1.0)),
                 threshold=0.01):
        self.resolution = int(resolution)
        self.aabb = aabb
        self.threshold = float(threshold)
        self.lo = np.asarray(aabb[0], np.float64)
        self.hi = np.asarray(aabb[1], np.float64)
        g = self.resolution
        dev = _lib.device()
        self.ema = torch.zeros((g, g, g), dtype=torch.float64, device=dev)
        self.bits = torch.zeros((g, g, g), dtype=torch.uint8, device=dev)
        self.step_size = float(np.linalg.norm(self.hi - self.lo)) / STEP_DIVISOR

    def set_all(self, value=True):
        self.bits.fill_(1 if value else 0)
        return self

    def set_bits(self, bits):
        self.bits.copy_(as_device(np.asarray(bits).astype(np.uint8), torch.uint8).view_as(self.bits))
        return self

    def cell_centers(self):
        g = self.resolution
        ax = [self.lo[a] + (np.arange(g) + 0.5) * (self.hi[a] - self.lo[a]) / g for a in range(3)]
        grid = np.meshgrid(*ax, indexing="ij")
        return np.stack([v.ravel() for v in grid], axis=1)

    def occupied_fraction(self):
        return float(self.bits.float().mean().item())

    def struct(self):
        o = _lib.OccT()
        o.resolution = self.resolution
        for k in range(3):
            o.lo[k] = float(self.lo[k])
            o.hi[k] = float(self.hi[k])
        o.step_size = self.step_size
        o.bits = ctypes.c_void_p(self.bits.data_ptr())
        return o


def cell_centers_device(occ):
    """`renderer.py:92-96` on the device: lo + (i + 0.5) * extent / G per axis (fp64,
    same operation order as the reference, so the same bits), C-order (G^3, 3)."""
    g = occ.resolution
    dev = occ.ema.device
    ax = [float(occ.lo[a]) + (torch.arange(g, dtype=torch.float64, device=dev) + 0.5)
          * float(occ.hi[a] - occ.lo[a]) / g for a in range(3)]
    xx, yy, zz = torch.meshgrid(*ax, indexing="ij")
    return torch.stack([xx.reshape(-1), yy.reshape(-1), zz.reshape(-1)], dim=1)


def update_occupancy(occ, params, max_level, rng=None, point_transform=None, chunk=1 << 18):
    """Refresh EMA / bits from the field (`renderer.py:108-128`), one kernel over all
    G^3 cell centres.  `rng` and `chunk` are accepted for interface parity.

    `point_transform` (dynamic scenes) maps the marching-space centres, an fp64 (N, 3)
    device tensor, into the field's canonical space; the moved centres are queried
    with ns2b_field_sdf and folded into the EMA by ns2b_occupancy_from_sdf."""
    na = enc.active_level_count(params.grid, max_level)
    if point_transform is not None:
        pts = as_device(point_transform(cell_centers_device(occ)), torch.float64).reshape(-1, 3)
        sdf = fieldmod.field_sdf_only(params, pts, max_level)
        _lib.call("ns2b_occupancy_from_sdf", _lib.ptr(sdf), sdf.numel(), params.sharpness, occ.step_size,
                  occ.threshold, _lib.ptr(occ.ema), _lib.ptr(occ.bits), _lib.stream_ptr())
        return occ
    f = params.field_struct(na)
    o = occ.struct()
    _lib.call("ns2b_occupancy_update", ctypes.byref(f), ctypes.byref(o), params.sharpness,
              occ.threshold, _lib.ptr(occ.ema), _lib.ptr(occ.bits), _lib.stream_ptr())
    return occ


def field_sdf_only(params, positions, max_level):
    return fieldmod.field_sdf_only(params, positions, max_level)


# ----------------------------------------------------------------- marching --
@dataclass
class MarchResult:
    ray_ids: torch.Tensor        # (P,) int32
    t: torch.Tensor | None       # (P,) fp64
    positions: torch.Tensor | None  # (P,3) fp64
    num_rays: int
    offsets: torch.Tensor = None  # (m+1,) int32, offsets[m] = P
    positions32: torch.Tensor = None  # (P,3) fp32
    count: torch.Tensor = None    # device int32 [P]
    sample_count: int = 0


class _ScanWorkspace:
    def __init__(self):
        self.buf = None

    def get(self, counts, nrays, offsets):
        need = ctypes.c_size_t(0)
        _lib.call("ns2b_scan_offsets", _lib.ptr(counts), nrays, _lib.ptr(offsets), None,
                  ctypes.byref(need), _lib.stream_ptr())
        if self.buf is None or self.buf.numel() < need.value:
            self.buf = torch.empty(max(int(need.value), 256), dtype=torch.uint8,
                                   device=counts.device)
        return self.buf, need


_scan_ws = _ScanWorkspace()


def march_count_and_scan(o, d, occ, counts, offsets, stream=None, keep_mask=None):
    """Kernel pass 1 + exclusive scan (device only, no sync).  With `keep_mask` (m x 16
    int32) pass 1 also records each ray's kept candidates for `ns2b_march_fill_masked`."""
    st = _lib.stream_ptr(stream)
    m = o.shape[0]
    s = occ.struct()
    if keep_mask is not None:
        _lib.call("ns2b_march_count_masked", _lib.ptr(o), _lib.ptr(d), m, ctypes.byref(s), _lib.ptr(counts),
                  _lib.ptr(keep_mask), st)
    else:
        _lib.call("ns2b_march_count", _lib.ptr(o), _lib.ptr(d), m, ctypes.byref(s), _lib.ptr(counts), st)
    buf, need = _scan_ws.get(counts, m, offsets)
    _lib.call("ns2b_scan_offsets", _lib.ptr(counts), m, _lib.ptr(offsets), _lib.ptr(buf),
              ctypes.byref(need), st)


def intersect_aabb(origins, dirs, lo, hi):
    """Slab test (`renderer.py:153-168`) as fp64 device tensor ops with the reference's
    operation order (1/d, then (lo-o)*inv), so the entry/exit values are bit-identical;
    the marcher (`ns2b_march_*`) runs the same arithmetic inline.  Returns device
    (t_enter, t_exit); exit < enter on a miss."""
    o = as_device(origins, torch.float64).reshape(-1, 3)
    d = as_device(dirs, torch.float64).reshape(-1, 3)
    lo_t = torch.as_tensor(np.asarray(lo, np.float64), device=o.device)
    hi_t = torch.as_tensor(np.asarray(hi, np.float64), device=o.device)
    inv = 1.0 / d
    t1 = (lo_t - o) * inv
    t2 = (hi_t - o) * inv
    near, far = torch.minimum(t1, t2), torch.maximum(t1, t2)
    par = d.abs() < 1e-12
    inside = (o >= lo_t) & (o <= hi_t)
    inf = torch.tensor(float("inf"), dtype=torch.float64, device=o.device)
    near = torch.where(par, torch.where(inside, -inf, inf), near)
    far = torch.where(par, torch.where(inside, inf, -inf), far)
    return torch.clamp(near.amax(dim=1), min=0.0), far.amin(dim=1)


def march_rays(origins, dirs, occ, need_t=True, need_pos64=True, masked=True):
    """Fixed-stride marching with empty-space skipping (`renderer.py:171-192`).  `masked`:
    pass 1 records the kept candidates and pass 2 computes only their positions (same
    outputs, bit for bit)."""
    o = as_device(origins, torch.float64).reshape(-1, 3).contiguous()
    d = as_device(dirs, torch.float64).reshape(-1, 3).contiguous()
    m = o.shape[0]
    dev = o.device
    counts = torch.empty(m, dtype=torch.int32, device=dev)
    offsets = torch.empty(m + 1, dtype=torch.int32, device=dev)
    keep = torch.empty((m, 16), dtype=torch.int32, device=dev) if masked else None
    march_count_and_scan(o, d, occ, counts, offsets, keep_mask=keep)
    P = int(offsets[m].item())
    ray_ids = torch.empty(P, dtype=torch.int32, device=dev)
    t = torch.empty(P, dtype=torch.float64, device=dev) if need_t else None
    p64 = torch.empty((P, 3), dtype=torch.float64, device=dev) if need_pos64 else None
    p32 = torch.empty((P, 3), dtype=torch.float32, device=dev)
    s = occ.struct()
    if masked:
        _lib.call("ns2b_march_fill_masked", _lib.ptr(o), _lib.ptr(d), m, ctypes.byref(s), _lib.ptr(offsets),
                  _lib.ptr(keep), _lib.ptr(ray_ids), _lib.ptr(t), _lib.ptr(p64), _lib.ptr(p32),
                  _lib.stream_ptr())
    else:
        _lib.call("ns2b_march_fill", _lib.ptr(o), _lib.ptr(d), m, ctypes.byref(s), _lib.ptr(offsets),
                  _lib.ptr(ray_ids), _lib.ptr(t), _lib.ptr(p64), _lib.ptr(p32), _lib.stream_ptr())
    return MarchResult(ray_ids, t, p64, m, offsets, p32, offsets[m:m + 1], P)


# ---------------------------------------------------------------- rendering --
@dataclass
class RenderRecords:
    """What the backward pass needs (`renderer.py:195-214`), device resident."""

    ray_ids: torch.Tensor
    t: torch.Tensor | None
    frame_positions: torch.Tensor | None
    sdf: torch.Tensor              # (P,) fp32 (the field's output; the reference upcasts)
    sample_colors: torch.Tensor    # (P,3) fp32
    alphas_per_sample: torch.Tensor   # (P,) fp64, valid at interval-first samples
    weights_per_sample: torch.Tensor
    trans_before_per_sample: torch.Tensor
    transmittance: torch.Tensor    # (m,) fp64
    sharpness: float
    num_rays: int
    offsets: torch.Tensor
    cache: object = None
    sample_count: int = 0

    @property
    def interval_first(self):
        r = self.ray_ids
        if r.numel() < 2:
            return torch.zeros(0, dtype=torch.int64, device=r.device)
        return torch.nonzero(r[1:] == r[:-1]).flatten()

    @property
    def alphas(self):
        return self.alphas_per_sample[self.interval_first]

    @property
    def weights(self):
        return self.weights_per_sample[self.interval_first]


def _empty_records(m, s, dev):
    z64 = torch.zeros(0, dtype=torch.float64, device=dev)
    return RenderRecords(torch.zeros(0, dtype=torch.int32, device=dev), z64, z64.view(0, 3),
                         torch.zeros(0, dtype=torch.float32, device=dev),
                         torch.zeros((0, 3), dtype=torch.float32, device=dev), z64, z64, z64,
                         torch.ones(m, dtype=torch.float64, device=dev), s, m,
                         torch.zeros(m + 1, dtype=torch.int32, device=dev), None, 0)


def composite_forward(offsets, m, sdf, colors, s, rendered, resid, alphas, weights, tb,
                      stream=None):
    _lib.call("ns2b_composite", _lib.ptr(offsets), m, _lib.ptr(sdf), _lib.ptr(colors), float(s),
              None, 0.0, 1.0, _lib.ptr(rendered), _lib.ptr(resid), _lib.ptr(alphas),
              _lib.ptr(weights), _lib.ptr(tb), None, None, None, _lib.stream_ptr(stream))


def render_rays(batch, params, occ, max_level, point_transform=None, dir_transform=None):
    """March, evaluate the field, composite (`renderer.py:234-291`).  Returns
    (colors (m,3) fp64 CUDA tensor, RenderRecords).  Like the reference, `params`
    may be an analytic object with `.sharpness` and `.evaluate(pos, dirs)`.

    `point_transform` / `dir_transform` (dynamic scenes, `renderer.py:257-264`) map
    the marched samples' fp64 positions (P,3) / per-sample view directions (P,3),
    device tensors, into the field's canonical space; marching and compositing stay
    in the marching space."""
    o = as_device(batch.origins, torch.float64).reshape(-1, 3).contiguous()
    d = as_device(batch.directions, torch.float64).reshape(-1, 3).contiguous()
    m = o.shape[0]
    s = float(params.sharpness)
    mr = march_rays(o, d, occ)
    P = mr.sample_count
    if P == 0:
        return torch.zeros((m, 3), dtype=torch.float64, device=o.device), _empty_records(m, s, o.device)
    pos32, fids, fdirs = mr.positions32, mr.ray_ids, d
    if point_transform is not None:
        pos32 = as_device(point_transform(mr.positions), torch.float64).reshape(-1, 3).float().contiguous()
    if dir_transform is not None:
        fdirs = as_device(dir_transform(d[mr.ray_ids.long()]), torch.float64).reshape(-1, 3).contiguous()
        fids = torch.arange(P, dtype=torch.int32, device=o.device)
    if hasattr(params, "evaluate"):
        pos_f = mr.positions if point_transform is None else point_transform(mr.positions)
        sdf, cols = params.evaluate(pos_f, fdirs[fids.long()])
        sdf = as_device(sdf, torch.float32).reshape(-1).contiguous()
        cols = as_device(cols, torch.float32).reshape(-1, 3).contiguous()
        cache = None
    else:
        na = enc.active_level_count(params.grid, max_level)
        sdf = torch.empty(P, dtype=torch.float32, device=o.device)
        cols = torch.empty((P, 3), dtype=torch.float32, device=o.device)
        normals = torch.empty((P, 3), dtype=torch.float32, device=o.device)
        geo = torch.empty((P, fieldmod.GEO_FEATURE_DIM), dtype=torch.float32, device=o.device)
        f = params.field_struct(na)
        ws = _lib.field_workspace(P, o.device)
        _lib.call("ns2b_field_forward", ctypes.byref(f), _lib.ptr(pos32), _lib.ptr(fids),
                  _lib.ptr(fdirs), _lib.ptr(mr.count), P, _lib.ptr(sdf), _lib.ptr(cols),
                  _lib.ptr(normals), _lib.ptr(geo), None, _lib.ptr(ws), _lib.stream_ptr())
        cache = fieldmod.FieldCache(pos32, max_level, na, fids, fdirs, mr.count, sdf, normals, cols,
                                    geo, True, ws)
    rendered = torch.empty((m, 3), dtype=torch.float64, device=o.device)
    resid = torch.empty(m, dtype=torch.float64, device=o.device)
    a = torch.zeros(P, dtype=torch.float64, device=o.device)
    w = torch.zeros(P, dtype=torch.float64, device=o.device)
    tb = torch.zeros(P, dtype=torch.float64, device=o.device)
    composite_forward(mr.offsets, m, sdf, cols, s, rendered, resid, a, w, tb)
    rec = RenderRecords(mr.ray_ids, mr.t, mr.positions, sdf, cols, a, w, tb, resid, s, m,
                        mr.offsets, cache, P)
    return rendered, rec


def expected_depth(records):
    """sum_i w_i t_i per ray (`renderer.py:294-300`)."""
    ii = records.interval_first
    out = torch.zeros(records.num_rays, dtype=torch.float64, device=records.ray_ids.device)
    out.index_add_(0, records.ray_ids[ii].long(), records.weights_per_sample[ii] * records.t[ii])
    return out


def backward_cotangents(records, dl_dray_colors):
    """Pixel-colour cotangent -> (dL/dc (P,3) fp32, dL/dsdf (P,) fp32, dL/dslog float)
    (`renderer.py:303-358`)."""
    P = records.sample_count
    dev = records.ray_ids.device
    dl_dc = torch.zeros((P, 3), dtype=torch.float32, device=dev)
    dl_df = torch.zeros(P, dtype=torch.float32, device=dev)
    if P == 0:
        return dl_dc, dl_df, 0.0
    g = as_device(dl_dray_colors, torch.float64).reshape(-1, 3).contiguous()
    sums = torch.zeros(4, dtype=torch.float64, device=dev)
    _lib.call("ns2b_composite_backward", _lib.ptr(records.offsets), records.num_rays,
              _lib.ptr(records.sdf), _lib.ptr(records.sample_colors), float(records.sharpness),
              _lib.ptr(records.alphas_per_sample), _lib.ptr(records.weights_per_sample),
              _lib.ptr(records.trans_before_per_sample), _lib.ptr(g), _lib.ptr(dl_dc),
              _lib.ptr(dl_df), _lib.ptr(sums), _lib.stream_ptr())
    return dl_dc, dl_df, float(sums[1].item()) * records.sharpness
