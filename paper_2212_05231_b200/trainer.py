"""Static-scene training step on B200 (API of `hashsdf/trainer.py`).

`train_step` runs the whole NeuS2 step on the device through libns2b:

  level schedule -> [occupancy refresh every 16 steps]            (host int / K-occ)
  host ray batch (same rng draws as the reference) -> pinned H2D
  march count -> scan -> fill                                    (K1)
  [DP: all-reduce P]
  field forward: encoding, SDF net, analytic normal, colour net   (K2)
  composite + Huber loss + compositing backward (per ray)         (K3/K4)
  field backward: recompute, colour bwd, SDF bwd, Eq. 9 scatter,
      Theorem-1 weight grads, Eikonal cotangent fused             (K5)
  [DP: all-reduce gradient prefix + step scalars]
  divergence check -> s_log Adam -> multi-group Adam             (K6)
  one D2H of the step scalars for the LossReport

Parameter groups, learning rates, per-group step counters, masked-level skipping
and the divergence error follow `trainer.py:152-172, 243-278`.
"""

from __future__ import annotations

import ctypes
import dataclasses
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from . import field as fieldmod
from . import hash_encoding as enc
from . import renderer, scene_io
from .hash_encoding import as_device
from .parallel import DataParallel


@dataclass
class TrainConfig:
    """`trainer.py:28-71` (same fields and defaults)."""

    total_steps: int = 15000
    batch_size: int = 4096
    seed: int = 0
    eikonal_weight: float = 0.1
    huber_delta: float = 0.1
    fg_fraction: float = 0.9
    lr_tables: float = 1e-2
    lr_mlp: float = 1e-3
    lr_final_fraction: float = 0.1
    adam_beta1: float = 0.9
    adam_beta2: float = 0.99
    adam_eps: float = 1e-15
    level_init: int = 2
    level_increment_fraction: float = 0.025
    occupancy_resolution: int = 128
    occupancy_update_every: int = 16
    occupancy_threshold: float = 0.01
    num_levels: int = 14
    min_resolution: int = 16
    max_resolution: int = 2048
    features_per_level: int = 2
    table_size: int = 2**19
    hidden_width: int = 64
    init_radius: float = 0.5
    init_sharpness: float = 20.0
    dtype: str = "float32"
    first_frame_steps: int = 2000
    frame_steps: int = 1100
    transform_only_steps: int = 100
    transform_lr: float = 1e-3
    transform_joint_lr: float = 1e-4
    frame_lr_scale: float = 0.3

    def replace(self, **kw):
        return dataclasses.replace(self, **kw)


@dataclass
class LossReport:
    step: int
    color: float
    eikonal: float
    total: float
    level: int
    psnr: float
    sample_count: int = 0


@dataclass
class AdamState:
    """Per-group moments (device views into the flat moment buffers) and step t."""

    m: torch.Tensor
    v: torch.Tensor
    t: int = 0


def level_schedule(step, config):
    """`trainer.py:123-126`."""
    window = config.level_increment_fraction * config.total_steps
    return int(min(config.num_levels, config.level_init + np.floor(step / window)))


def lr_factor(step, total_steps, final_fraction):
    """`trainer.py:129-131`."""
    t = np.clip(step / max(total_steps, 1), 0.0, 1.0)
    return final_fraction + (1.0 - final_fraction) * 0.5 * (1.0 + np.cos(np.pi * t))


def huber(residual, delta):
    r = np.asarray(residual)
    a = np.abs(r)
    return np.where(a <= delta, 0.5 * r * r / delta, a - 0.5 * delta)


def huber_grad(residual, delta):
    r = np.asarray(residual)
    return np.where(np.abs(r) <= delta, r / delta, np.sign(r))


def color_loss(rendered, targets, delta):
    """`trainer.py:108-112`: mean over rays of the channel-summed Huber (host arrays)."""
    r = np.asarray(rendered)
    if r.shape[0] < 1:
        raise ValueError("need at least one ray")
    return float(huber(r - np.asarray(targets), delta).sum(axis=1).mean())


def eikonal_loss(normals):
    """`trainer.py:115-120`: mean (||n|| - 1)^2 (host arrays)."""
    n = np.asarray(normals)
    if n.shape[0] < 1:
        raise ValueError("need at least one normal")
    nn = np.linalg.norm(np.atleast_2d(n), axis=1)
    return float(((nn - 1.0) ** 2).mean())


def psnr_from_mse(mse):
    return 100.0 if mse < 1e-10 else float(10.0 * np.log10(1.0 / mse))


def psnr(image_a, image_b):
    """`trainer.py:134-143` (host helper)."""
    a, b = np.asarray(image_a), np.asarray(image_b)
    if a.shape != b.shape:
        raise ValueError("psnr: shape mismatch")
    return psnr_from_mse(float(np.mean((a - b) ** 2)))


# group order of the divergence check in the reference (trainer.py:249-278)
_CHECK_ORDER = ["tables", "sdf_0", "sdf_1", "color_0", "color_1", "color_2", "sharpness_log"]


class StepWorkspace:
    """Device buffers of one step, grown geometrically with the kept-sample count."""

    def __init__(self, params, dev):
        self.dev = dev
        self.m = 0
        self.cap = 0
        self.grads = torch.zeros_like(params.flat)
        self.sums = torch.zeros(8, dtype=torch.float64, device=dev)
        self.count64 = torch.zeros(1, dtype=torch.int64, device=dev)
        self.flag = torch.zeros(1, dtype=torch.int32, device=dev)
        self.report = torch.zeros(8, dtype=torch.float64, device=dev)
        self.report_host = torch.zeros(8, dtype=torch.float64).pin_memory()
        self.p_host = torch.zeros(1, dtype=torch.int32).pin_memory()

    def rays(self, m):
        if m != self.m:
            d = self.dev
            self.o = torch.empty((m, 3), dtype=torch.float64, device=d)
            self.d = torch.empty((m, 3), dtype=torch.float64, device=d)
            self.tgt = torch.empty((m, 3), dtype=torch.float64, device=d)
            self.counts = torch.empty(m, dtype=torch.int32, device=d)
            self.keep_mask = torch.empty((m, 16), dtype=torch.int32, device=d)  # march pass 1 -> 2
            self.offsets = torch.empty(m + 1, dtype=torch.int32, device=d)
            self.rendered = torch.empty((m, 3), dtype=torch.float64, device=d)
            self.resid = torch.empty(m, dtype=torch.float64, device=d)
            self.m = m

    def samples(self, P):
        if P > self.cap:
            cap = max(int(P * 1.25), 1 << 16)
            d = self.dev
            self.ray_ids = torch.empty(cap, dtype=torch.int32, device=d)
            self.pos32 = torch.empty((cap, 3), dtype=torch.float32, device=d)
            self.sdf = torch.empty(cap, dtype=torch.float32, device=d)
            self.colors = torch.empty((cap, 3), dtype=torch.float32, device=d)
            self.alphas = torch.empty(cap, dtype=torch.float64, device=d)
            self.weights = torch.empty(cap, dtype=torch.float64, device=d)
            self.tb = torch.empty(cap, dtype=torch.float64, device=d)
            self.dl_dc = torch.empty((cap, 3), dtype=torch.float32, device=d)
            self.dl_dsdf = torch.empty(cap, dtype=torch.float32, device=d)
            self.field_ws = _lib.field_workspace(cap, d)
            self.cap = cap


class TrainState:
    """Parameters, moments, occupancy, rng and step (`trainer.py:175-212`)."""

    def __init__(self, params, occ, config, rng, step=0, dp=None):
        self.params, self.occ, self.config, self.step = params, occ, config, step
        self._rng, self._ahead = rng, None
        # with a device-resident dataset, draw the next step's ray picks on the host while
        # the device runs this step (the rng stream and its consumers are unchanged: `rng`
        # rewinds an unused draw before anyone else reads the generator)
        self.draw_ahead = True
        self.dp = dp or DataParallel.from_env()
        dev = params.flat.device
        self.m_flat = torch.zeros_like(params.flat)
        self.v_flat = torch.zeros_like(params.flat)
        lay = params.layout
        sdf_m, col_m, tab_m = lay.views(self.m_flat)
        sdf_v, col_v, tab_v = lay.views(self.v_flat)
        self.adam = {"tables": AdamState(tab_m, tab_v)}
        for i in range(len(sdf_m)):
            self.adam[f"sdf_{i}"] = AdamState(sdf_m[i], sdf_v[i])
        for i in range(len(col_m)):
            self.adam[f"color_{i}"] = AdamState(col_m[i], col_v[i])
        self.adam["sharpness_log"] = AdamState(torch.zeros(1, dtype=torch.float64, device=dev),
                                               torch.zeros(1, dtype=torch.float64, device=dev))
        self.ws = StepWorkspace(params, dev)

    @property
    def rng(self):
        """The reference's generator, at the reference's stream position: a pick draw
        `train_step` made ahead for the next step is rewound first."""
        _rewind_ahead(self)
        return self._rng

    @rng.setter
    def rng(self, g):
        self._rng, self._ahead = g, None

    @classmethod
    def create(cls, config, aabb=((-1, -1, -1), (1, 1, 1)), dp=None):
        """Seeded init in the reference's draw order (`trainer.py:192-212`)."""
        rng = np.random.default_rng(config.seed)
        fcfg = fieldmod.FieldConfig(config.num_levels, config.min_resolution,
                                    config.max_resolution, config.features_per_level,
                                    config.table_size, config.hidden_width, aabb)
        params = fieldmod.SdfFieldParams.create(fcfg, rng, sharpness=config.init_sharpness)
        fieldmod.sal_geometry_init(params, config.init_radius, rng)
        occ = renderer.OccupancyGrid(config.occupancy_resolution, aabb, config.occupancy_threshold)
        return cls(params, occ, config, rng, dp=dp)


class _Timer:
    """Optional per-kernel CUDA-event timing on the launching stream (bench.py)."""

    def __init__(self, store, name, stream):
        self.store, self.name, self.stream = store, name, stream

    def __enter__(self):
        if self.store is not None:
            self.e0 = torch.cuda.Event(enable_timing=True)
            self.e0.record(self.stream)
        return self

    def __exit__(self, *exc):
        if self.store is not None:
            e1 = torch.cuda.Event(enable_timing=True)
            e1.record(self.stream)
            self.store.setdefault(self.name, []).append((self.e0, e1))
        return False


def _upload_batch(ws, batch, sl, stream):
    """Copy the rays `sl` (this rank's shard) of the batch into the workspace."""
    for dst, src in ((ws.o, batch.origins), (ws.d, batch.directions), (ws.tgt, batch.target_colors)):
        if isinstance(src, torch.Tensor):
            s = src[sl]
            if s.device.type == "cpu" and not s.is_contiguous():
                s = s.contiguous().pin_memory()
            dst.copy_(s, non_blocking=True)
        else:
            h = torch.from_numpy(np.ascontiguousarray(src[sl], np.float64))
            dst.copy_(h.pin_memory(), non_blocking=True)


def _rewind_ahead(state):
    """Undo a pick draw made ahead (unless the generator moved since: then the caller
    replaced or re-seeded it and the draw is simply dropped)."""
    ah, state._ahead = state._ahead, None
    if ah is not None and state._rng.bit_generator.state == ah[2]:
        state._rng.bit_generator.state = ah[1]


def _take_ahead(state, key):
    """The draw made ahead if it is still the next draw of the stream with this key."""
    ah = state._ahead
    if ah is not None and ah[0] == key and state._rng.bit_generator.state == ah[2]:
        state._ahead = None
        return ah[3]
    _rewind_ahead(state)
    return None


def train_step(state, dataset, time_index=0, batch=None):
    """One optimisation step (`trainer.py:281-310`); returns a LossReport.

    `batch` (a RayBatch of numpy arrays or CUDA/pinned tensors) replays a given global
    batch instead of sampling; the rng is then not consumed."""
    cfg = state.config
    params, occ, ws, dp = state.params, state.occ, state.ws, state.dp
    st = torch.cuda.current_stream()
    sp = _lib.stream_ptr(st)
    level = level_schedule(state.step, cfg)
    if state.step % cfg.occupancy_update_every == 0:
        renderer.update_occupancy(occ, params, level)
    sampler = getattr(dataset, "_device_samplers", {}).get(time_index) if batch is None else None
    if sampler is not None:
        # f2 (`dataset.to_device()`): the reference's rng draws on the host, only this
        # rank's picks go up and only its rays are built, straight into the workspace
        m_total = cfg.batch_size
        ws.rays(dp.shard_size(m_total))
        draw_key = sampler.draw_key(m_total, cfg.fg_fraction)
        sampler.sample_into(m_total, cfg.fg_fraction, state._rng, ws.o, ws.d, ws.tgt, dp.rank, dp.world,
                            draw=_take_ahead(state, draw_key))
    else:
        if batch is None:
            batch = scene_io.sample_ray_batch(dataset, time_index, cfg.batch_size, cfg.fg_fraction,
                                              state.rng)
        m_total = batch.count
        ws.rays(dp.shard_size(m_total))
        _upload_batch(ws, batch, dp.shard(m_total), st)
    m = ws.m

    timers = getattr(state, "timers", None)
    # K1: march (count, scan) -> P -> fill
    with _Timer(timers, "march_count_scan", st):
        renderer.march_count_and_scan(ws.o, ws.d, occ, ws.counts, ws.offsets, st, keep_mask=ws.keep_mask)
    ws.p_host.copy_(ws.offsets[m:m + 1], non_blocking=True)
    st.synchronize()
    P = int(ws.p_host[0])
    P_glob = dp.allreduce_count(P, ws.dev)
    ws.samples(max(P, 1))
    o = occ.struct()
    with _Timer(timers, "march_fill", st):
        _lib.call("ns2b_march_fill_masked", _lib.ptr(ws.o), _lib.ptr(ws.d), m, ctypes.byref(o),
                  _lib.ptr(ws.offsets), _lib.ptr(ws.keep_mask), _lib.ptr(ws.ray_ids), None, None,
                  _lib.ptr(ws.pos32), sp)
    count = ws.offsets[m:m + 1]
    ws.sums.zero_()
    s = params.sharpness
    na = enc.active_level_count(params.grid, level)
    f = params.field_struct(na)
    # K2: gather (features + d feature/dx -> workspace), two-tile tcgen05 MLP forward
    # (+ Eikonal sum and its cotangent, fused)
    ws.count64.fill_(max(P_glob, 1))  # the Eikonal mean's divisor (global P)
    with _Timer(timers, "field_gather", st):
        _lib.call("ns2b_field_gather", ctypes.byref(f), _lib.ptr(ws.pos32), _lib.ptr(ws.ray_ids),
                  _lib.ptr(ws.d), _lib.ptr(count), P, _lib.ptr(ws.field_ws), sp)
    with _Timer(timers, "field_mlp_forward", st):
        _lib.call("ns2b_field_mlp_forward_eik", ctypes.byref(f), _lib.ptr(ws.pos32),
                  _lib.ptr(ws.ray_ids), _lib.ptr(ws.d), _lib.ptr(count), P, _lib.ptr(ws.sdf),
                  _lib.ptr(ws.colors), None, None, _lib.ptr(ws.sums[3:4]), cfg.eikonal_weight,
                  _lib.ptr(ws.count64), _lib.ptr(ws.field_ws), sp)
    # K3/K4: composite + Huber + compositing backward
    with _Timer(timers, "composite", st):
        _lib.call("ns2b_composite", _lib.ptr(ws.offsets), m, _lib.ptr(ws.sdf),
                  _lib.ptr(ws.colors), s, _lib.ptr(ws.tgt), cfg.huber_delta, float(m_total),
                  _lib.ptr(ws.rendered), _lib.ptr(ws.resid), _lib.ptr(ws.alphas),
                  _lib.ptr(ws.weights), _lib.ptr(ws.tb), _lib.ptr(ws.dl_dc), _lib.ptr(ws.dl_dsdf),
                  _lib.ptr(ws.sums), sp)
    lay = params.layout
    end = lay.active_end(na)
    ws.flag.zero_()
    stepped = []
    if P_glob > 0:
        ws.grads[:end].zero_()
        # K5: field backward with the fused Eikonal cotangent
        sdf_g, col_g, tab_g = lay.views(ws.grads)
        with _Timer(timers, "field_mlp_backward", st):
            _lib.call("ns2b_field_mlp_backward", ctypes.byref(f), _lib.ptr(ws.pos32),
                      _lib.ptr(ws.ray_ids), _lib.ptr(ws.d), _lib.ptr(count), P, _lib.ptr(ws.dl_dc),
                      _lib.ptr(ws.dl_dsdf), None, cfg.eikonal_weight, _lib.ptr(ws.count64),
                      _lib.ptr(sdf_g[0]), _lib.ptr(col_g[0]), _lib.ptr(ws.field_ws), sp)
        with _Timer(timers, "field_scatter", st):
            _lib.call("ns2b_field_scatter", ctypes.byref(f), _lib.ptr(ws.pos32), _lib.ptr(count), P,
                      _lib.ptr(tab_g), _lib.ptr(ws.field_ws), sp)
        if dp.active:
            with _Timer(timers, "allreduce", st):
                dp.allreduce_(ws.grads[:end])
                dp.allreduce_(ws.sums[:4])
        with _Timer(timers, "adam", st):
            stepped = _apply_gradients(state, na, s)
    elif dp.active:
        dp.allreduce_(ws.sums[:4])
    # one D2H: [huber sum, dslog, sq err, eik sum, flag, slog]
    ws.report[:4].copy_(ws.sums[:4])
    ws.report[4:5].copy_(ws.flag.to(torch.float64))
    ws.report[5:6].copy_(params.sharpness_log)
    ws.report_host.copy_(ws.report, non_blocking=True)
    if sampler is not None and state.draw_ahead:  # host rng work under the device step
        before = state._rng.bit_generator.state
        nxt = sampler._draw(m_total, cfg.fg_fraction, state._rng)
        state._ahead = (draw_key, before, state._rng.bit_generator.state, nxt)
    st.synchronize()
    rep = ws.report_host.tolist()
    if rep[4] != 0:
        _raise_divergence(state, int(rep[4]), stepped)
    params.refresh_host_mirror(rep[5])
    c_loss = rep[0] / m_total
    e_loss = rep[3] / P_glob if P_glob > 0 else 0.0
    report = LossReport(step=state.step, color=c_loss, eikonal=e_loss,
                        total=c_loss + cfg.eikonal_weight * e_loss, level=level,
                        psnr=psnr_from_mse(rep[2] / (3.0 * m_total)), sample_count=P_glob)
    state.last_dslog = rep[1] * s
    state.step += 1
    return report


def _raise_divergence(state, bits, stepped):
    """The device flag is set: no parameter or moment was written (the Adam kernels
    check it first), so the step counters advanced by `_apply_gradients` are rolled
    back before raising -- bias correction and checkpoints keep the reference's `t`
    (`trainer.py:158-159` raises before its group's `t` moves)."""
    for n in stepped:
        state.adam[n].t -= 1
    name = next(n for n in _CHECK_ORDER if bits & (1 << _CHECK_ORDER.index(n)))
    raise FloatingPointError(f"divergence: non-finite gradient for {name}")


def _apply_gradients(state, n_active, sharpness, lr_scale=1.0, schedule=True):
    """Divergence check, s_log Adam, then one multi-group Adam launch over
    [sdf_0 | sdf_1 | color_0..2 | tables[:n_active]] (`trainer.py:243-278`).
    `lr_scale` multiplies every group's learning rate (dynamic frames > 0 fine-tune
    with `frame_lr_scale`, `trainer.py:62-68`)."""
    cfg = state.config
    params, ws = state.params, state.ws
    lay = params.layout
    sp = _lib.stream_ptr()
    scale = (lr_factor(state.step, cfg.total_steps, cfg.lr_final_fraction) if schedule else 1.0) * lr_scale
    lr_t, lr_m = cfg.lr_tables * scale, cfg.lr_mlp * scale
    names = ["sdf_0", "sdf_1", "color_0", "color_1", "color_2", "tables"]
    offs = lay.sdf_offs + lay.color_offs + [lay.tables_off]
    lens = [a * b for a, b in lay.sdf_shapes + lay.color_shapes] + [n_active * lay.T * 2]
    lrs = [lr_m] * 5 + [lr_t]
    if n_active == 0:
        names, offs, lens, lrs = names[:5], offs[:5], lens[:5], lrs[:5]
    for n in names:
        state.adam[n].t += 1
    state.adam["sharpness_log"].t += 1
    # one finite check over all fp32 groups; segment k sets bit k, listed in the
    # reference's check order so bit k names _CHECK_ORDER[k]
    chk = [n for n in _CHECK_ORDER[:-1] if n in names]
    idx = [names.index(n) for n in chk]
    _lib.call("ns2b_check_finite", _lib.ptr(ws.grads), _lib.i64_array([offs[i] for i in idx]),
              _lib.i64_array([lens[i] for i in idx]), len(idx), _lib.ptr(ws.flag), sp)
    sl = state.adam["sharpness_log"]
    _lib.call("ns2b_adam_scalar_f64", _lib.ptr(params.sharpness_log), _lib.ptr(ws.sums[1:2]),
              float(sharpness), _lib.ptr(sl.m), _lib.ptr(sl.v), sl.t, lr_m, cfg.adam_beta1,
              cfg.adam_beta2, cfg.adam_eps, _lib.ptr(ws.flag), _lib.ptr(ws.flag),
              _CHECK_ORDER.index("sharpness_log"), sp)
    ts = [state.adam[n].t for n in names]
    _lib.call("ns2b_adam_multi", _lib.ptr(params.flat), _lib.ptr(ws.grads), _lib.ptr(state.m_flat),
              _lib.ptr(state.v_flat), _lib.i64_array(offs), _lib.i64_array(lens),
              _lib.f64_array(lrs), _lib.i64_array(ts), len(names), cfg.adam_beta1,
              cfg.adam_beta2, cfg.adam_eps, _lib.ptr(ws.flag), sp)
    return names + ["sharpness_log"]


def adam_update(state, param, grad, lr, config, name="param", m=None, v=None):
    """One bias-corrected Adam step in place on a contiguous CUDA tensor
    (`trainer.py:152-172`) through `ns2b_adam_step_f32/_f64`; `m`/`v` default to the
    AdamState's buffers (callers updating a leading slice, e.g. the active table levels,
    pass matching views).  Raises FloatingPointError("divergence: ...") on a non-finite
    gradient before touching anything."""
    g = as_device(grad, param.dtype).reshape(-1).contiguous()
    if not bool(torch.isfinite(g).all()):
        raise FloatingPointError(f"divergence: non-finite gradient for {name}")
    m = state.m if m is None else m
    v = state.v if v is None else v
    for t in (param, m, v):
        if not (t.is_cuda and t.is_contiguous()):
            raise ValueError("adam_update: param and moments must be contiguous CUDA tensors")
    state.t += 1
    fn = "ns2b_adam_step_f64" if param.dtype == torch.float64 else "ns2b_adam_step_f32"
    _lib.call(fn, _lib.ptr(param), _lib.ptr(g), _lib.ptr(m), _lib.ptr(v), param.numel(), int(state.t),
              float(lr), float(config.adam_beta1), float(config.adam_beta2), float(config.adam_eps),
              _lib.stream_ptr())


def compute_cotangents(state, batch, rendered, records):
    """Module-API loss + cotangents (`trainer.py:215-240`) for a rendered batch, on the
    device (train_step fuses the same arithmetic into ns2b_composite and the MLP
    kernels): Huber colour loss and its ray cotangent /m, `renderer.backward_cotangents`,
    and the Eikonal loss/cotangent over all P samples.  Returns (color_loss,
    eikonal_loss, total, dl_dcolors (P,3), dl_dsdf (P,), dl_dslog, dl_dn (P,3) or None)."""
    cfg = state.config
    m = batch.count
    r = as_device(rendered, torch.float64).reshape(-1, 3)
    resid = r - as_device(batch.target_colors, torch.float64).reshape(-1, 3)
    if m < 1:
        raise ValueError("need at least one ray")
    delta = cfg.huber_delta
    a = resid.abs()
    c_loss = float(torch.where(a <= delta, 0.5 * resid * resid / delta, a - 0.5 * delta).sum(1).mean())
    dl_dray = torch.where(a <= delta, resid / delta, torch.sign(resid)) / m
    dl_dcolors, dl_dsdf, dl_dslog = renderer.backward_cotangents(records, dl_dray)
    nsamp = records.sample_count
    if nsamp > 0:
        n = records.cache.normals
        norms = torch.linalg.vector_norm(n, dim=1)
        e_loss = float(((norms - 1.0) ** 2).mean())
        dl_dn = (cfg.eikonal_weight * (2.0 * (norms - 1.0) / torch.clamp(norms, min=1e-12))[:, None]
                 * n / nsamp)
    else:
        e_loss, dl_dn = 0.0, None
    return c_loss, e_loss, c_loss + cfg.eikonal_weight * e_loss, dl_dcolors, dl_dsdf, dl_dslog, dl_dn


def apply_gradients(state, grads, dl_dslog, lr_scale=1.0, max_active_level=None):
    """Module-API Adam step (`trainer.py:243-278`) for callers that assemble their own
    FieldGrads (train_step applies the same kernels to its fused gradient buffer):
    `lr_scale` is the full learning-rate factor as in the reference (train_step passes
    the cosine `lr_factor`), levels >= `max_active_level` are skipped, and a
    non-finite gradient raises FloatingPointError("divergence: ...") naming the first
    bad group in the reference's order (here no group has been stepped when it raises;
    the reference has already stepped the groups it checked before the bad one)."""
    params, ws = state.params, state.ws
    na = params.grid.num_levels if max_active_level is None else int(max_active_level)
    if grads.flat is not None:
        ws.grads.copy_(grads.flat)
    else:
        sdf, col, tab = params.layout.views(ws.grads)
        for dst, src in zip(sdf + col + [tab], list(grads.sdf_layers) + list(grads.color_layers)
                            + [grads.tables]):
            dst.copy_(as_device(src, torch.float32).reshape(dst.shape))
    ws.sums[1:2].fill_(float(dl_dslog))
    ws.flag.zero_()
    stepped = _apply_gradients(state, na, 1.0, lr_scale, schedule=False)
    bits = int(ws.flag.item())
    if bits:
        _raise_divergence(state, bits, stepped)
    params.refresh_host_mirror(float(params.sharpness_log.item()))


def masked_psnr(image_a, image_b, mask):
    """`trainer.py:145-149` (host helper)."""
    sel = np.asarray(mask) > 0.5
    if not np.any(sel):
        return 100.0
    return psnr(np.asarray(image_a)[sel], np.asarray(image_b)[sel])


@dataclass
class TrainResult:
    """`trainer.py:313-318`."""
    state: TrainState
    reports: list
    checkpoint_path: object = None
    wall_seconds: float = 0.0


def train_static(dataset, config, out_path=None, time_index=0, state=None, log_every=100):
    """Static training loop (`trainer.py:321-347`): `train_step` until
    `config.total_steps`, reports every `log_every` steps and at the last step, then the
    NS2C checkpoint at `out_path` plus the `.loss.csv` log next to it."""
    import time
    from pathlib import Path

    from . import checkpoint

    if state is None:
        state = TrainState.create(config, aabb=dataset.scene_aabb)
    reports = []
    t0 = time.perf_counter()
    while state.step < config.total_steps:
        rep = train_step(state, dataset, time_index)
        if rep.step % log_every == 0 or rep.step == config.total_steps - 1:
            reports.append(rep)
    wall = time.perf_counter() - t0
    ckpt = None
    if out_path is not None:
        ckpt = Path(out_path)
        checkpoint.save_checkpoint(ckpt, state)
        lines = ["step,color,eikonal,total,lambda,psnr"]
        lines += [f"{r.step},{r.color:.6f},{r.eikonal:.6f},{r.total:.6f},{r.level},{r.psnr:.3f}"
                  for r in reports]
        ckpt.with_suffix(ckpt.suffix + ".loss.csv").write_text("\n".join(lines) + "\n")
    return TrainResult(state, reports, ckpt, wall)


def render_frame(params, occ, frame, level=None, chunk=1 << 18, point_transform=None,
                 dir_transform=None):
    """Full camera view (`trainer.py:350-370`) through `render_rays` in ray chunks
    (rays are independent, so the chunk size does not change the result; the
    reference's 8192 is a host-memory bound).  Returns host (H,W,3) image and (H,W)
    expected depth, fp64 like the reference."""
    level = level if level is not None else params.grid.num_levels
    origins, dirs = scene_io.generate_rays_grid(frame)
    n = origins.shape[0]
    img = np.zeros((n, 3))
    depth = np.zeros(n)
    for s in range(0, n, chunk):
        e = min(s + chunk, n)
        batch = scene_io.RayBatch(origins[s:e], dirs[s:e], np.zeros((e - s, 3)), np.ones(e - s, bool))
        cols, rec = renderer.render_rays(batch, params, occ, level, point_transform=point_transform,
                                         dir_transform=dir_transform)
        img[s:e] = cols.cpu().numpy()
        depth[s:e] = renderer.expected_depth(rec).cpu().numpy()
    return img.reshape(frame.height, frame.width, 3), depth.reshape(frame.height, frame.width)


def evaluate_view(params, occ, frame, level=None, point_transform=None, dir_transform=None):
    """Masked and full-frame PSNR of a rendered view (`trainer.py:373-382`)."""
    img, _ = render_frame(params, occ, frame, level, point_transform=point_transform,
                          dir_transform=dir_transform)
    target = frame.image * frame.mask[:, :, None]
    return {"psnr_masked": masked_psnr(img, target, frame.mask), "psnr_full": psnr(img, target)}
