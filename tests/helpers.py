"""Test helpers: convert oracle (numpy) objects into product (device) objects."""

from __future__ import annotations

import numpy as np
import torch


def product_params_from_oracle(op):
    from paper_2212_05231_b200 import field as pf
    from paper_2212_05231_b200 import hash_encoding as pe
    from paper_2212_05231_b200.relu_mlp import MlpWeights

    g = op.grid
    lo = g.aabb_min
    hi = g.aabb_min + g.aabb_extent
    grid = pe.MultiResHashGrid(g.num_levels, int(g.resolutions[0]), int(g.resolutions[-1]), 2,
                               g.table_size, (tuple(lo), tuple(hi)),
                               tables=torch.from_numpy(g.tables.copy()).cuda())
    grid.resolutions = g.resolutions.copy()
    return pf.SdfFieldParams(grid, MlpWeights(op.sdf_net.layers), MlpWeights(op.color_net.layers),
                             op.sharpness_log.copy())


def np_(t):
    if isinstance(t, torch.Tensor):
        return t.detach().cpu().numpy()
    return np.asarray(t)


def product_state_from_oracle(ost, config_cls=None):
    """Product TrainState with the oracle state's parameters, occupancy and config."""
    from paper_2212_05231_b200 import renderer as pr
    from paper_2212_05231_b200 import trainer as pt

    cfg = pt.TrainConfig(**{k: getattr(ost.config, k) for k in vars(ost.config)})
    params = product_params_from_oracle(ost.params)
    occ = pr.OccupancyGrid(ost.occ.resolution, (tuple(ost.occ.lo), tuple(ost.occ.hi)),
                           ost.occ.threshold)
    occ.set_bits(ost.occ.bits)
    occ.ema.copy_(torch.from_numpy(ost.occ.ema))
    st = pt.TrainState(params, occ, cfg, rng=None, step=ost.step)
    return st


def sync_product_from_oracle(pst, ost):
    """Copy the oracle state's parameters, Adam moments and step counters into the
    product state, so the next step starts from identical inputs on both sides."""
    pp, op = pst.params, ost.params
    pp.grid.tables.copy_(torch.from_numpy(np.ascontiguousarray(op.grid.tables)))
    for dst, src in zip(list(pp.sdf_net.layers) + list(pp.color_net.layers),
                        list(op.sdf_net.layers) + list(op.color_net.layers)):
        dst.copy_(torch.from_numpy(np.ascontiguousarray(src)))
    slog = float(np.asarray(op.sharpness_log).ravel()[0])
    pp.sharpness_log.fill_(slog)
    pp.refresh_host_mirror(slog)
    lay = pp.layout
    for buf, key in ((pst.m_flat, "m"), (pst.v_flat, "v")):
        sdf, col, tab = lay.views(buf)
        tab.copy_(torch.from_numpy(getattr(ost.adam["tables"], key)))
        for i, d in enumerate(sdf):
            d.copy_(torch.from_numpy(getattr(ost.adam[f"sdf_{i}"], key)))
        for i, d in enumerate(col):
            d.copy_(torch.from_numpy(getattr(ost.adam[f"color_{i}"], key)))
    for name, a in ost.adam.items():
        pst.adam[name].t = a.t
    sl = pst.adam["sharpness_log"]
    sl.m.fill_(float(np.asarray(ost.adam["sharpness_log"].m).ravel()[0]))
    sl.v.fill_(float(np.asarray(ost.adam["sharpness_log"].v).ravel()[0]))
    pst.step = ost.step
