"""Dynamic-scene hooks against the reference's golden vectors
(tests/golden/dynamic_c1.npz, written by make_golden.py `dynamic`):

* hessian_contract (`_kernels.py:159-206`, `hash_encoding.py:240-254`);
* field_backward(need_input_grads=True) position / view cotangents (`field.py:332-349`);
* update_occupancy / render_rays with point and direction transforms
  (`renderer.py:108-128, 234-264`) under a fixed rigid transform x -> R (x + T).

The oracle is pinned on the CPU; the libns2b kernels are checked on the GPU."""

from __future__ import annotations

from pathlib import Path

import numpy as np
import pytest

import cases
from oracle import field as ofield
from oracle import kernels as ok
from oracle import render as orender
from oracle import scene as oscene
from oracle import train as otrain
from parity import assert_close, assert_exact
from test_oracle_golden import oracle_field_params

GOLD = dict(np.load(Path(__file__).resolve().parent / "golden" / "dynamic_c1.npz"))
R = cases.rodrigues(cases.RIGID_AXIS_ANGLE)


def _hess_inputs(name):
    spec = cases.GRIDS[name]
    L, T = spec["num_levels"], spec["table_size"]
    grid = ohg_grid(spec)
    tables = cases.trained_tables(L, T)
    xn = cases.grid_points(seed=3)
    inv = np.ascontiguousarray(1.0 / grid.aabb_extent, np.float32)
    coeff = np.random.default_rng(17).standard_normal((xn.shape[0], 2 * L)).astype(np.float32)
    return L, grid, tables, xn, inv, coeff


def ohg_grid(spec):
    from oracle import hashgrid as ohg

    return ohg.HashGrid(**spec)


def _ig_inputs(name, lam_index):
    p = oracle_field_params(name)
    x = cases.world_points(seed=5)
    rng = np.random.default_rng(9)
    v = rng.standard_normal((x.shape[0], 3))
    v /= np.linalg.norm(v, axis=1, keepdims=True)
    return p, x, v


def _c1_scene_state():
    ds = oscene.make_synthetic("sphere", views=8, image_size=64, seed=0)
    cfg = otrain.TrainConfig(batch_size=512, num_levels=8, table_size=2**14, seed=0, level_init=8)
    return ds, otrain.TrainState.create(cfg, aabb=ds.scene_aabb)


def _pt(x):
    return cases.rigid_apply(x, R, cases.RIGID_T)


def _dt(v):
    return cases.rigid_apply(v, R)


# ------------------------------------------------------------------ CPU ----
def test_rigid_helper_is_a_rotation():
    assert np.allclose(R @ R.T, np.eye(3), atol=1e-12) and abs(np.linalg.det(R) - 1) < 1e-12
    x = np.random.default_rng(0).standard_normal((5, 3))
    assert np.allclose(_pt(x), (x + np.asarray(cases.RIGID_T)) @ R.T, atol=1e-14)


@pytest.mark.parametrize("name", ["c1", "np2"])
def test_oracle_hessian_bit_exact(name):
    L, grid, tables, xn, inv, coeff = _hess_inputs(name)
    for na in (L, 3):
        out = ok.hessian_contract(xn, tables, grid.resolutions, na, inv, coeff)
        assert_exact(out, GOLD[f"hess_{name}_na{na}"], f"hessian {name} na{na}")


@pytest.mark.parametrize("name", ["c1", "c2"])
def test_oracle_input_grads(name):
    p, x, v = _ig_inputs(name, 0)
    for lam in (p.grid.num_levels, 3):
        k = f"ig_{name}_lam{lam}_"
        c = ofield.eval_field(p, x, v, lam)
        gr = ofield.field_backward(p, c, dl_dc=GOLD[k + "dl_dc"], dl_dd=GOLD[k + "dl_dd"],
                                   dl_dn=GOLD[k + "dl_dn"], need_input_grads=True)
        assert_close(gr.dl_dx, GOLD[k + "dl_dx"], 1e-6, "dl_dx")
        assert_close(gr.dl_dv, GOLD[k + "dl_dv"], 1e-6, "dl_dv")
        gr = ofield.field_backward(p, c, dl_dd=GOLD[k + "dl_dd"], dl_dn=GOLD[k + "dl_dn"],
                                   need_input_grads=True)
        assert_close(gr.dl_dx, GOLD[k + "nocolor_dl_dx"], 1e-6, "dl_dx (no colour)")


def test_oracle_transformed_render():
    ds, st = _c1_scene_state()
    orender.update_occupancy(st.occ, st.params, 8, point_transform=_pt)
    assert_exact(np.packbits(st.occ.bits.reshape(-1)), GOLD["occ_bits"], "occupancy bits")
    assert abs(st.occ.ema.sum() - GOLD["occ_ema_sum"]) <= 1e-9 * abs(GOLD["occ_ema_sum"])
    batch = oscene.RayBatch(GOLD["rt_origins"], GOLD["rt_dirs"], np.zeros((512, 3)), np.zeros(512, bool))
    out, rec = orender.render_rays(batch, st.params, st.occ, 8, point_transform=_pt, dir_transform=_dt)
    assert rec.sample_count == int(GOLD["rt_count"])
    assert_close(out, GOLD["rt_rendered"], 1e-6, "rendered")


# ------------------------------------------------------------------ GPU ----
def _gpu():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    return torch


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["c1", "np2"])
def test_gpu_hessian_contract(name):
    _gpu()
    from paper_2212_05231_b200 import _kernels as pk

    L, grid, tables, xn, inv, coeff = _hess_inputs(name)
    for na in (L, 3):
        out = pk.hessian_contract(xn, tables, grid.resolutions, na, inv, coeff)
        assert_exact(out, GOLD[f"hess_{name}_na{na}"], f"hessian {name} na{na}")


@pytest.mark.gpu
def test_gpu_hessian_module_api():
    torch = _gpu()
    from helpers import product_params_from_oracle

    from oracle import hashgrid as ohg
    from paper_2212_05231_b200 import hash_encoding as pe

    p = oracle_field_params("c2")
    pp = product_params_from_oracle(p)
    x = cases.world_points(seed=5)
    coeff = np.random.default_rng(3).standard_normal((x.shape[0], 32)).astype(np.float32)
    for lam in (16, 5):
        ref = ohg.hessian_contract(p.grid, x, lam, coeff)
        got = pe.hessian_contract(pp.grid, torch.from_numpy(x).cuda(), lam, torch.from_numpy(coeff).cuda())
        assert_exact(got.cpu().numpy(), ref, f"hessian lam {lam}")


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["c1", "c2"])
def test_gpu_input_grads(name):
    torch = _gpu()
    from helpers import product_params_from_oracle

    from paper_2212_05231_b200 import field as pf

    p, x, v = _ig_inputs(name, 0)
    pp = product_params_from_oracle(p)
    for lam in (p.grid.num_levels, 3):
        k = f"ig_{name}_lam{lam}_"
        c = pf.eval_field(pp, torch.from_numpy(x).cuda(), torch.from_numpy(v).cuda(), lam)
        gr = pf.field_backward(pp, c, dl_dc=GOLD[k + "dl_dc"], dl_dd=GOLD[k + "dl_dd"],
                               dl_dn=GOLD[k + "dl_dn"], need_input_grads=True)
        assert_close(gr.dl_dx.cpu().numpy(), GOLD[k + "dl_dx"], 1e-3, f"{k}dl_dx")
        assert_close(gr.dl_dv.cpu().numpy(), GOLD[k + "dl_dv"], 1e-3, f"{k}dl_dv")
        gr = pf.field_backward(pp, c, dl_dd=GOLD[k + "dl_dd"], dl_dn=GOLD[k + "dl_dn"],
                               need_input_grads=True)
        assert_close(gr.dl_dx.cpu().numpy(), GOLD[k + "nocolor_dl_dx"], 1e-3, f"{k}dl_dx no colour")
        assert float(gr.dl_dv.abs().max()) == 0.0


@pytest.mark.gpu
def test_gpu_transformed_occupancy_and_render():
    torch = _gpu()
    from helpers import product_state_from_oracle

    from paper_2212_05231_b200 import renderer as pr

    ds, ost = _c1_scene_state()
    st = product_state_from_oracle(ost)
    pr.update_occupancy(st.occ, st.params, 8, point_transform=_pt)
    bits = st.occ.bits.cpu().numpy().astype(bool).reshape(-1)
    assert_exact(np.packbits(bits), GOLD["occ_bits"], "occupancy bits")
    ema = float(st.occ.ema.sum())
    assert abs(ema - GOLD["occ_ema_sum"]) <= 1e-6 * abs(GOLD["occ_ema_sum"])
    batch = oscene.RayBatch(GOLD["rt_origins"], GOLD["rt_dirs"], np.zeros((512, 3)), np.zeros(512, bool))
    out, rec = pr.render_rays(batch, st.params, st.occ, 8, point_transform=_pt, dir_transform=_dt)
    assert rec.sample_count == int(GOLD["rt_count"])
    assert_close(out.cpu().numpy(), GOLD["rt_rendered"], 1e-3, "rendered")
    # the cache the transformed render hands back drives the input-gradient kernel
    P = rec.sample_count
    g = torch.Generator(device="cuda").manual_seed(0)
    dl_dc = torch.randn((P, 3), generator=g, device="cuda")
    from paper_2212_05231_b200 import field as pf

    gr = pf.field_backward(st.params, rec.cache, dl_dc=dl_dc, need_input_grads=True)
    assert bool(torch.isfinite(gr.dl_dx).all()) and bool(torch.isfinite(gr.dl_dv).all())
