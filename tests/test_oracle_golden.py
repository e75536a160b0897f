"""Pin the CPU oracle (oracle/) against golden vectors produced by the reference
itself (tests/golden/make_golden.py).  CPU only."""

from __future__ import annotations

import json
from pathlib import Path

import numpy as np
import pytest

import cases
from oracle import field as ofield
from oracle import hashgrid as ohg
from oracle import kernels as ok
from oracle import mlp as omlp
from oracle import render as orender
from oracle import scene as oscene
from oracle import train as otrain
from parity import assert_close, assert_exact

GOLD = Path(__file__).resolve().parent / "golden"


def load(name):
    return dict(np.load(GOLD / name, allow_pickle=False))


def test_kat():
    k = json.loads((GOLD / "kat.json").read_text())
    assert ohg.level_resolutions(14, 16, 2048) == k["level_resolutions_14_16_2048"]
    assert ohg.level_resolutions(16, 16, 2048) == k["level_resolutions_16_16_2048"]
    assert ohg.level_resolutions(8, 16, 2048) == k["level_resolutions_8_16_2048"]
    gd = ohg.HashGrid(num_levels=4, table_size=2**19)
    g15 = ohg.HashGrid(num_levels=4, table_size=2**15)
    assert ohg.hash_index([0, 0, 0], 0, gd) == k["hash_dense_000"] == 0
    assert ohg.hash_index([1, 0, 0], 0, gd) == k["hash_dense_100"] == 1
    assert ohg.hash_index([3, 5, 7], 3, g15) == k["hash_357_T2p15"] == 1381
    cdf, dens = orender.sdf_transforms(1.0, np.array([0.0]))
    assert [cdf[0], dens[0]] == k["sdf_transforms_s1_f0"]
    assert orender.sdf_transforms(1.0, np.array([0.5]))[0][0] == k["sdf_transforms_s1_f05"]
    assert orender.alpha(np.array([0.5]), np.array([-0.5]), 1.0)[0] == k["alpha_p05_m05"]
    assert orender.alpha(np.array([-0.5]), np.array([0.5]), 1.0)[0] == k["alpha_m05_p05"] == 0
    w = orender.composite([0.5, 0.5], [[1, 0, 0], [0, 1, 0]])[1]
    assert w.tolist() == k["composite_05_05_w"] == [0.5, 0.25]
    assert float(otrain.huber(np.array(1.0), 0.1)) == k["huber_1_01"]
    cfg = otrain.TrainConfig(total_steps=15000, num_levels=14)
    for s, lv in k["level_schedule"].items():
        assert otrain.level_schedule(int(s), cfg) == lv
    assert otrain.psnr(np.zeros((4, 4)), np.full((4, 4), 0.1)) == k["psnr_uniform_01"]
    assert [float(otrain.lr_factor(s, 100, 0.1)) for s in (0, 25, 50, 100, 150)] == k["lr_factor"]
    gnp = ohg.HashGrid(num_levels=6, min_resolution=16, max_resolution=512, table_size=393217)
    cells = [[5, 9, 200], [511, 3, 77], [100, 200, 300], [1, 1, 1]]
    assert [ohg.hash_index(c, 5, gnp) for c in cells] == k["hash_np2_python"]


@pytest.mark.parametrize("name", list(cases.GRIDS))
def test_kernels_bit_exact(name):
    gold = load(f"kernels_{name}.npz")
    spec = cases.GRIDS[name]
    L, T = spec["num_levels"], spec["table_size"]
    grid = ohg.HashGrid(**spec)
    tables = cases.trained_tables(L, T)
    xn = cases.grid_points(seed=3)
    inv = np.ascontiguousarray(1.0 / grid.aabb_extent, np.float32)
    for na in (L, 3):
        k = f"na{na}_"
        feats, jac, cidx, cw, cdw = ok.interp_full(xn, tables, grid.resolutions, na, inv)
        assert_exact(cidx.astype(np.int32), gold[k + "cidx"], "cidx")
        assert_exact(feats, gold[k + "feats"], "feats")
        assert_exact(jac, gold[k + "jac"], "jac")
        assert_exact(cw, gold[k + "cw"], "cw")
        assert_exact(cdw, gold[k + "cdw"], "cdw")
        assert_exact(ok.interp_features(xn, tables, grid.resolutions, na), feats, "features")
        rng = np.random.default_rng(11)
        dfeat = rng.standard_normal((xn.shape[0], L * 2)).astype(np.float32)
        u = rng.standard_normal((xn.shape[0], L * 2, 3)).astype(np.float32)
        g1 = np.zeros_like(tables)
        ok.scatter_first(g1, cidx, cw, dfeat, na)
        g2 = np.zeros_like(tables)
        ok.scatter_second(g2, cidx, cdw, u, na)
        for tag, g in (("g1", g1), ("g2", g2)):
            assert_exact(cases.level_norms(g), gold[k + tag + "_norms"], tag)
            assert_exact(g.reshape(-1)[gold[k + tag + "_idx"]], gold[k + tag + "_val"], tag)


def test_np2_kernel_hash_vs_python_hash():
    """The kernel's 64-bit-product hash (kept by the oracle) differs from the
    32-bit-masked python helper for non-power-of-two T, as in the reference."""
    k = json.loads((GOLD / "kat.json").read_text())
    gnp = ohg.HashGrid(num_levels=6, min_resolution=16, max_resolution=512, table_size=393217)
    xn = np.array([[5, 9, 200], [511, 3, 77], [100, 200, 300], [1, 1, 1]], np.float32) / 512.0
    # lower-cell rule: a point exactly on a vertex c lands in cell c-1 with frac 1,
    # so corner 7 (upper) of that cell is vertex c.
    _, _, cidx, cw, _ = ok.interp_full(xn, gnp.tables, gnp.resolutions, 6,
                                       np.full(3, 0.5, np.float32))
    got = []
    for p in range(4):
        hit = [int(cidx[p, 5, c]) for c in range(8) if cw[p, 5, c] == 1.0]
        got.append(hit[0])
    assert got == k["hash_np2_kernel"]


def test_mlp_theorem1():
    gold = load("mlp.npz")
    for depth in (1, 2, 3):
        k = f"d{depth}_"
        w = omlp.MlpWeights([gold[k + f"w{i}"] for i in range(depth)])
        y, tr = omlp.forward(w, gold[k + "x"])
        assert_close(y, gold[k + "y"], 1e-12, "y")
        g2 = omlp.backward_second(w, tr, gold[k + "m"])
        g2r = omlp.backward_second_row(w, tr, 0, gold[k + "mv"])
        g1, dx = omlp.backward_first(w, tr, gold[k + "dy"])
        assert_close(dx, gold[k + "dx"], 1e-12, "dx")
        for i in range(depth):
            assert_close(g2[i], gold[k + f"g2_{i}"], 1e-12, "g2")
            assert_close(g2r[i], gold[k + f"g2r_{i}"], 1e-12, "g2r")
            assert_close(g1[i], gold[k + f"g1_{i}"], 1e-12, "g1")


def oracle_field_params(name, seed=0):
    spec = cases.GRIDS[name]
    cfg = ofield.FieldConfig(num_levels=spec["num_levels"], table_size=spec["table_size"],
                             min_resolution=spec["min_resolution"],
                             max_resolution=spec["max_resolution"])
    rng = np.random.default_rng(seed)
    p = ofield.FieldParams.create(cfg, rng)
    ofield.sal_geometry_init(p, 0.5, rng)
    p.grid.tables[:] = cases.trained_tables(spec["num_levels"], spec["table_size"])
    return p


@pytest.mark.parametrize("name", ["c1", "c2"])
def test_field(name):
    gold = load(f"field_{name}.npz")
    p = oracle_field_params(name)
    x = cases.world_points(seed=5)
    rng = np.random.default_rng(9)
    v = rng.standard_normal((x.shape[0], 3))
    v /= np.linalg.norm(v, axis=1, keepdims=True)
    for lam in (p.grid.num_levels, 3):
        k = f"lam{lam}_"
        c = ofield.eval_field(p, x, v, lam)
        for key, val in (("d", c.d), ("g", c.g), ("normals", c.normals), ("colors", c.colors),
                         ("j_d", c.d_row_jacobian)):
            assert_close(val, gold[k + key], 1e-6, key)
        dl_dc = rng.standard_normal((x.shape[0], 3))
        dl_dd = rng.standard_normal(x.shape[0])
        dl_dn = rng.standard_normal((x.shape[0], 3)).astype(np.float32)
        assert_exact(dl_dn, gold[k + "dl_dn"], "cotangent replay")
        gr = ofield.field_backward(p, c, dl_dc=dl_dc, dl_dd=dl_dd, dl_dn=dl_dn)
        for i, g in enumerate(gr.sdf_layers):
            assert_close(g, gold[k + f"gsdf{i}"], 1e-6, f"gsdf{i}")
        for i, g in enumerate(gr.color_layers):
            assert_close(g, gold[k + f"gcol{i}"], 1e-6, f"gcol{i}")
        assert_close(cases.level_norms(gr.tables), gold[k + "gtab_norms"], 1e-6, "gtab norms")
        assert_close(gr.tables.reshape(-1)[gold[k + "gtab_idx"]], gold[k + "gtab_val"], 1e-6,
                     "gtab")
    assert_close(ofield.field_sdf_only(p, x, p.grid.num_levels), gold["sdf_only"], 1e-6)


def test_occupancy():
    gold = load("occupancy_c1.npz")
    st = otrain.TrainState.create(otrain.TrainConfig(num_levels=8, table_size=2**14, seed=0))
    orender.update_occupancy(st.occ, st.params, 8)
    assert_exact(np.packbits(st.occ.bits.reshape(-1)), gold["bits"], "occupancy bits")
    assert_close(st.occ.ema.reshape(-1)[gold["ema_idx"]], gold["ema_val"], 1e-9, "ema")


def make_scene(spec):
    return oscene.make_synthetic(spec["preset"], views=spec["views"], seed=spec["seed"],
                                 image_size=spec["image_size"])


@pytest.mark.parametrize("name", list(cases.STEP_CASES))
def test_train_step(name):
    gold = load(f"step_{name}.npz")
    spec = cases.STEP_CASES[name]
    ds = make_scene(spec["scene"])
    st = otrain.TrainState.create(otrain.TrainConfig(**spec["cfg"]), aabb=ds.scene_aabb)
    for s in range(spec["steps"]):
        k = f"s{s}_"
        tr = {}
        rep = otrain.train_step(st, ds, trace=tr)
        b, rec = tr["batch"], tr["records"]
        assert tr["level"] == int(gold[k + "level"])
        assert_exact(np.packbits(st.occ.bits.reshape(-1)), gold[k + "occ_bits"], "bits")
        assert_exact(b.origins, gold[k + "origins"], "origins")
        assert_exact(b.directions, gold[k + "dirs"], "dirs")
        assert_exact(b.target_colors, gold[k + "targets"], "targets")
        assert_exact(rec.ray_ids.astype(np.int32), gold[k + "ray_ids"], "ray_ids")
        assert_exact(rec.t, gold[k + "t"], "t")
        assert_exact(rec.interval_first.astype(np.int32), gold[k + "interval_first"], "intervals")
        for key, val in (("sdf", rec.sdf), ("colors", rec.sample_colors),
                         ("normals", rec.cache.normals), ("alphas", rec.alphas),
                         ("weights", rec.weights), ("transmittance", rec.transmittance),
                         ("rendered", tr["rendered"]), ("dl_dc", tr["dl_dc"]),
                         ("dl_dsdf", tr["dl_dsdf"]), ("dl_dn", tr["dl_dn"])):
            assert_close(val, gold[k + key], 1e-6, key)
        assert_close(np.array([rep.color, rep.eikonal, rep.total]), gold[k + "losses"], 1e-6)
        assert_close(tr["dl_dslog"], gold[k + "dl_dslog"], 1e-6, "dslog")
        assert abs(rep.psnr - float(gold[k + "psnr"])) < 1e-6
        g = tr["grads"]
        for i, a in enumerate(g.sdf_layers):
            assert_close(a, gold[k + f"gsdf{i}"], 1e-6, f"gsdf{i}")
        for i, a in enumerate(g.color_layers):
            assert_close(a, gold[k + f"gcol{i}"], 1e-6, f"gcol{i}")
        assert_close(cases.level_norms(g.tables), gold[k + "gtab_norms"], 1e-6, "gtab norms")
        assert_close(g.tables.reshape(-1)[gold[k + "gtab_idx"]], gold[k + "gtab_val"], 1e-6)
        p = st.params
        assert_close(p.grid.tables.reshape(-1)[gold[k + "new_tab_idx"]], gold[k + "new_tab_val"],
                     1e-6, "new tables")
        for i, h in enumerate(p.sdf_net.layers):
            assert_close(h, gold[k + f"new_sdf{i}"], 1e-6, f"new_sdf{i}")
        for i, h in enumerate(p.color_net.layers):
            assert_close(h, gold[k + f"new_col{i}"], 1e-6, f"new_col{i}")
        assert_close(p.sharpness_log, gold[k + "new_slog"], 1e-12, "slog")


def check_init(gold, name, resolutions, sdf, col, slog, tables, aabb, occ, rng):
    """TrainState.create parity against the reference's golden init (bit-exact)."""
    k = name + "_"
    assert_exact(np.asarray(resolutions, np.int64), gold[k + "resolutions"], "resolutions")
    for i, h in enumerate(sdf):
        assert_exact(np.asarray(h), gold[k + f"sdf{i}"], f"sdf{i}")
    for i, h in enumerate(col):
        assert_exact(np.asarray(h), gold[k + f"col{i}"], f"col{i}")
    assert_exact(np.asarray(slog, np.float64).reshape(-1), gold[k + "slog"].reshape(-1), "s_log")
    tables = np.ascontiguousarray(tables, np.float32)
    assert cases.sha256(tables) == str(gold[k + "tables_sha256"]), "tables differ (sha256)"
    assert_exact(tables.reshape(-1)[gold[k + "tables_idx"]], gold[k + "tables_val"], "tables sample")
    assert_exact(np.asarray(aabb, np.float64), gold[k + "aabb"], "aabb")
    assert_exact(np.asarray(occ, np.float64), gold[k + "occ"], "occupancy grid")
    assert_exact(rng.integers(0, 2**62, size=8), gold[k + "rng_next"], "rng stream after init")


@pytest.mark.parametrize("name", list(cases.INIT_CASES))
def test_oracle_init(name):
    """`trainer.py:192-212` / `field.py:81-165` / `hash_encoding.py:31-45`: the oracle's
    seeded TrainState.create equals the reference's, bit for bit."""
    gold = load("init.npz")
    st = otrain.TrainState.create(otrain.TrainConfig(**cases.INIT_CASES[name]))
    p = st.params
    check_init(gold, name, p.grid.resolutions, p.sdf_net.layers, p.color_net.layers, p.sharpness_log,
               p.grid.tables, [p.grid.aabb_min, p.grid.aabb_min + p.grid.aabb_extent],
               [st.occ.resolution, st.occ.threshold, st.occ.step_size], st.rng)


@pytest.mark.parametrize("name", list(cases.INIT_CASES))
def test_product_level_resolutions(name):
    """The product's `hash_encoding.level_resolutions` (host, no device needed)."""
    from paper_2212_05231_b200 import hash_encoding as pe

    kw = cases.INIT_CASES[name]
    res = pe.level_resolutions(kw["num_levels"], 16, kw.get("max_resolution", 2048))
    assert_exact(np.asarray(res, np.int64), load("init.npz")[name + "_resolutions"], "resolutions")
