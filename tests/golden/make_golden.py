"""Generate golden vectors by running the REFERENCE (`hashsdf`, imported from
/root/reference/pkg/src) on the seeded cases of cases.py.

Run in the build container only (the reference does not travel to the GPU box):
    python tests/golden/make_golden.py
Outputs tests/golden/*.npz and kat.json (committed).  The train-step fixtures are
produced by calling the reference's own functions in `trainer.train_step` order
(`trainer.py:281-310`) so intermediates can be captured; the script asserts that
the real `trainer.train_step` on a copy of the state lands on identical parameters.
"""

from __future__ import annotations

import copy
import json
import sys
import tempfile
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg/src")
sys.path.insert(0, str(REF))
sys.path.insert(0, str(Path(__file__).resolve().parent))

import cases  # noqa: E402
from hashsdf import _kernels, field, hash_encoding, relu_mlp, renderer, scene_io, trainer  # noqa: E402

OUT = Path(__file__).resolve().parent


def kat():
    g15 = hash_encoding.MultiResHashGrid(num_levels=4, table_size=2**15)
    gd = hash_encoding.MultiResHashGrid(num_levels=4, table_size=2**19)
    cfg = trainer.TrainConfig(total_steps=15000, num_levels=14)
    out = {
        "level_resolutions_14_16_2048": hash_encoding.level_resolutions(14, 16, 2048),
        "level_resolutions_16_16_2048": hash_encoding.level_resolutions(16, 16, 2048),
        "level_resolutions_8_16_2048": hash_encoding.level_resolutions(8, 16, 2048),
        "hash_dense_000": hash_encoding.hash_index([0, 0, 0], 0, gd),
        "hash_dense_100": hash_encoding.hash_index([1, 0, 0], 0, gd),
        "hash_357_T2p15": hash_encoding.hash_index([3, 5, 7], 3, g15),
        "sdf_transforms_s1_f0": [float(v) for v in renderer.sdf_transforms(1.0, np.array([0.0]))],
        "sdf_transforms_s1_f05": float(renderer.sdf_transforms(1.0, np.array([0.5]))[0][0]),
        "alpha_p05_m05": float(renderer.alpha(np.array([0.5]), np.array([-0.5]), 1.0)[0]),
        "alpha_m05_p05": float(renderer.alpha(np.array([-0.5]), np.array([0.5]), 1.0)[0]),
        "composite_05_05_w": renderer.composite([0.5, 0.5], [[1, 0, 0], [0, 1, 0]])[1].tolist(),
        "huber_1_01": float(trainer.huber(np.array(1.0), 0.1)),
        "level_schedule": {str(s): trainer.level_schedule(s, cfg) for s in (0, 374, 375, 4500)},
        "psnr_uniform_01": trainer.psnr(np.zeros((4, 4)), np.full((4, 4), 0.1)),
        "cell_and_frac": {f"{t}_{n}": list(_kernels._cell_and_frac(t, n))
                          for t, n in ((8.0, 16), (0.0, 16), (16.0, 16), (3.25, 16))},
        "lr_factor": [float(trainer.lr_factor(s, 100, 0.1)) for s in (0, 25, 50, 100, 150)],
    }
    # python hash_index masks to 32 bits; the kernel keeps 64-bit products.
    gnp = hash_encoding.MultiResHashGrid(num_levels=6, min_resolution=16, max_resolution=512,
                                         table_size=393217)
    cells = [[5, 9, 200], [511, 3, 77], [100, 200, 300], [1, 1, 1]]
    out["hash_np2_python"] = [hash_encoding.hash_index(c, 5, gnp) for c in cells]
    out["hash_np2_kernel"] = [int(_kernels._corner_index(c[0], c[1], c[2], 512, 393217))
                              for c in cells]
    (OUT / "kat.json").write_text(json.dumps(out, indent=1, sort_keys=True))


def kernels_case(name):
    spec = cases.GRIDS[name]
    L, T = spec["num_levels"], spec["table_size"]
    grid = hash_encoding.MultiResHashGrid(**spec)
    tables = cases.trained_tables(L, T)
    xn = cases.grid_points(seed=3)
    inv = np.ascontiguousarray(1.0 / grid.aabb_extent, np.float32)
    res = {}
    for na in (L, 3):
        feats, jac, cidx, cw, cdw = _kernels.interp_full(xn, tables, grid.resolutions, na, inv)
        f_only = _kernels.interp_features(xn, tables, grid.resolutions, na)
        assert np.array_equal(f_only, feats)
        rng = np.random.default_rng(11)
        dfeat = rng.standard_normal((xn.shape[0], L * 2)).astype(np.float32)
        u = rng.standard_normal((xn.shape[0], L * 2, 3)).astype(np.float32)
        g1 = np.zeros_like(tables)
        _kernels.scatter_first(g1, cidx, cw, dfeat, na)
        g2 = np.zeros_like(tables)
        _kernels.scatter_second(g2, cidx, cdw, u, na)
        k = f"na{na}_"
        res[k + "feats"] = feats
        res[k + "jac"] = jac
        res[k + "cidx"] = cidx.astype(np.int32)
        res[k + "cw"] = cw
        res[k + "cdw"] = cdw
        for tag, g in (("g1", g1), ("g2", g2)):
            res[k + tag + "_norms"] = cases.level_norms(g)
            res[k + tag + "_idx"], res[k + tag + "_val"] = cases.sparse_sample(g)
    np.savez_compressed(OUT / f"kernels_{name}.npz", **res)


def _field_params(name, seed=0):
    spec = cases.GRIDS[name]
    cfg = field.FieldConfig(num_levels=spec["num_levels"], table_size=spec["table_size"],
                            min_resolution=spec["min_resolution"],
                            max_resolution=spec["max_resolution"])
    rng = np.random.default_rng(seed)
    p = field.SdfFieldParams.create(cfg, rng)
    field.sal_geometry_init(p, 0.5, rng)
    p.grid.tables[:] = cases.trained_tables(spec["num_levels"], spec["table_size"])
    return p


def field_case(name):
    p = _field_params(name)
    x = cases.world_points(seed=5)
    rng = np.random.default_rng(9)
    v = rng.standard_normal((x.shape[0], 3))
    v /= np.linalg.norm(v, axis=1, keepdims=True)
    res = {}
    for lam in (p.grid.num_levels, 3):
        cache = field.eval_field(p, x, v, lam)
        dl_dc = rng.standard_normal((x.shape[0], 3))
        dl_dd = rng.standard_normal(x.shape[0])
        dl_dn = rng.standard_normal((x.shape[0], 3)).astype(np.float32)
        gr = field.field_backward(p, cache, dl_dc=dl_dc, dl_dd=dl_dd, dl_dn=dl_dn)
        k = f"lam{lam}_"
        res.update({k + "d": cache.d, k + "g": cache.g, k + "normals": cache.normals,
                    k + "colors": cache.colors, k + "j_d": cache.d_row_jacobian,
                    k + "dl_dc": dl_dc, k + "dl_dd": dl_dd, k + "dl_dn": dl_dn})
        for i, g in enumerate(gr.sdf_layers):
            res[k + f"gsdf{i}"] = g
        for i, g in enumerate(gr.color_layers):
            res[k + f"gcol{i}"] = g
        res[k + "gtab_norms"] = cases.level_norms(gr.tables)
        res[k + "gtab_idx"], res[k + "gtab_val"] = cases.sparse_sample(gr.tables)
        if lam == p.grid.num_levels:
            # the field's own lean SDF path (renderer.py:131-142)
            res["sdf_only"] = renderer.field_sdf_only(p, x, lam)
    np.savez_compressed(OUT / f"field_{name}.npz", **res)


def _state_snapshot(st):
    p = st.params
    return {"tables": p.grid.tables.copy(), "sdf": [h.copy() for h in p.sdf_net.layers],
            "color": [h.copy() for h in p.color_net.layers], "slog": p.sharpness_log.copy()}


def step_case(name):
    spec = cases.STEP_CASES[name]
    with tempfile.TemporaryDirectory() as td:
        sc = spec["scene"]
        ds = scene_io.make_synthetic(sc["preset"], td, views=sc["views"], seed=sc["seed"],
                                     image_size=sc["image_size"])
    cfg = trainer.TrainConfig(**spec["cfg"])
    st = trainer.TrainState.create(cfg, aabb=ds.scene_aabb)
    twin = copy.deepcopy(st)
    res = {}
    for s in range(spec["steps"]):
        k = f"s{s}_"
        level = trainer.level_schedule(st.step, cfg)
        if st.step % cfg.occupancy_update_every == 0:
            renderer.update_occupancy(st.occ, st.params, level)
        res[k + "occ_bits"] = np.packbits(st.occ.bits.reshape(-1))
        before = _state_snapshot(st)
        batch = scene_io.sample_ray_batch(ds, 0, cfg.batch_size, cfg.fg_fraction, st.rng)
        rendered, rec = renderer.render_rays(batch, st.params, st.occ, level)
        c_loss, e_loss, total, dl_dc, dl_dd, dl_dslog, dl_dn = trainer.compute_cotangents(
            st, batch, rendered, rec)
        gr = field.field_backward(st.params, rec.cache, dl_dc=dl_dc, dl_dd=dl_dd, dl_dn=dl_dn)
        scale = trainer.lr_factor(st.step, cfg.total_steps, cfg.lr_final_fraction)
        trainer.apply_gradients(st, gr, dl_dslog, lr_scale=scale, max_active_level=level)
        st.step += 1
        twin_rep = trainer.train_step(twin, ds)
        assert np.array_equal(twin.params.grid.tables, st.params.grid.tables)
        assert all(np.array_equal(a, b) for a, b in zip(twin.params.sdf_net.layers,
                                                        st.params.sdf_net.layers))
        assert twin_rep.sample_count == rec.sample_count
        res.update({
            k + "level": level, k + "origins": batch.origins, k + "dirs": batch.directions,
            k + "targets": batch.target_colors, k + "ray_ids": rec.ray_ids.astype(np.int32),
            k + "t": rec.t, k + "sdf": rec.sdf, k + "colors": rec.sample_colors,
            k + "normals": rec.cache.normals, k + "alphas": rec.alphas, k + "weights": rec.weights,
            k + "interval_first": rec.interval_first.astype(np.int32),
            k + "transmittance": rec.transmittance, k + "rendered": rendered,
            k + "losses": np.array([c_loss, e_loss, total]), k + "dl_dc": dl_dc,
            k + "dl_dsdf": dl_dd, k + "dl_dslog": dl_dslog, k + "dl_dn": dl_dn,
            k + "psnr": twin_rep.psnr, k + "lr_scale": scale,
        })
        for i, g in enumerate(gr.sdf_layers):
            res[k + f"gsdf{i}"] = g
        for i, g in enumerate(gr.color_layers):
            res[k + f"gcol{i}"] = g
        res[k + "gtab_norms"] = cases.level_norms(gr.tables)
        res[k + "gtab_idx"], res[k + "gtab_val"] = cases.sparse_sample(gr.tables)
        after = _state_snapshot(st)
        dtab = after["tables"].astype(np.float64) - before["tables"]
        res[k + "dtab_norms"] = cases.level_norms(dtab)
        res[k + "new_tab_idx"], _ = cases.sparse_sample(dtab, seed=13)
        res[k + "new_tab_val"] = after["tables"].reshape(-1)[res[k + "new_tab_idx"]]
        for i, h in enumerate(after["sdf"]):
            res[k + f"new_sdf{i}"] = h
        for i, h in enumerate(after["color"]):
            res[k + f"new_col{i}"] = h
        res[k + "new_slog"] = after["slog"]
    np.savez_compressed(OUT / f"step_{name}.npz", **res)


def mlp_case():
    """Theorem 1 on small fp64 nets: analytic general-M and row variants."""
    rng = np.random.default_rng(21)
    res = {}
    for depth in (1, 2, 3):
        dims = [7] + [9] * (depth - 1) + [4]
        w = relu_mlp.MlpWeights.random(dims, rng, dtype=np.float64)
        x = rng.standard_normal((16, 7))
        y, tr = relu_mlp.forward(w, x)
        m = rng.standard_normal((16, 4, 7))
        g2 = relu_mlp.backward_second(w, tr, m)
        mv = rng.standard_normal((16, 7))
        g2r = relu_mlp.backward_second_row(w, tr, 0, mv)
        dy = rng.standard_normal((16, 4))
        g1, dx = relu_mlp.backward_first(w, tr, dy)
        k = f"d{depth}_"
        res.update({k + "x": x, k + "y": y, k + "m": m, k + "mv": mv, k + "dy": dy, k + "dx": dx})
        for i, h in enumerate(w.layers):
            res[k + f"w{i}"] = h
            res[k + f"g2_{i}"] = g2[i]
            res[k + f"g2r_{i}"] = g2r[i]
            res[k + f"g1_{i}"] = g1[i]
    np.savez_compressed(OUT / "mlp.npz", **res)


def occupancy_case():
    """update_occupancy on the config-1 SAL init (renderer.py:108-128)."""
    cfg = trainer.TrainConfig(num_levels=8, table_size=2**14, seed=0)
    st = trainer.TrainState.create(cfg)
    renderer.update_occupancy(st.occ, st.params, 8)
    ema = st.occ.ema.reshape(-1)
    idx = np.sort(np.random.default_rng(3).choice(ema.size, 4000, replace=False))
    np.savez_compressed(OUT / "occupancy_c1.npz", bits=np.packbits(st.occ.bits.reshape(-1)),
                        ema_idx=idx, ema_val=ema[idx],
                        ema_sum=ema.sum(), frac=st.occ.bits.mean())


def checkpoint_case():
    """NS2C checkpoint (checkpoint.py:76-114) of a small trained state, written by the
    reference itself: the byte-level fixture for the checkpoint reader/writer."""
    from hashsdf import checkpoint

    with tempfile.TemporaryDirectory() as td:
        ds = scene_io.make_synthetic("sphere", td, views=4, image_size=32, seed=0)
    cfg = trainer.TrainConfig(batch_size=64, num_levels=4, table_size=2**10, seed=0,
                              occupancy_resolution=16, level_init=4)
    st = trainer.TrainState.create(cfg, aabb=ds.scene_aabb)
    for _ in range(2):
        trainer.train_step(st, ds)
    checkpoint.save_checkpoint(OUT / "ckpt_small.ns2c", st, extra_sections=[(b"XTRA", b"kept")])


def dynamic_case():
    """Dynamic-scene hooks: hessian_contract (_kernels.py:159-206),
    field_backward(need_input_grads=True) (field.py:332-349), and update_occupancy /
    render_rays with point/dir transforms (renderer.py:108-128, 234-264)."""
    res = {}
    for name in ("c1", "np2"):
        spec = cases.GRIDS[name]
        L, T = spec["num_levels"], spec["table_size"]
        grid = hash_encoding.MultiResHashGrid(**spec)
        tables = cases.trained_tables(L, T)
        xn = cases.grid_points(seed=3)
        inv = np.ascontiguousarray(1.0 / grid.aabb_extent, np.float32)
        coeff = np.random.default_rng(17).standard_normal((xn.shape[0], 2 * L)).astype(np.float32)
        for na in (L, 3):
            res[f"hess_{name}_na{na}"] = _kernels.hessian_contract(xn, tables, grid.resolutions, na,
                                                                   inv, coeff)
    for name in ("c1", "c2"):
        p = _field_params(name)
        x = cases.world_points(seed=5)
        rng = np.random.default_rng(9)
        v = rng.standard_normal((x.shape[0], 3))
        v /= np.linalg.norm(v, axis=1, keepdims=True)
        for lam in (p.grid.num_levels, 3):
            cache = field.eval_field(p, x, v, lam)
            dl_dc = rng.standard_normal((x.shape[0], 3))
            dl_dd = rng.standard_normal(x.shape[0])
            dl_dn = rng.standard_normal((x.shape[0], 3)).astype(np.float32)
            k = f"ig_{name}_lam{lam}_"
            gr = field.field_backward(p, cache, dl_dc=dl_dc, dl_dd=dl_dd, dl_dn=dl_dn,
                                      need_input_grads=True)
            res.update({k + "dl_dc": dl_dc, k + "dl_dd": dl_dd, k + "dl_dn": dl_dn,
                        k + "dl_dx": gr.dl_dx, k + "dl_dv": gr.dl_dv})
            gr = field.field_backward(p, cache, dl_dd=dl_dd, dl_dn=dl_dn, need_input_grads=True)
            res[k + "nocolor_dl_dx"] = gr.dl_dx
    # transforms: c1 scene, SAL init, occupancy refreshed in the moved frame
    R = cases.rodrigues(cases.RIGID_AXIS_ANGLE)
    pt = lambda x: cases.rigid_apply(x, R, cases.RIGID_T)  # noqa: E731
    dt = lambda v: cases.rigid_apply(v, R)  # noqa: E731
    with tempfile.TemporaryDirectory() as td:
        ds = scene_io.make_synthetic("sphere", td, views=8, image_size=64, seed=0)
    cfg = trainer.TrainConfig(batch_size=512, num_levels=8, table_size=2**14, seed=0, level_init=8)
    st = trainer.TrainState.create(cfg, aabb=ds.scene_aabb)
    renderer.update_occupancy(st.occ, st.params, 8, point_transform=pt)
    res["occ_bits"] = np.packbits(st.occ.bits.reshape(-1))
    res["occ_ema_sum"] = st.occ.ema.sum()
    batch = scene_io.sample_ray_batch(ds, 0, cfg.batch_size, cfg.fg_fraction, st.rng)
    rendered, rec = renderer.render_rays(batch, st.params, st.occ, 8, point_transform=pt,
                                         dir_transform=dt)
    res.update({"rt_origins": batch.origins, "rt_dirs": batch.directions, "rt_rendered": rendered,
                "rt_count": rec.sample_count, "rt_R": R})
    np.savez_compressed(OUT / "dynamic_c1.npz", **res)


def init_case():
    """TrainState.create at the INIT_CASES configs: resolutions, MLP layers, s_log and
    the rng state afterwards in full; tables as sha256 + level norms + a sparse sample
    (64 MiB at config 2)."""
    res = {}
    for name, kw in cases.INIT_CASES.items():
        cfg = trainer.TrainConfig(**kw)
        st = trainer.TrainState.create(cfg)
        p, k = st.params, name + "_"
        res[k + "resolutions"] = np.asarray(p.grid.resolutions, np.int64)
        for i, h in enumerate(p.sdf_net.layers):
            res[k + f"sdf{i}"] = h
        for i, h in enumerate(p.color_net.layers):
            res[k + f"col{i}"] = h
        res[k + "slog"] = np.asarray(p.sharpness_log, np.float64)
        res[k + "tables_sha256"] = np.array(cases.sha256(p.grid.tables))
        res[k + "tables_norms"] = cases.level_norms(p.grid.tables)
        res[k + "tables_idx"], res[k + "tables_val"] = cases.sparse_sample(p.grid.tables)
        res[k + "aabb"] = np.array([p.grid.aabb_min, p.grid.aabb_min + p.grid.aabb_extent])
        res[k + "occ"] = np.array([st.occ.resolution, st.occ.threshold, st.occ.step_size])
        res[k + "rng_next"] = st.rng.integers(0, 2**62, size=8)
    np.savez_compressed(OUT / "init.npz", **res)


def main():
    if sys.argv[1:] == ["dynamic"]:
        dynamic_case()
        return
    if sys.argv[1:] == ["init"]:
        init_case()
        return
    checkpoint_case()
    kat()
    mlp_case()
    for g in cases.GRIDS:
        kernels_case(g)
    for g in ("c1", "c2"):
        field_case(g)
    occupancy_case()
    init_case()
    for s in cases.STEP_CASES:
        step_case(s)
    for f in sorted(OUT.glob("*.npz")):
        print(f.name, f.stat().st_size)


if __name__ == "__main__":
    main()
