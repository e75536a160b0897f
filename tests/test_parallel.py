"""Data-parallel decomposition of the training step, on CPU with gloo, world size 2.

Each rank keeps its interleaved shard (rays rank, rank + N, ...) of the SAME global ray
batch and runs the step's
per-ray work (the oracle stands in for the device kernels here); the collectives are
`parallel.DataParallel`'s: all-reduce of the kept-sample count (global Eikonal mean)
and of the gradients and step scalars.  The reduced gradients must equal the
single-process step's (only the summation order differs).
"""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2212_05231_b200.parallel import DataParallel, shard_bounds, shard_size, shard_slice


def test_shard_bounds_cover_and_balance():
    for m in (1, 7, 4096, 262145):
        for w in (1, 2, 3, 8):
            spans = [shard_bounds(m, r, w) for r in range(w)]
            assert spans[0][0] == 0 and spans[-1][1] == m
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
            sizes = [hi - lo for lo, hi in spans]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        shard_bounds(10, 2, 2)


def test_interleaved_shards_cover():
    for m in (1, 7, 4096, 262145):
        for w in (1, 2, 3, 8):
            idx = np.concatenate([np.arange(m)[shard_slice(m, r, w)] for r in range(w)])
            assert np.array_equal(np.sort(idx), np.arange(m))
            assert [shard_size(m, r, w) for r in range(w)] == [len(range(m)[shard_slice(m, r, w)])
                                                                for r in range(w)]
    with pytest.raises(ValueError):
        shard_slice(10, 2, 2)


def test_interleaved_shards_balance_samples():
    """Per-rank kept-sample counts at the bench's weak-scaling shape (N x 2^18 rays,
    N = 8) with the per-ray sample counts of a real marched batch (config-1 sphere scene,
    the oracle's marcher on the SAL-init occupancy), resampled per foreground /
    background ray: the interleaved shard keeps every rank within 1 % of the mean, the
    contiguous split the reference-order batch would get does not."""
    from oracle import render as orender
    from oracle import scene as oscene
    from oracle import train as otrain

    ds = oscene.make_synthetic("sphere", views=8, seed=0, image_size=64)
    cfg = otrain.TrainConfig(batch_size=8192, num_levels=8, table_size=2**14, seed=0, level_init=8)
    st = otrain.TrainState.create(cfg)
    orender.update_occupancy(st.occ, st.params, 8)
    b = oscene.sample_ray_batch(ds, 0, cfg.batch_size, cfg.fg_fraction, np.random.default_rng(1))
    rec = orender.march_rays(b.origins, b.directions, st.occ)
    per_ray = np.bincount(rec.ray_ids, minlength=b.count)
    fg, bg = per_ray[b.foreground_flags], per_ray[~b.foreground_flags]
    world, m_rank = 8, 1 << 18
    m = world * m_rank
    n_fg = int(np.floor(0.9 * m))
    rng = np.random.default_rng(0)
    counts = np.concatenate([rng.choice(fg, n_fg), rng.choice(bg, m - n_fg)])
    inter = np.array([counts[shard_slice(m, r, world)].sum() for r in range(world)], np.float64)
    contig = np.array([counts[slice(*shard_bounds(m, r, world))].sum() for r in range(world)], np.float64)
    dev_i = np.abs(inter / inter.mean() - 1).max()
    dev_c = np.abs(contig / contig.mean() - 1).max()
    print(f"max per-rank P deviation at N=8: interleaved {dev_i:.4%}, contiguous {dev_c:.2%}")
    assert dev_i < 0.01
    assert dev_c > 0.05  # the imbalance the interleaved shard removes


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def sharded_step(dp, state, ds, batch):
    """One oracle step with the product's DP collectives (trainer.train_step order)."""
    from oracle import field as ofield
    from oracle import render as orender
    from oracle import scene as oscene
    from oracle import train as otrain

    cfg = state.config
    m_total = batch.count
    sl = dp.shard(m_total)
    local = oscene.RayBatch(batch.origins[sl], batch.directions[sl],
                            batch.target_colors[sl], batch.foreground_flags[sl])
    level = otrain.level_schedule(state.step, cfg)
    rendered, rec = orender.render_rays(local, state.params, state.occ, level)
    P_glob = dp.allreduce_count(rec.sample_count, "cpu")
    resid = rendered - local.target_colors
    dl_dray = otrain.huber_grad(resid, cfg.huber_delta) / m_total
    dl_dc, dl_df, dl_dslog = orender.backward_cotangents(rec, dl_dray)
    n = rec.cache.normals
    norms = np.linalg.norm(n, axis=1)
    dl_dn = (cfg.eikonal_weight * (2.0 * (norms - 1.0) / np.maximum(norms, 1e-12))[:, None]
             * n / P_glob)
    g = ofield.field_backward(state.params, rec.cache, dl_dc=dl_dc, dl_dd=dl_df, dl_dn=dl_dn)
    flat = torch.from_numpy(np.concatenate([g.tables.ravel()] + [h.ravel() for h in g.sdf_layers]
                                           + [h.ravel() for h in g.color_layers]).astype(np.float64))
    sums = torch.tensor([otrain.huber(resid, cfg.huber_delta).sum(), dl_dslog,
                         float(((norms - 1.0) ** 2).sum())], dtype=torch.float64)
    dp.allreduce_(flat)
    dp.allreduce_(sums)
    return flat.numpy(), sums.numpy(), P_glob


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import render as orender
        from oracle import scene as oscene
        from oracle import train as otrain

        ds = oscene.make_synthetic("sphere", views=4, seed=0, image_size=32)
        cfg = otrain.TrainConfig(batch_size=256, num_levels=8, table_size=2**12, seed=0,
                                 level_init=8)
        st = otrain.TrainState.create(cfg)
        orender.update_occupancy(st.occ, st.params, 8)
        st.step = 1
        batch = oscene.sample_ray_batch(ds, 0, cfg.batch_size, cfg.fg_fraction,
                                        np.random.default_rng(3))
        flat, sums, P = sharded_step(DataParallel.from_env(), st, ds, batch)
        if rank == 0:
            single, ssums, sP = sharded_step(DataParallel(0, 1), st, ds, batch)
            out.put((flat, sums, P, single, ssums, sP))
    finally:
        dist.destroy_process_group()


def test_two_rank_gloo_step_equals_single_process():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    flat, sums, P, single, ssums, sP = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert P == sP
    rel = np.linalg.norm(flat - single) / np.linalg.norm(single)
    assert rel < 1e-6, rel
    np.testing.assert_allclose(sums, ssums, rtol=1e-6, atol=1e-12)
