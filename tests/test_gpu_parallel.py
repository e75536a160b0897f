"""Data-parallel product step on one GPU: two processes, `gloo` on CUDA
tensors (the collectives run on the host, so neither rank's kernels wait on the
other's), each running the PRODUCT `trainer.train_step` on its interleaved shard of the
same global batch.  After two steps the parameters and loss reports must equal a
single-process product run (only the gradient summation order differs) and the
oracle's first step (`trainer.py:281-310`: P_glob as the Eikonal divisor, the global m as
the Huber divisor, the gradient prefix and step scalars all-reduced)."""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402

STEPS = 2


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _run(dp, device_sampler):
    """STEPS product steps from the oracle's init; returns reports and parameters."""
    import sys
    from pathlib import Path

    root = Path(__file__).resolve().parents[1]
    for p in (root, root / "tests", root / "tests" / "golden"):
        sys.path.insert(0, str(p))
    from helpers import np_, product_state_from_oracle
    from oracle import render as orender
    from oracle import scene as oscene
    from oracle import train as otrain
    from paper_2212_05231_b200 import scene_io as pscene
    from paper_2212_05231_b200 import trainer as ptrain

    cfg = otrain.TrainConfig(batch_size=2048, num_levels=8, table_size=2**14, seed=0, level_init=8)
    ost = otrain.TrainState.create(cfg)
    orender.update_occupancy(ost.occ, ost.params, 8)
    ost.step = 1
    pst = product_state_from_oracle(ost)
    pst.dp = dp
    reps, batches, first = [], [], []
    toff = pst.params.layout.tables_off
    if device_sampler:
        ds = pscene.make_synthetic("sphere", views=8, image_size=64, seed=0)
        ds.to_device()
        pst.rng = np.random.default_rng(9)
        for _ in range(STEPS):
            reps.append(ptrain.train_step(pst, ds))
            first.append(np_(pst.params.sdf_net.layers[0]).copy())
    else:
        ds = oscene.make_synthetic("sphere", views=8, seed=0, image_size=64)
        rng = np.random.default_rng(9)
        for _ in range(STEPS):
            b = oscene.sample_ray_batch(ds, 0, cfg.batch_size, cfg.fg_fraction, rng)
            batches.append(b)
            reps.append(ptrain.train_step(pst, ds, batch=b))
            first.append(np_(pst.params.sdf_net.layers[0]).copy())
    torch.cuda.synchronize()
    out = {"reports": [(r.sample_count, r.color, r.eikonal, r.total, r.psnr) for r in reps],
           "flat": np_(pst.params.flat).copy(), "slog": float(pst.params.sharpness_log.item()),
           "toff": toff, "sdf0_after_first": first[0]}
    if not device_sampler:  # the oracle's first step on the same batch
        ro = otrain.train_step(ost, ds, batch=batches[0])
        out["oracle_first"] = (ro.sample_count, ro.total, ost.params.sdf_net.layers[0].copy())
    return out


def _check_oracle(res):
    from parity import assert_close

    P0, total0, sdf0 = res["oracle_first"]
    assert res["reports"][0][0] == P0
    assert abs(res["reports"][0][3] - total0) <= 1e-3 * abs(total0)
    assert_close(res["sdf0_after_first"], sdf0, 1e-3, "sdf0 after the first step")


def _worker(rank, world, port, device_sampler, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2212_05231_b200.parallel import DataParallel

        res = _run(DataParallel.from_env(), device_sampler)
        q.put((rank, res))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("device_sampler", [False, True])
def test_two_rank_product_step_equals_single_process(device_sampler):
    from paper_2212_05231_b200.parallel import DataParallel

    single = _run(DataParallel(0, 1), device_sampler)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, device_sampler, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = dict(q.get(timeout=600) for _ in range(2))
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    for r in range(2):
        res = got[r]
        for a, b in zip(res["reports"], single["reports"]):
            assert a[0] == b[0], "global sample count"
            for x, y in zip(a[1:], b[1:]):  # fp64 step sums, reassociated across ranks
                assert abs(x - y) <= 1e-7 * max(abs(y), 1e-12), (a, b)
        k = res["toff"]
        a, b = res["flat"][:k], single["flat"][:k]
        rel = np.linalg.norm(a - b) / np.linalg.norm(b)
        assert rel < 1e-5, f"MLP parameters: relL2 {rel:.2e}"
        # tables: Adam turns gradients at the reassociation floor into +-lr steps, so a
        # few entries may step differently (see test_gpu_parity.assert_adam_tables)
        diff = np.abs(res["flat"][k:] - single["flat"][k:]) > 1e-5
        assert diff.mean() <= 1e-3, f"{diff.sum()} table entries differ"
        assert abs(res["slog"] - single["slog"]) <= 1e-9 * abs(single["slog"])  # reassociated fp64 sums
        if not device_sampler:
            _check_oracle(res)
    assert np.array_equal(got[0]["flat"], got[1]["flat"]), "ranks must hold identical parameters"
    if not device_sampler:
        _check_oracle(single)
