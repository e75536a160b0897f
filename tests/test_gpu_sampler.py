"""Device ray sampler vs the host restatement of `sample_ray_batch`
(`scene_io.py:129-172`): same rng consumption, same picks, identical targets and
origins; directions equal to the last bit wherever the host's BLAS evaluates the
3x3 matmul as an FMA chain (the order ns2b_rays_from_picks uses), else within 2 ulp."""

from __future__ import annotations

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2212_05231_b200 import scene_io  # noqa: E402


def _pair(ds, count, seed, fg=0.9):
    r1, r2 = np.random.default_rng(seed), np.random.default_rng(seed)
    host = scene_io.sample_ray_batch(ds, 0, count, fg, r1)
    dev = scene_io.DeviceSampler(ds).sample(count, fg, r2)
    assert r1.bit_generator.state == r2.bit_generator.state
    return host, dev


@pytest.mark.parametrize("shape", ["square", "rect"])
def test_device_batches_match_host(shape):
    if shape == "square":
        ds = scene_io.make_synthetic("sphere", views=8, image_size=64, seed=0)
    else:
        ds = scene_io.make_synthetic("two-spheres", views=5, seed=3, width=96, height=72, focal=100.8)
    for seed in (0, 1):
        host, dev = _pair(ds, 4096, seed)
        assert np.array_equal(dev.origins.cpu().numpy(), host.origins)
        assert np.array_equal(dev.target_colors.cpu().numpy(), host.target_colors)
        assert np.array_equal(dev.foreground_flags.cpu().numpy(), host.foreground_flags)
        d, h = dev.directions.cpu().numpy(), host.directions
        ulp = np.abs(d - h) / np.spacing(np.abs(h))
        assert ulp.max() <= 2, f"max {ulp.max()} ulp"
        print(f"{shape} seed {seed}: {np.mean(d == h):.4f} of direction components bit-exact")


def test_training_uses_device_sampler():
    from paper_2212_05231_b200 import trainer

    ds_h = scene_io.make_synthetic("sphere", views=8, image_size=64, seed=0)
    ds_d = scene_io.make_synthetic("sphere", views=8, image_size=64, seed=0)
    ds_d.to_device()
    cfg = trainer.TrainConfig(batch_size=2048, num_levels=8, table_size=2**14, seed=0, level_init=8)
    a, b = trainer.TrainState.create(cfg), trainer.TrainState.create(cfg)
    for _ in range(2):
        ra = trainer.train_step(a, ds_h)
        rb = trainer.train_step(b, ds_d)
        assert ra.sample_count == rb.sample_count
        assert abs(ra.total - rb.total) <= 1e-6 * abs(ra.total)
    assert a.rng.bit_generator.state == b.rng.bit_generator.state


def test_draw_ahead_keeps_the_reference_stream():
    """`train_step` draws the next step's picks while the device runs (`draw_ahead`): the
    batches, the losses and the rng position any caller observes are those of drawing at
    the start of each step -- across an external read of `state.rng`, a step on the host
    sampler (other dataset), a re-seed and a checkpoint-style state read."""
    from paper_2212_05231_b200 import trainer

    ds_d = scene_io.make_synthetic("sphere", views=8, image_size=64, seed=0)
    ds_d.to_device()
    ds_h = scene_io.make_synthetic("sphere", views=8, image_size=64, seed=0)
    cfg = trainer.TrainConfig(batch_size=2048, num_levels=8, table_size=2**14, seed=0, level_init=8)
    a, b = trainer.TrainState.create(cfg), trainer.TrainState.create(cfg)
    b.draw_ahead = False

    def both(ds):
        ra, rb = trainer.train_step(a, ds), trainer.train_step(b, ds)
        assert ra.sample_count == rb.sample_count
        # (same batches; the float-atomic order of the scatter drifts the parameters ~1e-7
        # per step, so the losses of later steps agree to ~1e-6, not bit for bit)
        assert abs(ra.total - rb.total) <= 1e-4 * abs(rb.total)

    both(ds_d)
    assert a._ahead is not None  # a draw is pending ...
    both(ds_d)                   # ... and used
    assert a.rng.bit_generator.state == b.rng.bit_generator.state  # rewinds the pending draw
    both(ds_d)
    both(ds_h)                   # host sampler: the pending draw is rewound first
    both(ds_d)
    a.rng, b.rng = np.random.default_rng(3), np.random.default_rng(3)
    both(ds_d)
    both(ds_d)
    assert a.rng.bit_generator.state == b.rng.bit_generator.state
    assert a._ahead is None


@pytest.mark.parametrize("world", [2, 3])
def test_device_sampler_shards(world):
    """`DeviceSampler.sample_into` (the data-parallel path of train_step): each rank's
    interleaved shard equals the same rows of the full global batch, and every rank's
    rng ends in the same state as a single-process draw."""
    from paper_2212_05231_b200.parallel import shard_size, shard_slice

    ds = scene_io.make_synthetic("sphere", views=8, image_size=64, seed=0)
    smp = scene_io.DeviceSampler(ds)
    count = 1001
    full = smp.sample(count, 0.9, np.random.default_rng(5))
    ref_state = np.random.default_rng(5)
    smp._draw(count, 0.9, ref_state)
    for r in range(world):
        n = shard_size(count, r, world)
        o, d, t = (torch.empty((n, 3), dtype=torch.float64, device="cuda") for _ in range(3))
        rng = np.random.default_rng(5)
        smp.sample_into(count, 0.9, rng, o, d, t, r, world)
        sl = shard_slice(count, r, world)
        for got, ref in ((o, full.origins), (d, full.directions), (t, full.target_colors)):
            assert torch.equal(got, ref[sl])
        assert rng.bit_generator.state == ref_state.bit_generator.state


def test_device_sampler_matches_reference_golden():
    """The device sampler after the product's own seeded `TrainState.create` reproduces
    the reference's first two batches (tests/golden/step_c1_full.npz): origins and
    targets bit-exact, directions within 2 ulp, foreground flags exact."""
    from pathlib import Path

    import cases

    from paper_2212_05231_b200 import trainer

    g = dict(np.load(Path(__file__).resolve().parent / "golden" / "step_c1_full.npz"))
    spec = cases.STEP_CASES["c1_full"]
    sc = spec["scene"]
    ds = scene_io.make_synthetic(sc["preset"], views=sc["views"], seed=sc["seed"], image_size=sc["image_size"])
    cfg = trainer.TrainConfig(**spec["cfg"])
    st = trainer.TrainState.create(cfg)
    smp = scene_io.DeviceSampler(ds)
    for s in range(2):
        b = smp.sample(cfg.batch_size, cfg.fg_fraction, st.rng)
        assert np.array_equal(b.origins.cpu().numpy(), g[f"s{s}_origins"])
        assert np.array_equal(b.target_colors.cpu().numpy(), g[f"s{s}_targets"])
        d, h = b.directions.cpu().numpy(), g[f"s{s}_dirs"]
        assert (np.abs(d - h) / np.spacing(np.abs(h))).max() <= 2
