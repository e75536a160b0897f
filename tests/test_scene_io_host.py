"""Host-side scene I/O of the trainer seam (`scene_io.py:44-57, 86-126, 178-213,
261-266`): pinhole ray / projection round trip, agreement of the per-pixel and grid ray
generators with the oracle, the union-of-spheres SDF, and dataset loading from a
`transforms.json` directory written here (RGBA and RGB frames).  CPU only."""

from __future__ import annotations

import json

import numpy as np
import pytest

from oracle import scene as oscene
from paper_2212_05231_b200 import scene_io as ps


def test_generate_ray_and_projection():
    ds = oscene.make_synthetic("sphere", views=2, seed=0, image_size=32)
    f = ds.frames[1]
    o, d = oscene.generate_rays_grid(f)
    for px, py in [(0, 0), (31, 0), (7, 19), (31, 31)]:
        ro, rd = ps.generate_ray(f, px, py)
        k = py * f.width + px
        assert np.allclose(ro, o[k], atol=0) and np.allclose(rd, d[k], rtol=0, atol=1e-15)
        qx, qy = ps.project_point(f, ro + 2.5 * rd)
        assert abs(qx - px) < 1e-9 and abs(qy - py) < 1e-9
    with pytest.raises(ValueError, match="pixel out of range"):
        ps.generate_ray(f, 32, 0)
    go, gd = ps.generate_rays_grid(f)
    assert np.array_equal(go, o) and np.array_equal(gd, d)


def test_scene_sdf():
    spheres, _ = oscene.preset_scene("two-spheres")
    pts = np.random.default_rng(0).uniform(-1, 1, (1000, 3))
    want = np.min([np.linalg.norm(pts - np.asarray(c), axis=1) - r for c, r, _ in spheres], axis=0)
    assert np.array_equal(ps.scene_sdf(spheres, pts), want)


def test_load_dataset(tmp_path):
    from PIL import Image

    rng = np.random.default_rng(3)
    rgba = rng.integers(0, 256, (6, 8, 4), dtype=np.uint8)
    rgb = rng.integers(0, 256, (6, 8, 3), dtype=np.uint8)
    Image.fromarray(rgba, "RGBA").save(tmp_path / "a.png")
    Image.fromarray(rgb, "RGB").save(tmp_path / "b.png")
    pose = np.eye(4)
    pose[:3, 3] = [0.0, 0.0, -2.5]
    meta = {"fl_x": 10.0, "fl_y": 11.0, "cx": 4.0, "cy": 3.0, "w": 8, "h": 6,
            "frames": [{"file_path": "a.png", "transform_matrix": pose.tolist()},
                       {"file_path": "b.png", "transform_matrix": pose.tolist(), "time_index": 2}]}
    (tmp_path / "transforms.json").write_text(json.dumps(meta))
    ds = ps.load_dataset(tmp_path)
    assert ds.num_time_steps == 3 and len(ds.frames) == 2
    a, b = ds.frames
    assert np.array_equal(a.image, rgba[:, :, :3] / 255.0)
    assert np.array_equal(a.mask, (rgba[:, :, 3] / 255.0 > 0.5).astype(np.float64))
    assert np.array_equal(b.mask, np.ones((6, 8))) and b.time_index == 2
    assert ds.scene_aabb == ((-1, -1, -1), (1, 1, 1))
    with pytest.raises(FileNotFoundError, match="dataset not found"):
        ps.load_dataset(tmp_path / "missing")
    bad = dict(meta)
    bad["frames"] = [{"file_path": "a.png", "transform_matrix": (2 * np.eye(4)).tolist()}]
    (tmp_path / "transforms.json").write_text(json.dumps(bad))
    with pytest.raises(ValueError, match="invalid pose"):
        ps.load_dataset(tmp_path)


def _golden_batches():
    """The reference's first two `sample_ray_batch` draws after `TrainState.create`
    (tests/golden/step_c1_full.npz, written by make_golden.py from the reference)."""
    from pathlib import Path

    import cases

    g = dict(np.load(Path(__file__).resolve().parent / "golden" / "step_c1_full.npz"))
    spec = cases.STEP_CASES["c1_full"]
    return g, spec


def test_host_sampler_matches_reference_golden():
    """`scene_io.sample_ray_batch` (`scene_io.py:129-172`) on the product's in-memory
    `make_synthetic` dataset, drawing from the rng the seeded init leaves (the oracle's
    `TrainState.create`, pinned to the reference's rng stream in test_oracle_golden):
    the reference's golden batches, origins and targets bit-exact, directions within
    1 ulp (the 3x3 rotation's BLAS summation order), and so is the oracle's sampler."""
    from oracle import train as otrain

    g, spec = _golden_batches()
    sc = spec["scene"]
    ds = ps.make_synthetic(sc["preset"], views=sc["views"], seed=sc["seed"], image_size=sc["image_size"])
    ods = oscene.make_synthetic(sc["preset"], views=sc["views"], seed=sc["seed"], image_size=sc["image_size"])
    cfg = otrain.TrainConfig(**spec["cfg"])
    rng = otrain.TrainState.create(cfg).rng
    orng = otrain.TrainState.create(cfg).rng
    for s in range(2):
        b = ps.sample_ray_batch(ds, 0, cfg.batch_size, cfg.fg_fraction, rng)
        ob = oscene.sample_ray_batch(ods, 0, cfg.batch_size, cfg.fg_fraction, orng)
        for got in (b, ob):
            assert np.array_equal(got.origins, g[f"s{s}_origins"])
            assert np.array_equal(got.target_colors, g[f"s{s}_targets"])
            ulp = np.abs(got.directions - g[f"s{s}_dirs"]) / np.spacing(np.abs(g[f"s{s}_dirs"]))
            assert ulp.max() <= 1, f"step {s}: directions {ulp.max()} ulp"
    assert rng.bit_generator.state == orng.bit_generator.state
