"""NS2C checkpoints: byte compatibility with the reference's writer
(`tests/golden/ckpt_small.ns2c`, written by `hashsdf.checkpoint.save_checkpoint` in
make_golden.py) and, on the GPU, load -> save identity and resume parity with the
oracle from the same file."""

from __future__ import annotations

import dataclasses
from pathlib import Path

import numpy as np
import pytest

from paper_2212_05231_b200 import checkpoint as ck

GOLDEN = Path(__file__).resolve().parent / "golden" / "ckpt_small.ns2c"
GROUPS = {"tables", "sdf_0", "sdf_1", "color_0", "color_1", "color_2", "sharpness_log"}


def test_decode_encode_is_byte_identical():
    raw = GOLDEN.read_bytes()
    d = ck.decode(raw)
    assert ck.encode(d) == raw


def test_golden_contents():
    d = ck.decode(GOLDEN.read_bytes())
    assert d.step == 2
    assert set(d.adam) == GROUPS
    assert all(t == 2 for _, _, t in d.adam.values())
    assert d.tables.shape == (4, 1024, 2) and d.tables.dtype == np.float32
    assert [h.shape for h in d.sdf_layers] == [(64, 12), (16, 64)]
    assert [h.shape for h in d.color_layers] == [(64, 25), (64, 64), (3, 64)]
    assert d.adam["tables"][0].shape == d.tables.shape
    assert d.adam["sharpness_log"][0].dtype == np.float64
    assert d.occ_ema.shape == (16, 16, 16) and d.occ_bits.dtype == np.uint8
    assert d.extra == [(b"XTRA", b"kept")]
    assert d.rng_state["bit_generator"] == "PCG64"


def test_config_fields_match_the_reference():
    from paper_2212_05231_b200.trainer import TrainConfig

    d = ck.decode(GOLDEN.read_bytes())
    cfg = TrainConfig(**d.config)
    assert dataclasses.asdict(cfg) == d.config


def test_errors_match_the_reference(tmp_path):
    raw = GOLDEN.read_bytes()
    with pytest.raises(ValueError, match="not a checkpoint: bad magic"):
        ck.split_sections(b"XXXX" + raw[4:])
    with pytest.raises(ValueError, match="unsupported checkpoint version 7"):
        ck.split_sections(raw[:4] + (7).to_bytes(4, "little") + raw[8:])


def _oracle_state(d):
    """Oracle TrainState from checkpoint values (mirrors checkpoint.py:134-189)."""
    from oracle import field as ofield
    from oracle import hashgrid as ohg
    from oracle import mlp as omlp
    from oracle import render as orender
    from oracle import train as otrain

    gm = d.grid_meta
    lo = np.asarray(gm["aabb_min"])
    grid = ohg.HashGrid(gm["num_levels"], gm["resolutions"][0], gm["resolutions"][-1],
                        gm["features_per_level"], gm["table_size"],
                        (lo.tolist(), (lo + np.asarray(gm["aabb_extent"])).tolist()))
    grid.tables = d.tables.copy()
    params = ofield.FieldParams(grid, omlp.MlpWeights([h.copy() for h in d.sdf_layers]),
                                omlp.MlpWeights([h.copy() for h in d.color_layers]), d.sharpness_log)
    fields = {f.name for f in dataclasses.fields(otrain.TrainConfig)}
    cfg = otrain.TrainConfig(**{k: v for k, v in d.config.items() if k in fields})
    occ = orender.OccupancyGrid(d.occ_resolution, (tuple(d.occ_aabb[0]), tuple(d.occ_aabb[1])),
                                d.occ_threshold)
    occ.ema = d.occ_ema.copy()
    occ.bits = d.occ_bits.astype(bool)
    rng = np.random.default_rng(0)
    rng.bit_generator.state = d.rng_state
    st = otrain.TrainState(params, occ, cfg, rng, step=d.step)
    for k, (m, v, t) in d.adam.items():
        st.adam[k].m, st.adam[k].v, st.adam[k].t = m.copy(), v.copy(), t
    return st


def test_oracle_reads_the_golden():
    st = _oracle_state(ck.decode(GOLDEN.read_bytes()))
    assert st.step == 2 and st.adam["tables"].t == 2


@pytest.mark.gpu
def test_device_load_save_identity(tmp_path):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    st, sec = ck.load_checkpoint(GOLDEN)
    out = tmp_path / "again.ns2c"
    ck.save_checkpoint(out, st, extra_sections=[(b"XTRA", sec[b"XTRA"])])
    assert out.read_bytes() == GOLDEN.read_bytes()


@pytest.mark.gpu
def test_resume_matches_oracle():
    """One step from the golden checkpoint on the GPU and in the oracle: the restored
    rng draws the same batch (same sample count), Adam resumes at t = 2."""
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    from parity import assert_close

    from oracle import scene as oscene
    from oracle import train as otrain
    from paper_2212_05231_b200 import scene_io as pscene
    from paper_2212_05231_b200 import trainer as ptrain

    ds = oscene.make_synthetic("sphere", views=4, image_size=32, seed=0)
    pds = pscene.make_synthetic("sphere", views=4, image_size=32, seed=0)
    d = ck.decode(GOLDEN.read_bytes())
    ost = _oracle_state(d)
    pst, _ = ck.load_checkpoint(GOLDEN)
    ro = otrain.train_step(ost, ds)
    rp = ptrain.train_step(pst, pds)
    assert rp.sample_count == ro.sample_count
    assert rp.level == ro.level
    for k in ("color", "eikonal", "total"):
        a, r = getattr(rp, k), getattr(ro, k)
        assert abs(a - r) <= 1e-3 * max(abs(r), 1e-9), f"{k}: {a} vs {r}"
    for i in range(2):
        assert_close(pst.params.sdf_net.layers[i].cpu().numpy(), ost.params.sdf_net.layers[i], 1e-3, f"sdf{i}")
    for i in range(3):
        assert_close(pst.params.color_net.layers[i].cpu().numpy(), ost.params.color_net.layers[i], 1e-3,
                     f"color{i}")
    assert pst.adam["tables"].t == ost.adam["tables"].t == 3
    assert pst.step == ost.step == 3
