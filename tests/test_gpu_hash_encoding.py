"""Value parity of the `hash_encoding` module API (`hash_encoding.py:170-272`) on the
device against the oracle: encode (features, Jacobian, corner records),
encode_features_only, backward_first and backward_second accumulating into a given
`out`, at the config-1, config-2 and odd-table-size grids, with all levels and with a
fractional level cutoff.  Corner indices bit-exact; values within 1e-5 (relL2 and
max-abs / max|ref|) -- the fp32 gather/scatter differ from the oracle's only in the
order of fp32 additions."""

from __future__ import annotations

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import cases  # noqa: E402
from helpers import np_  # noqa: E402
from oracle import hashgrid as ohg  # noqa: E402
from paper_2212_05231_b200 import hash_encoding as pe  # noqa: E402
from parity import assert_close, assert_exact  # noqa: E402

TOL = 1e-5


def grids(name):
    spec = cases.GRIDS[name]
    og = ohg.HashGrid(**spec)
    og.tables = cases.trained_tables(spec["num_levels"], spec["table_size"])
    pg = pe.MultiResHashGrid(spec["num_levels"], spec["min_resolution"], spec["max_resolution"], 2,
                             spec["table_size"], tables=torch.from_numpy(og.tables.copy()).cuda())
    assert_exact(pg.resolutions, og.resolutions, "resolutions")
    return og, pg


@pytest.mark.parametrize("name", list(cases.GRIDS))
@pytest.mark.parametrize("max_level", ["all", 3.7])
def test_encode_and_backward_values(name, max_level):
    og, pg = grids(name)
    ml = og.num_levels if max_level == "all" else max_level
    x = cases.world_points(seed=11, n=6000)
    oe = ohg.encode(og, x, ml, need_jacobian=True)
    pe_ = pe.encode(pg, x, ml, need_jacobian=True)
    assert_close(np_(pe_.e), oe.e, TOL, "e")
    assert_close(np_(pe_.jacobian), oe.jacobian, TOL, "jacobian")
    rec_o, rec_p = oe.corner_records, pe_.corner_records
    assert rec_p.active_levels == rec_o.active_levels == pe.active_level_count(pg, ml)
    na = rec_o.active_levels
    assert_exact(np_(rec_p.indices)[:, :na], rec_o.indices[:, :na], "corner indices")
    assert_close(np_(rec_p.weights)[:, :na], rec_o.weights[:, :na], TOL, "corner weights")
    assert_close(np_(rec_p.weight_gradients)[:, :na], rec_o.weight_gradients[:, :na], TOL, "corner dw")
    assert_close(np_(pe.encode_features_only(pg, x, ml)), ohg.encode_features_only(og, x, ml), TOL,
                 "features only")
    rng = np.random.default_rng(3)
    dl_de = rng.standard_normal(oe.e.shape).astype(np.float32)
    u = rng.standard_normal(oe.jacobian.shape).astype(np.float32)
    # accumulate into a non-zero `out`, as field_backward does (first, then second order)
    base = rng.standard_normal(og.tables.shape).astype(np.float32) * 1e-2
    out_o = base.copy()
    ohg.backward_first(og, oe, dl_de, out=out_o)
    ohg.backward_second(og, oe, u, out=out_o)
    out_p = torch.from_numpy(base.copy()).cuda()
    r1 = pe.backward_first(pg, pe_, dl_de, out=out_p)
    r2 = pe.backward_second(pg, pe_, u, out=out_p)
    assert r1 is out_p and r2 is out_p, "backward_* accumulate into and return `out`"
    for lv in range(og.num_levels):
        assert_close(np_(out_p)[lv], out_o[lv], TOL, f"table gradient level {lv}")
    # fresh outputs when out is None
    assert_close(np_(pe.backward_first(pg, pe_, dl_de)), ohg.backward_first(og, oe, dl_de), TOL, "first")
    assert_close(np_(pe.backward_second(pg, pe_, u)), ohg.backward_second(og, oe, u), TOL, "second")


def test_stale_sample_and_invalid_position():
    og, pg = grids("c1")
    x = cases.world_points(seed=1, n=64)
    lean = pe.encode(pg, x, 8, need_jacobian=False)
    with pytest.raises(ValueError, match="stale sample"):
        pe.backward_first(pg, lean, np.zeros((64, pg.encoding_dim), np.float32))
    with pytest.raises(ValueError, match="stale sample"):
        pe.backward_second(pg, lean, np.zeros((64, pg.encoding_dim, 3), np.float32))
    bad = x.copy()
    bad[3, 1] = np.nan
    with pytest.raises(ValueError, match="invalid position"):
        pe.encode(pg, bad, 8)
