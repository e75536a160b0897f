"""GPU parity of the standalone MLP seam (`relu_mlp.forward / input_jacobian_rows /
backward_first / backward_second_row`, reference `relu_mlp.py:94-216`) against the
reference's golden vectors (tests/golden/mlp.npz, fp64) and the CPU oracle on the
field's own shapes; plus the reference's shape errors (`relu_mlp.py:39-42,100,138`).
fp32 device arithmetic: per-tensor bar 1e-3 (relL2 and max-abs over max|ref|)."""

from __future__ import annotations

from pathlib import Path

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover - CPU containers skip at collection
    pytest.skip("needs a CUDA device", allow_module_level=True)

from oracle import mlp as omlp  # noqa: E402
from paper_2212_05231_b200 import relu_mlp as pmlp  # noqa: E402
from parity import assert_close  # noqa: E402

TOL = 1e-3
GOLD = Path(__file__).resolve().parent / "golden"


def _np(t):
    return t.detach().cpu().numpy()


@pytest.mark.parametrize("depth", [1, 2, 3])
def test_mlp_golden(depth):
    gold = dict(np.load(GOLD / "mlp.npz", allow_pickle=False))
    k = f"d{depth}_"
    w = pmlp.MlpWeights([gold[k + f"w{i}"] for i in range(depth)])
    y, tr = pmlp.forward(w, gold[k + "x"])
    assert_close(_np(y), gold[k + "y"], TOL, "y")
    g1, dx = pmlp.backward_first(w, tr, gold[k + "dy"])
    assert_close(_np(dx), gold[k + "dx"], TOL, "dx")
    g2r = pmlp.backward_second_row(w, tr, 0, gold[k + "mv"])
    for i in range(depth):
        assert_close(_np(g1[i]), gold[k + f"g1_{i}"], TOL, f"g1_{i}")
        assert_close(_np(g2r[i]), gold[k + f"g2r_{i}"], TOL, f"g2r_{i}")


@pytest.mark.parametrize("dims", [(36, 64, 16), (25, 64, 64, 3)])
def test_mlp_field_shapes_vs_oracle(dims):
    """c2 SDF net (36->64->16) and the colour net (25->64->64->3), 4096 seeded rows."""
    rng = np.random.default_rng(0)
    layers = [rng.standard_normal((b, a)).astype(np.float32) * np.float32(np.sqrt(2.0 / a))
              for a, b in zip(dims[:-1], dims[1:])]
    x = rng.standard_normal((4096, dims[0])).astype(np.float32)
    dy = rng.standard_normal((4096, dims[-1])).astype(np.float32)
    mv = rng.standard_normal((4096, dims[0])).astype(np.float32)
    ow = omlp.MlpWeights(layers)
    oy, otr = omlp.forward(ow, x)
    w = pmlp.MlpWeights(layers)
    y, tr = pmlp.forward(w, x)
    assert_close(_np(y), oy, TOL, "y")
    for a, b in zip(tr.masks, otr.masks):
        # strict z > 0 masks; a flip needs |z| at fp32 rounding level
        assert np.mean(_np(a) != b) < 1e-4
    assert_close(_np(pmlp.input_jacobian_rows(w, tr, [0])), omlp.input_jacobian_rows(ow, otr, [0]),
                 TOL, "jrow")
    g1, dx = pmlp.backward_first(w, tr, dy)
    og1, odx = omlp.backward_first(ow, otr, dy)
    assert_close(_np(dx), odx, TOL, "dx")
    g2r = pmlp.backward_second_row(w, tr, 0, mv)
    og2r = omlp.backward_second_row(ow, otr, 0, mv)
    for i in range(len(layers)):
        assert_close(_np(g1[i]), og1[i], TOL, f"g1_{i}")
        assert_close(_np(g2r[i]), og2r[i], TOL, f"g2r_{i}")


def test_mlp_shape_errors():
    w = pmlp.MlpWeights([np.ones((4, 3), np.float32), np.ones((2, 4), np.float32)])
    with pytest.raises(pmlp.ShapeError, match="shape error: input dim mismatch"):
        pmlp.forward(w, np.ones((5, 4), np.float32))
    _, tr = pmlp.forward(w, np.ones((5, 3), np.float32))
    with pytest.raises(pmlp.ShapeError, match="shape error: cotangent does not match output"):
        pmlp.backward_first(w, tr, np.ones((5, 3), np.float32))
    with pytest.raises(pmlp.ShapeError, match="shape error: consecutive layer dims do not chain"):
        pmlp.MlpWeights([np.ones((4, 3), np.float32), np.ones((2, 5), np.float32)])
    with pytest.raises(pmlp.ShapeError, match="shape error: need at least one layer"):
        pmlp.MlpWeights([])
    assert issubclass(pmlp.ShapeError, ValueError)


def test_reference_error_contract():
    """The wrappers raise the reference's exception types and messages
    (`hash_encoding.py:151,180,232,267`, `field.py:70-74,283,302`)."""
    from paper_2212_05231_b200 import field as pfield
    from paper_2212_05231_b200 import hash_encoding as penc

    params = pfield.SdfFieldParams.create(pfield.FieldConfig(num_levels=8, table_size=2**14))
    grid = params.grid
    bad = np.array([[0.0, np.nan, 0.0]], np.float32)
    with pytest.raises(ValueError, match="invalid position"):
        penc.encode(grid, bad, 8)
    with pytest.raises(ValueError, match="invalid position"):
        pfield.eval_field(params, bad, view_dirs=np.ones((1, 3)))
    with pytest.raises(ValueError, match="view_dirs required for color evaluation"):
        pfield.eval_field(params, np.zeros((1, 3), np.float32))
    pt = penc.encode(grid, np.zeros((4, 3), np.float32), 8)  # no caches
    dl_de = torch.zeros((4, grid.encoding_dim), device="cuda")
    with pytest.raises(ValueError, match="stale sample: encode was called without caches"):
        penc.backward_first(grid, pt, dl_de)
    with pytest.raises(ValueError, match="stale sample: encode was called without caches"):
        penc.backward_second(grid, pt, torch.zeros((4, grid.encoding_dim, 3), device="cuda"))
    n = int(grid.resolutions[0])
    with pytest.raises(ValueError, match="cell out of bounds"):
        penc.hash_index([0, 0, n + 1], 0, grid)
    with pytest.raises(ValueError, match="cell out of bounds"):
        penc.hash_index([-1, 0, 0], 0, grid)
    with pytest.raises(ValueError, match="stale sample"):
        pfield.field_backward(params, None)
    cache = pfield.eval_field(params, np.zeros((4, 3), np.float32), need_color=False)
    with pytest.raises(ValueError, match="stale sample"):
        pfield.field_backward(params, cache, dl_dc=np.zeros((4, 3), np.float32))
    with pytest.raises(pmlp.ShapeError, match="shape error: sdf net must output 16 values"):
        pfield.SdfFieldParams(grid, pmlp.MlpWeights([np.ones((64, grid.encoding_dim + 1), np.float32),
                                                     np.ones((15, 64), np.float32)]),
                              params.color_net, 0.0)


@pytest.mark.parametrize("depth", [1, 2, 3])
def test_mlp_full_jacobian_and_backward_second_golden(depth):
    """`relu_mlp.input_jacobian` / `backward_second` (full cotangent M) vs the golden
    vectors (`relu_mlp.py:114-188`)."""
    gold = dict(np.load(GOLD / "mlp.npz", allow_pickle=False))
    k = f"d{depth}_"
    w = pmlp.MlpWeights([gold[k + f"w{i}"] for i in range(depth)])
    _, tr = pmlp.forward(w, gold[k + "x"])
    ow = omlp.MlpWeights([gold[k + f"w{i}"] for i in range(depth)])
    _, otr = omlp.forward(ow, gold[k + "x"])
    assert_close(_np(pmlp.input_jacobian(w, tr)),
                 omlp.input_jacobian_rows(ow, otr, list(range(ow.out_dim))), TOL, "jac")
    g2 = pmlp.backward_second(w, tr, gold[k + "m"])
    for i in range(depth):
        assert_close(_np(g2[i]), gold[k + f"g2_{i}"], TOL, f"g2_{i}")


def test_intersect_aabb_bit_exact():
    from oracle import render as orender
    from paper_2212_05231_b200 import renderer as prender

    rng = np.random.default_rng(4)
    o = rng.uniform(-3, 3, (4096, 3))
    d = rng.standard_normal((4096, 3))
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    d[:8, 1] = 0.0  # axis-parallel rays, inside and outside the slab
    o[:4, 1] = 0.5
    lo, hi = np.array([-1.0, -1.0, -1.0]), np.array([1.0, 1.0, 1.0])
    te, tx = prender.intersect_aabb(o, d, lo, hi)
    re, rx = orender.intersect_aabb(o, d, lo, hi)
    assert np.array_equal(_np(te), re) and np.array_equal(_np(tx), rx)


def test_eval_color_and_sigmoid():
    from helpers import product_params_from_oracle
    from oracle import field as ofield
    from paper_2212_05231_b200 import field as pfield
    from test_oracle_golden import oracle_field_params

    z = np.linspace(-50, 50, 101)
    assert np.array_equal(pfield.sigmoid(z), ofield.sigmoid(z))
    op = oracle_field_params("c1")
    pp = product_params_from_oracle(op)
    rng = np.random.default_rng(2)
    x = rng.uniform(-0.9, 0.9, (2048, 3)).astype(np.float32)
    v1, v2 = (rng.standard_normal((2048, 3)) for _ in range(2))
    v1 /= np.linalg.norm(v1, axis=1, keepdims=True)
    v2 /= np.linalg.norm(v2, axis=1, keepdims=True)
    cache = pfield.eval_field(pp, x, v1, 8)
    cols = pfield.eval_color(pp, cache, v2)
    assert_close(_np(cols), ofield.eval_field(op, x, v2, 8).colors, TOL, "colors")


def test_second_order_input_residual():
    """`relu_mlp.second_order_input_residual` (`relu_mlp.py:219-250`): a ReLU net is
    piecewise linear, so away from mask boundaries the residual is fp32 rounding only;
    a point on a boundary raises."""
    rng = np.random.default_rng(0)
    w = pmlp.MlpWeights([0.25 * rng.standard_normal((16, 5)).astype(np.float32),
                         0.25 * rng.standard_normal((3, 16)).astype(np.float32)])
    for _ in range(20):
        x = rng.standard_normal(5).astype(np.float32)
        try:
            # margin 0.05 > h |row of H1| excludes a flip between x and x +- h d
            r = pmlp.second_order_input_residual(w, x, np.random.default_rng(1), h=1e-2, margin=0.05)
        except ValueError:
            continue
        assert r < 5e-2  # fp32 cancellation / h^2
        break
    else:
        pytest.fail("no point away from the activation boundaries")
    x = np.zeros(5, np.float32)  # every pre-activation is exactly 0
    with pytest.raises(ValueError, match="near activation boundary"):
        pmlp.second_order_input_residual(w, x, np.random.default_rng(1))


def test_theorem1_bench_rows():
    """`autodiff_oracle.bench_second_order` (`autodiff_oracle.py:208-270`): the analytic
    second-order backward agrees with generic double autodiff and the CSV has the
    reference's columns."""
    from paper_2212_05231_b200 import autodiff_oracle as ad

    rows = ad.bench_second_order(16, 3, [8, 64], runs=3)
    assert [r["batch"] for r in rows] == [8, 64] and all(r["speedup"] > 0 for r in rows)
    csv = ad.bench_rows_to_csv(rows).splitlines()
    assert csv[0] == "width,depth,batch,analytic_us,oracle_us,speedup" and len(csv) == 3
    # the graph side itself against the golden vectors (generic M)
    gold = dict(np.load(GOLD / "mlp.npz", allow_pickle=False))
    w = pmlp.MlpWeights([gold[f"d3_w{i}"] for i in range(3)])
    x = torch.from_numpy(gold["d3_x"].astype(np.float32)).cuda()
    m = torch.from_numpy(gold["d3_m"].astype(np.float32)).cuda()
    for i, g in enumerate(ad.graph_grad_of_grad(w, x, m)):
        assert_close(_np(g), gold[f"d3_g2_{i}"], TOL, f"graph g2_{i}")
