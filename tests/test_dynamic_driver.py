"""Dynamic-sequence driver (the SPEC `dynamic` module, Eqs. 11-12).
The reference ships no driver, so these are the SPEC's own examples and invariants
(CPU) plus, on the GPU, recovery of a known per-frame translation."""

from __future__ import annotations

import numpy as np
import pytest
import torch

from paper_2212_05231_b200 import dynamic as dyn


def test_to_previous_frame_examples():
    x = np.array([[0.0, 0.0, 0.0], [1.0, 0.0, 0.0]])
    assert np.array_equal(dyn.GlobalTransform.identity().to_previous_frame(x), x)
    gt = dyn.GlobalTransform(np.zeros(3), np.array([1.0, 0.0, 0.0]))
    assert np.allclose(gt.to_previous_frame(x[:1]), [[1.0, 0.0, 0.0]])
    gt = dyn.GlobalTransform(np.array([0.0, 0.0, np.pi / 2]), np.zeros(3))
    assert np.allclose(gt.to_previous_frame(x[1:]), [[0.0, 1.0, 0.0]], atol=1e-6)


def test_accumulate_examples():
    ident = dyn.TransformChain()
    c = ident.accumulate(dyn.GlobalTransform.identity())
    assert np.allclose(c.R, np.eye(3)) and np.allclose(c.T, 0) and c.frame == 1
    ta, tb = np.array([0.1, -0.2, 0.3]), np.array([0.05, 0.0, -0.1])
    c = ident.accumulate(dyn.GlobalTransform(np.zeros(3), ta)).accumulate(dyn.GlobalTransform(np.zeros(3), tb))
    assert np.allclose(c.T, ta + tb)
    q = dyn.GlobalTransform(np.array([0.0, 0.0, np.pi / 2]), np.zeros(3))
    c = ident.accumulate(q).accumulate(q)
    assert np.allclose(c.R, dyn.rodrigues([0.0, 0.0, np.pi]), atol=1e-12)
    p = np.array([[0.3, -0.7, 0.2]])
    assert np.allclose(c.canonicalize(p), q.to_previous_frame(q.to_previous_frame(p)), atol=1e-12)


def test_chain_consistency_and_orthonormality():
    rng = np.random.default_rng(0)
    chain = dyn.TransformChain()
    gts = []
    for _ in range(50):
        gt = dyn.GlobalTransform(rng.normal(0, 0.1, 3), rng.normal(0, 0.05, 3))
        prev = chain
        chain = chain.accumulate(gt)
        gts.append(gt)
        x = rng.normal(size=(4, 3))
        # canonicalize(x, chain_i) == canonicalize(to_previous_frame(x, gt_i), chain_{i-1})
        assert np.allclose(chain.canonicalize(x), prev.canonicalize(gt.to_previous_frame(x)), atol=1e-6)
        assert np.allclose(chain.R @ chain.R.T, np.eye(3), atol=1e-6)
        assert abs(np.linalg.det(chain.R) - 1) < 1e-6
    # Eq. 11 applied frame by frame down to 0 equals the chain (within 1e-5 over 50 frames)
    x = rng.normal(size=(8, 3))
    y = x.copy()
    for gt in reversed(gts):
        y = gt.to_previous_frame(y)
    assert np.allclose(chain.canonicalize(x), y, atol=1e-5)


def test_frame_transform_is_the_accumulated_chain():
    rng = np.random.default_rng(1)
    chain = dyn.TransformChain().accumulate(dyn.GlobalTransform(rng.normal(0, 0.2, 3), rng.normal(0, 0.1, 3)))
    gt = dyn.GlobalTransform(rng.normal(0, 0.2, 3), rng.normal(0, 0.1, 3))
    ft = chain.frame_transform(gt)
    x = rng.normal(size=(6, 3))
    assert np.allclose(ft.point(x), chain.accumulate(gt).canonicalize(x), atol=1e-12)
    xt = torch.from_numpy(x)
    assert np.allclose(ft.point(xt).numpy(), ft.point(x), atol=1e-14)
    assert np.allclose(ft.direction(x), x @ (chain.R @ gt.rotation).T, atol=1e-12)


def test_rodrigues_jacobian_matches_finite_differences():
    rng = np.random.default_rng(2)
    for w in (np.zeros(3), rng.normal(0, 0.3, 3), np.array([0.0, 0.0, 2.5])):
        J = dyn.rodrigues_jacobian(w)
        for k in range(3):
            e = np.zeros(3)
            e[k] = 1e-6
            fd = (dyn.rodrigues(w + e) - dyn.rodrigues(w - e)) / 2e-6
            assert np.allclose(J[k], fd, atol=1e-7), (w, k)


def test_param_gradient_matches_autograd():
    """d/d(w, T) of a loss of (x_c, v_c) through the chained transform, against
    torch autograd of the same composition."""
    rng = np.random.default_rng(3)
    chain = dyn.TransformChain().accumulate(dyn.GlobalTransform(rng.normal(0, 0.2, 3), rng.normal(0, 0.1, 3)))
    gt = dyn.GlobalTransform(rng.normal(0, 0.3, 3), rng.normal(0, 0.1, 3))
    x = torch.from_numpy(rng.normal(size=(64, 3)))
    v = torch.from_numpy(rng.normal(size=(64, 3)))
    A = torch.from_numpy(rng.normal(size=(3, 3)))

    def loss_of(xc, vc):
        return (torch.sin(xc) @ A).pow(2).sum() + (vc * xc).sum()

    ft = chain.frame_transform(gt)
    xc = ft.point(x).requires_grad_(True)
    vc = ft.direction(v).requires_grad_(True)
    gx, gv = torch.autograd.grad(loss_of(xc, vc), [xc, vc])
    ours = ft.param_gradient(x, v, gx, gv)

    p = torch.from_numpy(gt.params.copy()).requires_grad_(True)
    w, t = p[:3], p[3:]
    th = w.norm()
    k = w / th
    K = torch.zeros(3, 3, dtype=torch.float64)
    K = K.index_put((torch.tensor([0, 0, 1, 1, 2, 2]), torch.tensor([1, 2, 0, 2, 0, 1])),
                    torch.stack([-k[2], k[1], k[2], -k[0], -k[1], k[0]]))
    Ri = torch.eye(3, dtype=torch.float64) + torch.sin(th) * K + (1 - torch.cos(th)) * (K @ K)
    Rc = torch.from_numpy(chain.R)
    Tc = torch.from_numpy(chain.T)
    xc2 = ((x + t) @ Ri.T + Tc) @ Rc.T
    vc2 = v @ Ri.T @ Rc.T
    (ref,) = torch.autograd.grad(loss_of(xc2, vc2), [p])
    assert np.allclose(ours, ref.numpy(), rtol=1e-9, atol=1e-9)


def test_sequence_order_violation():
    seq = dyn.SequenceState(train=None)
    with pytest.raises(ValueError, match="sequence order violation"):
        dyn.train_frame(seq, None, 1)


@pytest.mark.gpu
def test_gpu_translating_sphere_recovers_translation():
    """Frame 0 of the translating-sphere preset trained (1.5k steps, 8 levels up to res
    128); on frame 1 (the sphere moved +0.05 in x, so Eq. 11 wants T_1 = (-0.05, 0, 0))
    the transform-only phase (field frozen bit-for-bit) must recover T_1.  Observed on
    B200: T_1 = (-0.0474, -0.0014, -0.0006), within the SPEC's 0.01; asserted with 2x
    margin because frame 0's training uses atomic (order-free) gradient scatters."""
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    from paper_2212_05231_b200 import scene_io, trainer

    ds = scene_io.make_synthetic("translating-sphere", views=12, image_size=64, seed=0, frames=2)
    cfg = trainer.TrainConfig(batch_size=4096, num_levels=8, table_size=2**14, seed=0, level_init=8,
                              max_resolution=128, init_radius=0.25, total_steps=3000)
    seq = dyn.SequenceState(trainer.TrainState.create(cfg, aabb=ds.scene_aabb))
    rep0 = dyn.train_frame(seq, ds, 0, dyn.DynamicConfig(first_frame_steps=1500))
    assert rep0[-1].psnr > 25.0, rep0[-1]
    before = seq.train.params.flat.clone()
    slog = seq.train.params.sharpness_log.clone()
    rep1 = dyn.train_frame(seq, ds, 1, dyn.DynamicConfig(transform_steps=200, frame_steps=200))
    assert torch.equal(before, seq.train.params.flat), "field must stay frozen in the transform phase"
    assert torch.equal(slog, seq.train.params.sharpness_log)
    t = seq.transforms[1].t
    angle = np.linalg.norm(seq.transforms[1].w)
    print("recovered T", t, "angle", angle, "loss", rep1[0].total, "->", rep1[-1].total)
    assert np.linalg.norm(t - np.array([-0.05, 0.0, 0.0])) < 0.02, t
    assert angle < np.deg2rad(2.0)
    assert np.mean([r.total for r in rep1[-20:]]) < np.mean([r.total for r in rep1[:20]])
    assert seq.chain.frame == 1 and np.allclose(seq.chain.T, t)
