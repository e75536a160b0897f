"""Bias-free ReLU MLP weights on the GPU (container API of `hashsdf/relu_mlp.py`).

On the training path the per-sample MLP arithmetic (forward, input-Jacobian row,
first-order backward and the Theorem-1 row contraction, `relu_mlp.py:94-216`) is fused
into the tcgen05 field kernels of libns2b (csrc/field_tc.cu).  This module holds the
layer matrices as CUDA tensors (views into the flat parameter buffer), mirrors the
reference's shape validation and seeded initialisation, and keeps the reference's
standalone array functions (`forward`, `input_jacobian_rows`, `backward_first`,
`backward_second_row`) for callers outside the step: those are plain batched GEMMs
(cuBLAS through torch) on device tensors, fp32, same masks (strict z > 0), same errors.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from ._lib import ShapeError

__all__ = ["ShapeError", "MlpWeights", "ForwardTrace", "forward", "input_jacobian_rows",
           "backward_first", "backward_second", "backward_second_row", "input_jacobian",
           "second_order_input_residual"]


class MlpWeights:
    """Layer l maps n_{l-1} -> n_l as an (n_l, n_{l-1}) fp32 CUDA tensor
    (`relu_mlp.py:33-77`)."""

    def __init__(self, layers):
        layers = [_to_device(h) for h in layers]
        if not layers:
            raise ShapeError("shape error: need at least one layer")
        for a, b in zip(layers[:-1], layers[1:]):
            if b.shape[1] != a.shape[0]:
                raise ShapeError("shape error: consecutive layer dims do not chain")
        for h in layers:
            if not bool(torch.isfinite(h).all()):
                raise ValueError("non-finite layer weights")
        self.layers = layers

    @staticmethod
    def random_host(dims, rng, dtype=np.float32, scale=None):
        """He-style init drawn exactly like `relu_mlp.py:45-52` (host arrays)."""
        out = []
        for n_in, n_out in zip(dims[:-1], dims[1:]):
            std = scale if scale is not None else np.sqrt(2.0 / n_in)
            out.append((rng.standard_normal((n_out, n_in)) * std).astype(dtype))
        return out

    @classmethod
    def random(cls, dims, rng, dtype=np.float32, scale=None):
        return cls(cls.random_host(dims, rng, dtype, scale))

    @property
    def depth(self):
        return len(self.layers)

    @property
    def in_dim(self):
        return self.layers[0].shape[1]

    @property
    def out_dim(self):
        return self.layers[-1].shape[0]

    @property
    def dtype(self):
        return np.dtype(np.float32)

    def copy(self):
        return MlpWeights([h.clone() for h in self.layers])

    def zero_gradients(self):
        return [torch.zeros_like(h) for h in self.layers]


def _to_device(h):
    if isinstance(h, torch.Tensor):
        if h.dtype != torch.float32 or not h.is_cuda:
            h = h.to(device=_lib.device(), dtype=torch.float32)
        return h
    return torch.from_numpy(np.ascontiguousarray(h, dtype=np.float32)).to(_lib.device())


@dataclass
class ForwardTrace:
    """`relu_mlp.py:80-91`: batched input, post-ReLU activations and 0/1 masks per
    hidden layer, and the output (all (P, n) fp32 CUDA tensors)."""
    x: torch.Tensor
    activations: list
    masks: list
    y: torch.Tensor


def _as_batch(a):
    t = _to_device(a)
    return (t[None, :] if t.dim() == 1 else t), t.dim() == 1


def forward(weights, x):
    """`relu_mlp.py:94-111`: returns (y, trace); x may be (n_0,) or (P, n_0)."""
    xb, single = _as_batch(x)
    if xb.shape[1] != weights.in_dim:
        raise ShapeError("shape error: input dim mismatch")
    acts, masks = [], []
    a = xb
    for h in weights.layers[:-1]:
        z = a @ h.T
        m = (z > 0).to(torch.float32)
        a = z * m
        masks.append(m)
        acts.append(a)
    y = a @ weights.layers[-1].T
    return (y[0] if single else y), ForwardTrace(xb, acts, masks, y)


def input_jacobian_rows(weights, trace, rows):
    """`relu_mlp.py:123-129`: selected rows of dy/dx, (P, len(rows), n_0)."""
    rows = list(rows)
    jac = weights.layers[-1][rows].expand(trace.x.shape[0], -1, -1)
    for h, m in zip(weights.layers[-2::-1], trace.masks[::-1]):
        jac = (jac * m[:, None, :]) @ h
    return jac


def backward_first(weights, trace, dl_dy):
    """`relu_mlp.py:132-147`: ([dL/dH_l], dL/dx)."""
    g, single = _as_batch(dl_dy)
    if tuple(g.shape) != tuple(trace.y.shape):
        raise ShapeError("shape error: cotangent does not match output")
    grads = [None] * weights.depth
    up = g
    for l in range(weights.depth - 1, 0, -1):
        grads[l] = up.T @ trace.activations[l - 1]
        up = (up @ weights.layers[l]) * trace.masks[l - 1]
    grads[0] = up.T @ trace.x
    dl_dx = up @ weights.layers[0]
    return grads, (dl_dx[0] if single else dl_dx)


def backward_second_row(weights, trace, row, row_cotangent):
    """`relu_mlp.py:191-216` (Theorem 1 for one Jacobian row): dH_l = svec_l^T pvec_l."""
    mvec, _ = _as_batch(row_cotangent)
    depth = weights.depth
    svec = [None] * depth
    svec[-1] = torch.zeros((mvec.shape[0], weights.out_dim), dtype=torch.float32, device=mvec.device)
    svec[-1][:, row] = 1.0
    for l in range(depth - 2, -1, -1):
        svec[l] = (svec[l + 1] @ weights.layers[l + 1]) * trace.masks[l]
    grads, pvec = [], mvec
    for l in range(depth):
        grads.append(svec[l].T @ pvec)
        if l < depth - 1:
            pvec = (pvec @ weights.layers[l].T) * trace.masks[l]
    return grads


def input_jacobian(weights, trace):
    """`relu_mlp.py:114-120`: full dy/dx per sample, (P, n_L, n_0)."""
    return input_jacobian_rows(weights, trace, range(weights.out_dim))


def backward_second(weights, trace, jac_cotangent):
    """`relu_mlp.py:150-188`: gradients of sum_p <M_p, (dy/dx)_p> w.r.t. each layer
    (masks constant), from the per-sample partial products S_l (output side) and P_l
    (input side): dH_l = sum_p S_l^T M_p P_l^T."""
    m = _to_device(jac_cotangent)
    if m.dim() == 2:
        m = m[None]
    npts, depth = m.shape[0], weights.depth
    back = [None] * depth
    back[-1] = torch.eye(weights.out_dim, device=m.device).expand(npts, -1, -1)
    for l in range(depth - 2, -1, -1):
        back[l] = (back[l + 1] @ weights.layers[l + 1]) * trace.masks[l][:, None, :]
    fwd = [None] * depth
    fwd[0] = torch.eye(weights.in_dim, device=m.device).expand(npts, -1, -1)
    for l in range(1, depth):
        fwd[l] = trace.masks[l - 1][:, :, None] * (weights.layers[l - 1] @ fwd[l - 1])
    return [torch.tensordot(back[l].transpose(1, 2) @ m, fwd[l], dims=([0, 2], [0, 2]))
            for l in range(depth)]


def second_order_input_residual(weights, x, rng, h=1e-3, margin=1e-3, num_directions=8):
    """Largest |f(x+hd) + f(x-hd) - 2f(x)| / h^2 over random unit directions
    (`relu_mlp.py:219-250`): zero for a ReLU net unless a mask flips, which the margin
    precondition on every pre-activation rules out ("near activation boundary")."""
    x = np.asarray(x, np.float32)
    worst = 0.0
    for _ in range(num_directions):
        d = rng.standard_normal(x.shape[0])
        d = (d / np.linalg.norm(d)).astype(np.float32)
        pts = np.stack([x, x + h * d, x - h * d])
        a = _to_device(pts)
        for hl in weights.layers[:-1]:
            z = a @ hl.T
            if float(z.abs().min()) <= margin:
                raise ValueError("near activation boundary")
            a = torch.clamp(z, min=0)
        y, _ = forward(weights, pts)
        worst = max(worst, float((y[1] + y[2] - 2.0 * y[0]).abs().max()) / h**2)
    return worst
