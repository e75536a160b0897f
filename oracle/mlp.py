"""Oracle: bias-free ReLU MLP with the Theorem-1 backward (TEST INFRASTRUCTURE ONLY).

Restates `hashsdf/relu_mlp.py`.  Layer l is an (n_l, n_{l-1}) matrix; hidden
layers use the strict mask z > 0 stored as 0/1 in the weight dtype.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np


class ShapeError(ValueError):
    """`relu_mlp.py:29-30`."""


class MlpWeights:
    """`relu_mlp.py:33-77`."""

    def __init__(self, layers):
        layers = [np.asarray(h) for h in layers]
        if not layers:
            raise ShapeError("shape error: need at least one layer")
        for lo, hi in zip(layers[:-1], layers[1:]):
            if hi.shape[1] != lo.shape[0]:
                raise ShapeError("shape error: consecutive layer dims do not chain")
        if not all(np.all(np.isfinite(h)) for h in layers):
            raise ValueError("non-finite layer weights")
        self.layers = layers

    @classmethod
    def random(cls, dims, rng, dtype=np.float32, scale=None):
        out = []
        for n_in, n_out in zip(dims[:-1], dims[1:]):
            std = np.sqrt(2.0 / n_in) if scale is None else scale
            out.append((rng.standard_normal((n_out, n_in)) * std).astype(dtype))
        return cls(out)

    depth = property(lambda self: len(self.layers))
    in_dim = property(lambda self: self.layers[0].shape[1])
    out_dim = property(lambda self: self.layers[-1].shape[0])
    dtype = property(lambda self: self.layers[0].dtype)

    def copy(self):
        return MlpWeights([h.copy() for h in self.layers])

    def zero_gradients(self):
        return [np.zeros_like(h) for h in self.layers]


@dataclass
class Trace:
    """`relu_mlp.py:80-91`."""

    x: np.ndarray
    activations: list
    masks: list
    y: np.ndarray


def forward(weights, x):
    """`relu_mlp.py:94-111`."""
    x = np.asarray(x, weights.dtype)
    single = x.ndim == 1
    a = x[None, :] if single else x
    if a.shape[1] != weights.in_dim:
        raise ShapeError("shape error: input dim mismatch")
    xin, acts, masks = a, [], []
    for h in weights.layers[:-1]:
        z = a @ h.T
        mask = (z > 0).astype(weights.dtype)
        a = z * mask
        masks.append(mask)
        acts.append(a)
    y = a @ weights.layers[-1].T
    return (y[0] if single else y), Trace(xin, acts, masks, y)


def input_jacobian_rows(weights, trace, rows):
    """`relu_mlp.py:123-129`: rows of dy/dx as (P, len(rows), n_0)."""
    npts = trace.x.shape[0]
    top = weights.layers[-1][rows]
    jac = np.broadcast_to(top, (npts,) + top.shape).copy()
    for h, mask in zip(weights.layers[-2::-1], trace.masks[::-1]):
        jac = (jac * mask[:, None, :]) @ h
    return jac


def backward_first(weights, trace, dl_dy):
    """`relu_mlp.py:132-147`: ([dL/dH_l], dL/dx)."""
    g = np.asarray(dl_dy, weights.dtype)
    single = g.ndim == 1
    g = g[None, :] if single else g
    if g.shape != trace.y.shape:
        raise ShapeError("shape error: cotangent does not match output")
    grads = [None] * weights.depth
    for l in range(weights.depth - 1, 0, -1):
        grads[l] = g.T @ trace.activations[l - 1]
        g = (g @ weights.layers[l]) * trace.masks[l - 1]
    grads[0] = g.T @ trace.x
    dx = g @ weights.layers[0]
    return grads, (dx[0] if single else dx)


def backward_second(weights, trace, jac_cotangent):
    """General-M Theorem 1 (`relu_mlp.py:150-188`): d<M, dy/dx>/dH_l =
    sum_p S_l^T M P_l^T with S_l / P_l the masked partial products."""
    m = np.asarray(jac_cotangent, weights.dtype)
    m = m[None] if m.ndim == 2 else m
    npts, depth = trace.x.shape[0], weights.depth
    back = [None] * depth
    back[-1] = np.broadcast_to(np.eye(weights.out_dim, dtype=weights.dtype),
                               (npts, weights.out_dim, weights.out_dim))
    for l in range(depth - 2, -1, -1):
        back[l] = (back[l + 1] @ weights.layers[l + 1]) * trace.masks[l][:, None, :]
    fwd = [None] * depth
    fwd[0] = np.broadcast_to(np.eye(weights.in_dim, dtype=weights.dtype),
                             (npts, weights.in_dim, weights.in_dim))
    for l in range(1, depth):
        fwd[l] = trace.masks[l - 1][:, :, None] * (weights.layers[l - 1] @ fwd[l - 1])
    out = []
    for l in range(depth):
        left = np.matmul(back[l].transpose(0, 2, 1), m)
        out.append(np.tensordot(left, fwd[l], axes=([0, 2], [0, 2])))
    return out


def backward_second_row(weights, trace, row, row_cotangent):
    """`relu_mlp.py:191-216`: Theorem 1 for a rank-1 cotangent e_row (x) mvec.
    svec_l is row `row` of the masked backward product, pvec_l the masked
    forward product applied to mvec; dH_l += svec_l^T pvec_l."""
    mvec = np.asarray(row_cotangent, weights.dtype)
    mvec = mvec[None, :] if mvec.ndim == 1 else mvec
    npts, depth = mvec.shape[0], weights.depth
    svec = [None] * depth
    svec[-1] = np.zeros((npts, weights.out_dim), weights.dtype)
    svec[-1][:, row] = 1.0
    for l in range(depth - 2, -1, -1):
        svec[l] = (svec[l + 1] @ weights.layers[l + 1]) * trace.masks[l]
    grads, pvec = [], mvec
    for l in range(depth):
        grads.append(svec[l].T @ pvec)
        if l < depth - 1:
            pvec = (pvec @ weights.layers[l].T) * trace.masks[l]
    return grads
