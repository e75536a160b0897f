"""Bias-free ReLU MLP weights on the GPU (container API of `hashsdf/relu_mlp.py`).

The per-sample MLP arithmetic (forward, input-Jacobian row, first-order backward
and the Theorem-1 row contraction, `relu_mlp.py:94-216`) is fused into the field
kernels of libns2b (csrc/field.cu); this module only holds the layer matrices as
CUDA tensors (views into the flat parameter buffer) and mirrors the reference's
shape validation and seeded initialisation.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _lib
from ._lib import ShapeError

__all__ = ["ShapeError", "MlpWeights"]


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
