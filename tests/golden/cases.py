"""Seeded parity cases shared by make_golden.py (reference side) and the tests.

Inputs are regenerated from seeds so the committed fixtures only hold outputs.
Nothing here imports the reference or the product package.
"""

from __future__ import annotations

import numpy as np

# (name, num_levels, table_size, min_res, max_res) hash-grid shapes:
#   c1  = config 1 (8 levels, 2^14), c2 = config 2 (16 levels, 2^19, 5 dense levels),
#   np2 = a non-power-of-two table (exercises the 64-bit modulo path).
GRIDS = {
    "c1": dict(num_levels=8, table_size=2**14, min_resolution=16, max_resolution=2048),
    "c2": dict(num_levels=16, table_size=2**19, min_resolution=16, max_resolution=2048),
    "np2": dict(num_levels=6, table_size=393217, min_resolution=16, max_resolution=512),
}


def grid_points(seed=0, n_uniform=384, n_vertex=96, n_edge=32):
    """Normalized positions in [0,1]^3: uniform, near/on grid vertices of several
    resolutions (lower-cell convention), and the box faces."""
    rng = np.random.default_rng(seed)
    u = rng.uniform(0, 1, (n_uniform, 3))
    res = rng.choice([16, 22, 31, 81, 154, 1482, 2048], size=(n_vertex, 1))
    v = np.floor(rng.uniform(0, 1, (n_vertex, 3)) * res) / res
    v = v + rng.choice([0.0, 1e-7, -1e-7], size=v.shape)
    e = rng.choice([0.0, 1.0, 0.5], size=(n_edge, 3))
    return np.clip(np.concatenate([u, v, e]), 0, 1).astype(np.float32)


def world_points(seed=0, n=512):
    """World positions in the default aabb [-1,1]^3, incl. clamped outside points."""
    rng = np.random.default_rng(seed)
    x = rng.uniform(-1.05, 1.05, (n, 3))
    return x.astype(np.float32)


def trained_tables(num_levels, table_size, seed=1, scale=0.1, features=2):
    """'Trained-like' tables U(+-scale) (fp32)."""
    rng = np.random.default_rng(seed)
    return rng.uniform(-scale, scale, (num_levels, table_size, features)).astype(np.float32)


# Train-step cases: mini sphere scene (config-1 field), small ray batches.
STEP_CASES = {
    # default progressive schedule: lambda = 2 at steps 0,1
    "c1_sched": dict(scene=dict(preset="sphere", views=8, image_size=64, seed=0),
                     cfg=dict(batch_size=128, num_levels=8, table_size=2**14, seed=0),
                     steps=2),
    # all levels active from step 0 (level_init = L)
    "c1_full": dict(scene=dict(preset="sphere", views=8, image_size=64, seed=0),
                    cfg=dict(batch_size=128, num_levels=8, table_size=2**14, seed=0,
                             level_init=8),
                    steps=2),
}


# TrainState.create cases (`trainer.py:192-212`): seeded init of the parameters in the
# reference's draw order, for the config-1 and config-2 field shapes.
INIT_CASES = {
    "c1": dict(batch_size=4096, num_levels=8, table_size=2**14, seed=0),
    "c2": dict(batch_size=1 << 18, num_levels=16, table_size=2**19, seed=0),
    "np2": dict(batch_size=512, num_levels=6, table_size=393217, max_resolution=512, seed=3),
}


def sha256(a):
    import hashlib

    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def sparse_sample(a, k=4000, seed=7):
    """(flat indices, values) of up to k nonzeros of a, deterministic."""
    flat = a.reshape(-1)
    nz = np.flatnonzero(flat)
    if nz.size > k:
        nz = np.sort(np.random.default_rng(seed).choice(nz, size=k, replace=False))
    return nz.astype(np.int64), flat[nz]


def level_norms(g):
    """Per-level (L2 norm, sum, nnz) of a (L, T, F) table-shaped array (float64)."""
    g = g.astype(np.float64).reshape(g.shape[0], -1)
    return np.stack([np.sqrt((g * g).sum(1)), g.sum(1), (g != 0).sum(1)], axis=1)


# Dynamic-scene hooks: a fixed rigid transform x -> R (x + T) (Eq. 11),
# evaluated elementwise in one fixed order so numpy (reference / oracle side) and
# torch (device side) produce identical bits.
RIGID_AXIS_ANGLE = (0.05, -0.12, 0.2)
RIGID_T = (0.03, -0.02, 0.04)


def rodrigues(w):
    w = np.asarray(w, np.float64)
    th = float(np.linalg.norm(w))
    k = w / th
    kx = np.array([[0, -k[2], k[1]], [k[2], 0, -k[0]], [-k[1], k[0], 0]])
    return np.eye(3) + np.sin(th) * kx + (1 - np.cos(th)) * (kx @ kx)


def rigid_apply(x, R, T=None):
    """R (x + T) per row; x numpy (N,3) or torch (N,3)."""
    cols = [x[:, k] + float(T[k]) if T is not None else x[:, k] for k in range(3)]
    out = [(cols[0] * float(R[k][0]) + cols[1] * float(R[k][1])) + cols[2] * float(R[k][2])
           for k in range(3)]
    if type(x).__module__.startswith("torch"):
        import torch

        return torch.stack(out, dim=1)
    return np.stack(out, axis=1)
