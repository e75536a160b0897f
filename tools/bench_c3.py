"""Config 3: SDF forward + analytic normal + Eikonal backward on 2^22
points, the analytic second-order path (Theorem 1 / Eq. 9, the tcgen05 field kernels
through field.eval_field / field.field_backward) against torch.autograd's double
backward of the same field written in plain PyTorch fp32.

    python tools/bench_c3.py [--points 22] [--order uniform|rays]

Prints one JSON line: per-step ms of both, their ratio and the relative L2 distance
of the table / SDF-layer gradients.  Run on the GPU box.
"""

from __future__ import annotations

import argparse
import json
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

from paper_2212_05231_b200 import field as pfield  # noqa: E402
from paper_2212_05231_b200 import trainer  # noqa: E402

P1, P2 = 2654435761, 805459861


def torch_sdf(x, tables, resolutions, lo, ext, h1, h2):
    """SDF value of the reference field (field.py:208-221) in autograd-able torch, in
    the dtype of `tables` with the reference's coordinate numerics: the normalised
    coordinate is fp32 (hash_encoding.py:102-106) and t = x n is formed in fp64
    (_kernels.py:20-29), so both precisions select the reference's cells."""
    dt = tables.dtype
    T = tables.shape[1]
    xn = ((x.float() - lo.float()) / ext.float()).clamp(0.0, 1.0)
    feats = []
    for l, n in enumerate(resolutions):
        t = xn.double() * float(n)
        c = (torch.ceil(t.detach()) - 1).clamp(0, n - 1)
        fr = (t - c).to(dt)
        ci = c.to(torch.int64)
        dense = (n + 1) ** 3 <= T
        acc = 0.0
        for cidx in range(8):
            o = torch.tensor([(cidx >> 2) & 1, (cidx >> 1) & 1, cidx & 1], device=x.device)
            cc = ci + o
            if dense:
                row = cc[:, 0] + cc[:, 1] * (n + 1) + cc[:, 2] * (n + 1) ** 2
            else:
                row = (cc[:, 0] ^ (cc[:, 1] * P1) ^ (cc[:, 2] * P2)) % T
            w = torch.where(o.bool(), fr, 1.0 - fr).prod(dim=1, keepdim=True)
            acc = acc + w * tables[l][row]
        feats.append(acc)
    xe = x.to(dt)
    e = torch.cat([xe] + feats + [torch.ones_like(xe[:, :1])], dim=1)
    a1 = torch.relu(e @ h1.T)
    return (a1 @ h2.T)[:, 0]


_OFFS = {}


def torch_sdf_vec(x, tables, resolutions, lo, ext, h1, h2):
    """The same SDF as `torch_sdf`, vectorised: all levels and all 8 corners of a point
    in one index tensor (L, P, 8) and ONE gather from the flattened tables, weights as
    one (L, P, 8) product -- the fair plain-PyTorch formulation of the encoding."""
    dt = tables.dtype
    L, T = tables.shape[0], tables.shape[1]
    dev = x.device
    key = (dev, L)
    if key not in _OFFS:
        o = torch.tensor([[(c >> 2) & 1, (c >> 1) & 1, c & 1] for c in range(8)], device=dev)
        res = torch.tensor(resolutions, device=dev, dtype=torch.int64)
        dense = (res + 1) ** 3 <= T
        _OFFS[key] = (o, res, dense)
    o, res, dense = _OFFS[key]
    xn = ((x.float() - lo.float()) / ext.float()).clamp(0.0, 1.0)
    t = xn.double()[None] * res[:, None, None].double()              # (L, P, 3)
    c = (torch.ceil(t.detach()) - 1).clamp(min=0)
    c = torch.minimum(c, (res - 1)[:, None, None].double())
    fr = (t - c).to(dt)                                               # (L, P, 3)
    cc = c.to(torch.int64)[:, :, None, :] + o[None, None]             # (L, P, 8, 3)
    n1 = (res + 1)[:, None, None]
    row_d = cc[..., 0] + cc[..., 1] * n1 + cc[..., 2] * n1 * n1
    row_h = (cc[..., 0] ^ (cc[..., 1] * P1) ^ (cc[..., 2] * P2)) % T
    row = torch.where(dense[:, None, None], row_d, row_h)
    row = row + (torch.arange(L, device=dev) * T)[:, None, None]
    ob = o.bool()[None, None]                                         # (1, 1, 8, 3)
    w = torch.where(ob, fr[:, :, None, :], 1.0 - fr[:, :, None, :]).prod(dim=3)  # (L, P, 8)
    v = tables.reshape(L * T, -1)[row]                                # (L, P, 8, F)
    feats = (w[..., None] * v).sum(dim=2)                             # (L, P, F)
    feats = feats.permute(1, 0, 2).reshape(x.shape[0], -1)
    xe = x.to(dt)
    e = torch.cat([xe, feats, torch.ones_like(xe[:, :1])], dim=1)
    a1 = torch.relu(e @ h1.T)
    return (a1 @ h2.T)[:, 0]


def autograd_step(x, tables, resolutions, lo, ext, h1, h2, chunk=1 << 18, sdf=None):
    """Eikonal loss mean((|grad_x d| - 1)^2) and its parameter gradients by double
    backward, in chunks of points (the mean is split exactly) to bound autograd memory."""
    n_all = x.shape[0]
    grads = [torch.zeros_like(tables), torch.zeros_like(h1), torch.zeros_like(h2)]
    total = 0.0
    for s in range(0, n_all, chunk):
        xc = x[s:s + chunk].detach().to(tables.dtype).requires_grad_(True)
        d = (sdf or torch_sdf)(xc, tables, resolutions, lo, ext, h1, h2)
        (n,) = torch.autograd.grad(d.sum(), xc, create_graph=True)
        loss = ((n.norm(dim=1) - 1.0) ** 2).sum() / n_all
        g = torch.autograd.grad(loss, [tables, h1, h2])
        for acc, gi in zip(grads, g):
            acc += gi
        total += float(loss.detach())
    return total, grads


def ours_step(params, x):
    cache = pfield.eval_field(params, x, need_color=False)
    n = cache.normals
    nn = n.norm(dim=1, keepdim=True)
    dl_dn = (2.0 * (nn - 1.0) / nn.clamp_min(1e-12) * n / x.shape[0]).float()
    gr = pfield.field_backward(params, cache, dl_dn=dl_dn)
    return ((nn - 1.0) ** 2).mean(), gr


def setup(points, order, seed=0):
    cfg = trainer.TrainConfig(num_levels=16, table_size=2**19, seed=seed, level_init=16)
    st = trainer.TrainState.create(cfg)
    p = st.params
    # trained-like tables so the second-order terms are not negligible
    g = torch.Generator(device="cuda").manual_seed(1)
    p.grid.tables.uniform_(-0.1, 0.1, generator=g)
    n = 1 << points
    if order == "uniform":
        x = torch.rand((n, 3), generator=g, device="cuda") * 2 - 1
    else:  # ray-ordered: fixed-stride samples along rays, kept strictly inside the box
        rays = 1 << max(points - 5, 1)
        o = torch.randn((rays, 3), generator=g, device="cuda", dtype=torch.float64)
        o = 2.6 * o / o.norm(dim=1, keepdim=True)
        tgt = (torch.rand((rays, 3), generator=g, device="cuda", dtype=torch.float64) - 0.5) * 0.8
        d = tgt - o
        d = d / d.norm(dim=1, keepdim=True)
        t = 2.6 - 1.0 + torch.linspace(0, 2.0, 128, device="cuda", dtype=torch.float64)
        x = (o[:, None, :] + t[None, :, None] * d[:, None, :]).reshape(-1, 3).float()
        x = x[(x.abs() < 1).all(dim=1)][:n]
    return p, x.contiguous()


def rel(a, b):
    a, b = a.double(), b.double()
    return float((a - b).norm() / b.norm().clamp_min(1e-30))


def _autograd_at(p, x, dtype):
    res = p.grid.resolutions.tolist()
    lo = torch.tensor(p.grid.aabb_min, device="cuda", dtype=dtype)
    ext = torch.tensor(p.grid.aabb_extent, device="cuda", dtype=dtype)
    args = [t.detach().clone().to(dtype).requires_grad_(True)
            for t in (p.grid.tables, p.sdf_net.layers[0], p.sdf_net.layers[1])]
    return autograd_step(x, args[0], res, lo, ext, args[1], args[2], sdf=torch_sdf_vec)


def compare(points=14, order="uniform"):
    """Eikonal loss and gradients of the tcgen05 path and of torch fp32 autograd, each
    against torch fp64 autograd (the exact reference for both)."""
    p, x = setup(points, order)
    l64, g64 = _autograd_at(p, x, torch.float64)
    l32, g32 = _autograd_at(p, x, torch.float32)
    lo_, gr = ours_step(p, x)
    ours = (gr.tables, gr.sdf_layers[0], gr.sdf_layers[1])
    out = {"loss": (float(lo_), float(l32), float(l64))}
    for k, a, b, ref in zip(("tables", "h1", "h2"), ours, g32, g64):
        out[k] = (rel(a, ref), rel(b, ref))
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--points", type=int, default=22)
    ap.add_argument("--order", default="uniform", choices=["uniform", "rays"])
    ap.add_argument("--iters", type=int, default=5)
    ap.add_argument("--compile", action="store_true", help="also time a torch.compile'd baseline")
    ap.add_argument("--check64", action="store_true",
                    help="accuracy of ours and torch fp32 against torch fp64 double backward at --points")
    a = ap.parse_args()
    if a.check64:
        print(json.dumps({"config": f"c3 accuracy vs torch fp64 double backward, 2^{a.points} points ({a.order})",
                          **compare(a.points, a.order)}))
        return
    p, x = setup(a.points, a.order)
    res = p.grid.resolutions.tolist()
    lo = torch.tensor(p.grid.aabb_min, device="cuda", dtype=torch.float32)
    ext = torch.tensor(p.grid.aabb_extent, device="cuda", dtype=torch.float32)
    tab = p.grid.tables.detach().clone().requires_grad_(True)
    h1 = p.sdf_net.layers[0].detach().clone().requires_grad_(True)
    h2 = p.sdf_net.layers[1].detach().clone().requires_grad_(True)

    def timed(fn):
        for _ in range(2):
            fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(a.iters):
            out = fn()
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / a.iters, out

    t_ours, (lo_, gr) = timed(lambda: ours_step(p, x))
    out = {"config": f"c3: SDF fwd + normal + Eikonal bwd, 2^{a.points} points ({a.order}), 16 levels 2^19",
           "points": x.shape[0], "ours_ms": t_ours, "loss_ours": float(lo_), "baselines": {}}
    variants = {"loop": torch_sdf, "vectorised": torch_sdf_vec}
    if a.compile:
        variants["vectorised+torch.compile"] = torch.compile(torch_sdf_vec, dynamic=False)
    for name, fn in variants.items():
        try:
            t_ag, (la, (gt, g1, g2)) = timed(lambda: autograd_step(x, tab, res, lo, ext, h1, h2, sdf=fn))
            out["baselines"][name] = {
                "autograd_ms": t_ag, "speedup": t_ag / t_ours, "loss": float(la),
                "grad_rel_l2": {"tables": rel(gr.tables, gt), "h1": rel(gr.sdf_layers[0], g1),
                                "h2": rel(gr.sdf_layers[1], g2)}}
        except Exception as exc:  # e.g. torch.compile without double-backward support
            out["baselines"][name] = {"unavailable": f"{type(exc).__name__}: {str(exc).splitlines()[0][:200]}"}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
