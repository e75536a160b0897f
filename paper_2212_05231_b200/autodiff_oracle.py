"""Theorem-1 benchmark (`autodiff_oracle.py:208-270`): the analytic second-order MLP
backward against a generic graph autodiff of the same quantity.

The reference times its numpy `relu_mlp.backward_second` against its own small
reverse-mode graph (`Node`/`backward`, :22-205) on the CPU.  Here both sides run on the
device: the analytic side is `relu_mlp.backward_second` (batched GEMMs, masks constant),
the generic side is torch.autograd differentiating sum_p <M_p, (dy/dx)_p> twice (one
create_graph VJP per output row to build dy/dx, then the gradient with respect to every
layer).  Timing is CUDA events on the current stream, median over `runs`.  On the
training step itself the same contraction runs fused in the tcgen05 MLP backward
(`tools/bench_c3.py` times that against torch double backward).
"""

from __future__ import annotations

import numpy as np
import torch

from . import relu_mlp

__all__ = ["graph_grad_of_grad", "bench_second_order", "bench_rows_to_csv"]


def graph_grad_of_grad(weights, x, jac_cotangent):
    """Gradients of sum_p <M_p, dy/dx_p> w.r.t. each layer by generic double autodiff
    (the role of `oracle_grad_of_grad`, `autodiff_oracle.py:181-205`)."""
    hs = [h.detach().clone().requires_grad_(True) for h in weights.layers]
    xb = x.detach().clone().requires_grad_(True)
    a = xb
    for h in hs[:-1]:
        a = torch.relu(a @ h.T)
    y = a @ hs[-1].T
    total = 0.0
    for i in range(y.shape[1]):
        (row,) = torch.autograd.grad(y[:, i].sum(), xb, create_graph=True)
        total = total + (row * jac_cotangent[:, i, :]).sum()
    return list(torch.autograd.grad(total, hs))


def _median_ms(fn, runs):
    times = []
    for _ in range(runs):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        fn()
        e.record()
        e.synchronize()
        times.append(s.elapsed_time(e))
    return float(np.median(times))


def bench_second_order(width, depth, batch_sizes, rng=None, runs=20):
    """Square MLP (all dims `width`, `depth` matrices), fp32, generic Jacobian
    cotangent; one dict per batch size with median microseconds per backward and the
    speed-up (`autodiff_oracle.py:208-258`).  Refuses to time disagreeing paths."""
    rng = rng or np.random.default_rng(0)
    dims = [width] * (depth + 1)
    weights = relu_mlp.MlpWeights.random(dims, rng)
    dev = weights.layers[0].device
    rows = []
    for batch in batch_sizes:
        x = torch.from_numpy(rng.standard_normal((batch, width)).astype(np.float32)).to(dev)
        m = torch.from_numpy(rng.standard_normal((batch, width, width)).astype(np.float32)).to(dev)

        def run_analytic():
            _, trace = relu_mlp.forward(weights, x)
            return relu_mlp.backward_second(weights, trace, m)

        def run_graph():
            return graph_grad_of_grad(weights, x, m)

        for a, b in zip(run_analytic(), run_graph()):
            scale = float(b.abs().max()) + 1e-12
            if float((a - b).abs().max()) > 2e-2 * scale:
                raise AssertionError("analytic and graph second-order gradients disagree")
        run_analytic(), run_graph()  # warm-up
        t_a = _median_ms(run_analytic, runs) * 1e3
        t_g = _median_ms(run_graph, runs) * 1e3
        rows.append({"width": width, "depth": depth, "batch": batch, "analytic_us": t_a,
                     "oracle_us": t_g, "speedup": t_g / t_a})
    return rows


def bench_rows_to_csv(rows):
    """`autodiff_oracle.py:261-270`."""
    lines = ["width,depth,batch,analytic_us,oracle_us,speedup"]
    lines += [f"{r['width']},{r['depth']},{r['batch']},{r['analytic_us']:.1f},{r['oracle_us']:.1f},"
              f"{r['speedup']:.2f}" for r in rows]
    return "\n".join(lines) + "\n"
