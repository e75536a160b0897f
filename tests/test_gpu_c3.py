"""Config 3 parity: the analytic second-order Eikonal gradient of the
tcgen05 field kernels (Theorem 1 + Eq. 9) against torch.autograd's double backward of
the same SDF in plain PyTorch fp32 -- an oracle independent of oracle/."""

from __future__ import annotations

import sys
from pathlib import Path

import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

sys.path.insert(0, str(Path(__file__).resolve().parents[1] / "tools"))
import bench_c3  # noqa: E402


@pytest.mark.parametrize("order", ["uniform", "rays"])
def test_eikonal_second_order_matches_autograd(order):
    """Loss and gradients vs torch fp64 double backward within 1e-3 relL2 (or twice
    torch fp32 autograd's own distance from fp64, whichever is larger)."""
    r = bench_c3.compare(points=14, order=order)
    lo, l32, l64 = r["loss"]
    assert abs(lo - l64) <= max(1e-4 * abs(l64), 2 * abs(l32 - l64))
    for k in ("tables", "h1", "h2"):
        ours, t32 = r[k]
        assert ours <= max(1e-3, 2 * t32), f"{k}: relL2 {ours} (torch fp32: {t32})"
