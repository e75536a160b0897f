"""tcgen05 building blocks (csrc/umma.cuh) against an fp64 host reference."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2212_05231_b200 import _lib  # noqa: E402


def run(mode, A, B, dshape):
    a = torch.from_numpy(A.astype(np.float32)).cuda()
    b = torch.from_numpy(B.astype(np.float32)).cuda()
    d = torch.full(dshape, float("nan"), dtype=torch.float32, device="cuda")
    _lib.call("ns2b_selftest_umma", _lib.ptr(a), _lib.ptr(b), _lib.ptr(d), mode, _lib.stream_ptr())
    torch.cuda.synchronize()
    return d.cpu().numpy().astype(np.float64)


@pytest.mark.parametrize("mode", [0, 1, 2, 3, 4])
def test_umma_split_gemm(mode):
    rng = np.random.default_rng(mode)
    if mode in (0, 3):
        A = rng.standard_normal((128, 48)).astype(np.float32)
        B = rng.standard_normal((64, 48)).astype(np.float32)
        ref = A.astype(np.float64) @ B.astype(np.float64).T
        got = run(mode, A, B, (128, 64))
    elif mode in (1, 4):
        A = rng.standard_normal((128, 48)).astype(np.float32)
        B = rng.standard_normal((48, 64)).astype(np.float32)
        ref = A.astype(np.float64) @ B.astype(np.float64)
        got = run(mode, A, B, (128, 64))
    else:
        A = rng.standard_normal((128, 64)).astype(np.float32) * 1e-6  # cotangent-like range
        B = rng.standard_normal((128, 48)).astype(np.float32)
        ref = A.astype(np.float64).T @ B.astype(np.float64)
        got = run(mode, A, B, (64, 48))
    err = np.abs(got - ref).max() / np.abs(ref).max()
    bar = 2e-6 if mode in (0, 1, 4) else 5e-5  # f16x3 ~ fp32; bf16x3 ~ 2^-16
    assert np.isfinite(got).all(), "unwritten / NaN outputs"
    assert err < bar, f"mode {mode}: max rel err {err:.3e}"
