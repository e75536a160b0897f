"""Host loss helpers of the trainer seam (`trainer.py:96-120`) against the oracle, and
the reference's empty-input errors.  CPU only."""

from __future__ import annotations

import numpy as np
import pytest

from oracle import train as otrain
from paper_2212_05231_b200 import trainer as ptrain


def test_color_and_eikonal_loss_match_oracle():
    rng = np.random.default_rng(0)
    rendered, target = rng.random((257, 3)), rng.random((257, 3))
    assert ptrain.color_loss(rendered, target, 0.1) == otrain.color_loss(rendered, target, 0.1)
    n = rng.standard_normal((1000, 3)).astype(np.float32)
    nn = np.linalg.norm(n, axis=1)
    assert ptrain.eikonal_loss(n) == pytest.approx(float(((nn - 1.0) ** 2).mean()), rel=1e-12)


def test_loss_empty_inputs_raise():
    with pytest.raises(ValueError, match="need at least one ray"):
        ptrain.color_loss(np.zeros((0, 3)), np.zeros((0, 3)), 0.1)
    with pytest.raises(ValueError, match="need at least one normal"):
        ptrain.eikonal_loss(np.zeros((0, 3)))
    with pytest.raises(ValueError, match="psnr: shape mismatch"):
        ptrain.psnr(np.zeros((2, 3)), np.zeros((3, 3)))
