"""Parity metrics shared by the tests.

Per tensor: ||a-b||_2 / ||b||_2 <= tol  and  max|a-b| <= tol * max|b|.
Integer / index tensors are compared bit-exactly with np.array_equal.
"""

from __future__ import annotations

import numpy as np


def rel_err(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    den = np.linalg.norm(b.ravel())
    num = np.linalg.norm((a - b).ravel())
    if den == 0:
        return float(num)
    return float(num / den)


def max_err(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    scale = np.max(np.abs(b)) if b.size else 0.0
    d = np.max(np.abs(a - b)) if b.size else 0.0
    return float(d / scale) if scale > 0 else float(d)


def assert_close(a, b, tol, name="", max_tol=None):
    a = np.asarray(a)
    b = np.asarray(b)
    assert a.shape == b.shape, f"{name}: shape {a.shape} vs {b.shape}"
    r = rel_err(a, b)
    m = max_err(a, b)
    mt = tol if max_tol is None else max_tol
    assert r <= tol and m <= mt, f"{name}: relL2 {r:.3e} (tol {tol:.1e}), max {m:.3e} (tol {mt:.1e})"
    return r, m


def assert_exact(a, b, name=""):
    a = np.asarray(a)
    b = np.asarray(b)
    assert a.shape == b.shape, f"{name}: shape {a.shape} vs {b.shape}"
    if not np.array_equal(a, b):
        bad = np.flatnonzero(a.ravel() != b.ravel())
        raise AssertionError(f"{name}: {bad.size} mismatches, first at {bad[:8]}")
