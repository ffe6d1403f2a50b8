"""Shared helpers for the parity tests."""

import os

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")


def relerr(got, want):
    """Error metric of test_acceptance.py:56-61: max|got-want| / max(1, max|want|)."""
    want = np.asarray(want, dtype=np.float64)
    got = np.asarray(got, dtype=np.float64)
    if want.size == 0:
        return 0.0
    return float(np.abs(got - want).max()) / max(1.0, float(np.abs(want).max()))


def load_golden(name):
    return np.load(os.path.join(GOLDEN, name))


def residual_error(pinv, A):
    """|P A - I|_2 / (|A|_2 |P|_2), restated from metrics.residual_error (metrics.py:168-182)."""
    A = np.asarray(A, dtype=np.float64)
    P = np.asarray(pinv, dtype=np.float64)
    return float(np.linalg.norm(P @ A - np.eye(A.shape[1]), 2)
                 / (np.linalg.norm(A, 2) * np.linalg.norm(P, 2)))
