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


def penrose_residuals(A, P):
    """The four Penrose equations' 2-norm residuals (A P A = A and P A P = P
    scaled by |A|_2 and |P|_2, the symmetry of A P and P A by |A|_2 and |P|_2;
    a zero scale leaves the raw norm), restated from metrics.penrose_residuals
    (metrics.py:185-207)."""
    A = np.asarray(A, dtype=np.float64)
    P = np.asarray(P, dtype=np.float64)
    ap, pa = A @ P, P @ A
    an = float(np.linalg.norm(A, 2)) if A.size else 0.0
    pn = float(np.linalg.norm(P, 2)) if P.size else 0.0
    out = []
    for res, scale in ((ap @ A - A, an), (pa @ P - P, pn), (ap.T - ap, an), (pa.T - pa, pn)):
        nrm = float(np.linalg.norm(res, 2)) if res.size else 0.0
        out.append(nrm / scale if scale > 0.0 else nrm)
    return tuple(out)


def conditioned_stream(rng, n, m, r):
    """Rank-r rows whose first r are orthogonal with scales in [0.5, 2] and the
    rest random combinations of them (test_acceptance.py:31-38, test_solver.py:12-28)."""
    q, _ = np.linalg.qr(rng.standard_normal((m, r)))
    head = rng.uniform(0.5, 2.0, r)[:, None] * q.T
    if n > r:
        return np.vstack([head, rng.standard_normal((n - r, r)) @ head])
    return head[:n]
