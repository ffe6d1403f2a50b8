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


# -- branch parity with the rank-test ambiguity band ------------------------------

# A dependent row's rejection is rounding noise whose size depends on the
# summation order and on the rounding history of the factors, so two correct
# fp64 implementations can take opposite branches on a row whose margin
# rho = |rej| / (eps max(1, |a|)) is within a small factor of 1 (SURVEY.md
# section 7, hard part 1).  Measured (tests/golden/full_c5.npz, the C oracle
# against the reference, both sequential fp64): on the ill-conditioned streams
# where one of them runs away, the first disagreement sits at a reference
# margin as low as 0.111 while the other side's margin at that row is
# 1.05-1.91; well-conditioned streams keep every dependent margin below 0.03.
# The band is therefore [1/16, 16], and a first disagreement must lie inside it
# on BOTH sides (the device side's margin is measured by replay where needed).
BAND = (1.0 / 16.0, 16.0)


def compare_branches(got_branch, got_nobs, ref_branch, ref_rho, band=BAND, got_rho=None):
    """Row-by-row branch comparison of a run against a reference trace.

    For every stream the first row where the two branch logs differ is found;
    everything after it is a different trajectory and is not compared.  A
    first disagreement is allowed only on a row whose reference margin (and
    the run's own margin, when ``got_rho`` is given) lies in ``band``; one
    outside is a parity failure.  Streams the run froze (``got_nobs`` < rows)
    are compared over the rows it folded.

    Returns counts: ``exact`` (every folded row agrees), ``band_disagree``
    (first disagreement inside the band) and ``outside_disagree`` (must be
    0), ``streams_with_band_rows``, and the ``disagreements`` as
    (stream, row, rho_ref, rho_got or None)."""
    got_branch = np.asarray(got_branch)
    ref_branch = np.asarray(ref_branch)
    ref_rho = np.asarray(ref_rho, dtype=np.float64)
    S, T = ref_branch.shape
    out = {"streams": S, "exact": 0, "band_disagree": 0, "outside_disagree": 0, "streams_with_band_rows": 0,
           "band": list(band), "disagreements": []}
    for b in range(S):
        n = int(got_nobs[b]) if got_nobs is not None else T
        rho = ref_rho[b, :n]
        if ((rho >= band[0]) & (rho <= band[1])).any():
            out["streams_with_band_rows"] += 1
        diff = np.nonzero(got_branch[b, :n] != ref_branch[b, :n])[0]
        if diff.size == 0:
            out["exact"] += 1
            continue
        i = int(diff[0])
        r = float(ref_rho[b, i])
        rg = None if got_rho is None else float(got_rho[b, i])
        inside = band[0] <= r <= band[1] and (rg is None or band[0] <= rg <= band[1])
        out["band_disagree" if inside else "outside_disagree"] += 1
        out["disagreements"].append((b, i, r, rg))
    return out


def agreeing_streams(got_branch, got_nobs, ref_branch):
    """Streams whose folded rows all take the reference's branch."""
    T = ref_branch.shape[1]
    return np.array([bool(np.array_equal(got_branch[b, :int(got_nobs[b])], ref_branch[b, :int(got_nobs[b])]))
                     and int(got_nobs[b]) == T for b in range(ref_branch.shape[0])])
