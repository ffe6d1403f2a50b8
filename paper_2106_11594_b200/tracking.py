"""Drop-in trackers over the device factors (mirrors rankrls.tracking).

The reference updates A+ column by column in Theta(mn) per row
(tracking.py:76-85) and V = A+ A+^T in O(m^2) per row (tracking.py:103-119).
Here the solver only logs each row's coordinate-factor row (the rows of B in
A = B C, tracking.py:59-74) and the trackers evaluate the closed forms

    A+ = C~^T P^-1 B^T        (pinned by test_tracking.py:87-98)
    V  = C~^T P^-1 C~         (pinned by test_tracking.py:188-198)

on demand with one librgb.so launch (rgb_pinv / rgb_covariance).
"""

from __future__ import annotations

import numpy as np

from .scalars import FLOAT64
from .solver import RecursiveSolver, _readonly


class PseudoinverseTracker:
    """Pseudoinverse of all ingested observations (tracking.py:19-46)."""

    def __init__(self, solver):
        if solver.num_observations:
            raise ValueError("attach trackers before ingesting observations")
        self._solver = solver
        solver._trackers.append(self)

    def _coords_padded(self):
        s = self._solver
        cap = s._bs.r_cap
        chunks = [np.pad(c, ((0, 0), (0, cap - c.shape[1]))) for c in s._coords_chunks]
        if not chunks:
            return np.zeros((0, cap), dtype=s._kind.dtype)
        return np.concatenate(chunks, axis=0)

    @property
    def coords(self):
        """n x r coordinate factor B (read-only)."""
        return _readonly(self._coords_padded()[:, : self._solver.rank])

    @property
    def pinv(self):
        """Current m x n pseudoinverse (read-only host copy)."""
        s = self._solver
        Bf = self._coords_padded()
        n = Bf.shape[0]
        if n == 0:
            return _readonly(np.zeros((s.num_regressors, 0), dtype=s._kind.dtype))
        torch = s._torch
        t = torch.as_tensor(Bf, device=s._bs.device).view(1, n, -1)
        return _readonly(s._bs.pinv(t)[0].cpu().numpy())


class CovarianceTracker:
    """V = A+ (A+)^T across solver updates (tracking.py:88-101)."""

    def __init__(self, solver):
        if solver.num_observations:
            raise ValueError("attach trackers before ingesting observations")
        self._solver = solver
        solver._trackers.append(self)

    @property
    def covariance(self):
        return _readonly(self._solver._bs.covariance()[0].cpu().numpy())


def pinv_from_scratch(matrix, *, variant="general", eps=None, scalar=FLOAT64, alpha=1):
    """Pseudoinverse of a whole matrix by streaming its rows (tracking.py:128-142)."""
    A = scalar.matrix(matrix)
    n, m = A.shape
    solver = RecursiveSolver(m, variant=variant, eps=eps, scalar=scalar, alpha=alpha)
    tracker = PseudoinverseTracker(solver)
    if n:
        solver.ingest(A, np.zeros(n, dtype=scalar.dtype))
    return np.array(tracker.pinv, copy=True)
