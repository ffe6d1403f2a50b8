"""B200-native rank-Greville recursive least squares (arXiv 2106.11594).

Drop-in for the hot path of rankrls 0.1.0: the same solver API
(``RecursiveSolver``, ``solve_batch``, ``PseudoinverseTracker``,
``CovarianceTracker``, ``pinv_from_scratch``, ``EpsPolicy``) backed by
hand-written sm_100a kernels in ``librgb.so`` (C ABI: include/rgb.h), plus the
batched multi-stream / multi-RHS device API ``BatchedSolver``.
"""

from .scalars import FLOAT32, FLOAT64, KINDS, RATIONAL, CapabilityError, ScalarKind
from .solver import (
    VARIANTS,
    EpsPolicy,
    ProjectionResult,
    RecursiveSolver,
    UpdateReport,
    solve_batch,
)
from .tracking import CovarianceTracker, PseudoinverseTracker, pinv_from_scratch

__version__ = "0.1.0"


def BatchedSolver(*args, **kwargs):  # noqa: N802 -- lazy import keeps torch optional at import time
    from .batched import BatchedSolver as _B

    return _B(*args, **kwargs)


__all__ = [
    "FLOAT32", "FLOAT64", "KINDS", "RATIONAL", "CapabilityError", "ScalarKind",
    "VARIANTS", "EpsPolicy", "ProjectionResult", "RecursiveSolver", "UpdateReport",
    "solve_batch", "CovarianceTracker", "PseudoinverseTracker", "pinv_from_scratch",
    "BatchedSolver", "__version__",
]
