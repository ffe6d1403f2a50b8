"""The reference's own property pins for this path,
run through the drop-in API on the GPU: Gram-inverse identity and symmetry
(test_solver.py:345-355), zero-residual dependent update (test_solver.py:331-342),
Penrose residuals (test_tracking.py:101-111), variant agreement and covariance
(test_acceptance.py:181-213), solve_batch small systems (test_solver.py:192-209)."""

import numpy as np
import pytest

from rgb_testutil import conditioned_stream, penrose_residuals

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


def test_gram_inverse_matches_reconstructed_coordinates():
    import paper_2106_11594_b200 as p

    rng = np.random.default_rng(47)
    A = conditioned_stream(rng, 9, 5, 3)
    s = p.RecursiveSolver(5)
    s.ingest(A, rng.standard_normal(9))
    _, _, P = s.basis()
    B = np.array([s.project(row).coords for row in A])
    assert np.abs(P @ (B.T @ B) - np.eye(s.rank)).max() <= 1e-8
    assert np.abs(P - P.T).max() <= 1e-12


def test_dependent_update_with_zero_residual_leaves_x_unchanged():
    """Exact integers, so a.x is exact in any summation order and the residual is 0."""
    import paper_2106_11594_b200 as p

    s = p.RecursiveSolver(3)
    s.ingest([[1, 0, 0], [0, 1, 0]], [2, 3])
    before = np.array(s.solution, copy=True)
    rep = s.update([4, -2, 0], 2.0)  # 4*2 - 2*3
    assert rep.branch == "dependent"
    assert np.array_equal(s.solution, before)


def test_penrose_residuals_small_float_suite():
    import paper_2106_11594_b200 as p

    rng = np.random.default_rng(9)
    for _ in range(25):
        n, m = (int(v) for v in rng.integers(1, 10, 2))
        r = int(rng.integers(1, min(n, m) + 1))
        head = conditioned_stream(rng, r, m, r)
        A = np.vstack([head, rng.standard_normal((n, r)) @ head])
        assert max(penrose_residuals(A, p.pinv_from_scratch(A))) <= 1e-9


def test_variant_agreement_and_covariance():
    import paper_2106_11594_b200 as p

    rng = np.random.default_rng(909)
    worst = 0.0
    for _ in range(50):
        n = int(rng.integers(1, 101))
        m = int(rng.integers(1, 51))
        r = int(rng.integers(1, min(n, m) + 1))
        A = conditioned_stream(rng, n, m, r)
        y = rng.standard_normal(n)
        xs = [p.solve_batch(A, y, variant=v)[0] for v in p.VARIANTS]
        scale = max(1.0, float(np.abs(xs[0]).max()))
        for i in range(3):
            for j in range(i + 1, 3):
                worst = max(worst, float(np.abs(xs[i] - xs[j]).max()) / scale)
    assert worst <= 1e-8, worst
    for _ in range(10):
        n = int(rng.integers(1, 21))
        m = int(rng.integers(1, 21))
        r = int(rng.integers(1, min(n, m) + 1))
        A = conditioned_stream(rng, n, m, r)
        s = p.RecursiveSolver(m)
        tr = p.PseudoinverseTracker(s)
        cov = p.CovarianceTracker(s)
        for row in A:
            s.update(row, float(rng.standard_normal()))
            assert np.abs(cov.covariance - tr.pinv @ tr.pinv.T).max() <= 1e-9


def test_solve_batch_small_systems():
    import paper_2106_11594_b200 as p

    x, rank = p.solve_batch(np.eye(2), [1.0, 2.0])
    assert rank == 2 and np.allclose(x, [1, 2])
    x, rank = p.solve_batch([[1.0, 0.0], [2.0, 0.0]], [1.0, 2.0])
    assert rank == 1 and np.allclose(x, [1, 0])
    x, rank = p.solve_batch([[1.0, 0.0], [1.0, 0.0]], [0.0, 2.0])
    assert rank == 1 and np.allclose(x, [1, 0])
