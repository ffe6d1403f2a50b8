"""Pin the CPU oracle (oracle/rgb_oracle.c, oracle/oracle.py) against golden
vectors that the reference produced (tests/golden/make_golden.py).  CPU only."""

import numpy as np
import pytest

from oracle import oracle
from rgb_testutil import relerr, residual_error

VARIANTS = ("general", "orthogonal", "orthonormal")


def test_c1_branches_rank_x_pinv(golden):
    g = golden("c1.npz")
    out = oracle.ingest(g["A"][None], g["y"][None], r_cap=64)
    assert int(out["rank"][0]) == int(g["rank"])
    assert np.array_equal(out["branch"][0], g["branch"])
    assert relerr(oracle.solution(out)[0, :, 0], g["x"]) <= 1e-12
    assert relerr(oracle.pinv_closed_form(out), g["pinv"]) <= 1e-12
    # numpy restatement of the tracker is the reference's own op sequence
    assert relerr(oracle.pinv_tracker(g["A"]), g["pinv"]) <= 1e-15


@pytest.mark.parametrize("name", ["c5_sample.npz", "c3_sample.npz"])
def test_batched_samples(golden, name):
    g = golden(name)
    out = oracle.ingest(g["rows"], g["targets"], r_cap=64, nthreads=4)
    assert np.array_equal(out["rank"], g["rank"])
    assert np.array_equal(out["branch"], g["branch"])
    X = oracle.solution(out)
    for b in range(X.shape[0]):
        assert relerr(X[b], g["x"][b]) <= 1e-11


def test_variants_small_streams(golden):
    g = golden("variants.npz")
    for case in range(12):
        A, y = g[f"A{case}"], g[f"y{case}"]
        for v in VARIANTS:
            out = oracle.ingest(A[None], y[None], variant=v)
            assert int(out["rank"][0]) == int(g[f"{v}_rank{case}"])
            assert np.array_equal(out["branch"][0], g[f"{v}_branch{case}"])
            assert relerr(oracle.solution(out)[0, :, 0], g[f"{v}_x{case}"]) <= 1e-12
            assert relerr(oracle.pinv_closed_form(out, variant=v), g[f"{v}_pinv{case}"]) <= 1e-10
            assert relerr(oracle.pinv_tracker(A, variant=v), g[f"{v}_pinv{case}"]) <= 1e-15


def test_kahan_absolute_clause(golden):
    g = golden("kahan.npz")
    K = g["K"]
    out = oracle.ingest(K[None], np.zeros((1, 100)), eps=1e-8, r_cap=100)
    assert int(out["rank"][0]) == int(g["rank_fixed"]) == 99
    out = oracle.ingest(K[None], np.zeros((1, 100)), r_cap=100)
    assert int(out["rank"][0]) == int(g["rank_auto"])
    # kappa_2(K) = 2.2e9, so forward agreement is bounded by kappa * eps ~ 5e-7;
    # the reference's own stability band is the residual error <= 1e-14
    # (test_acceptance.py:159-178)
    pinv = oracle.pinv_closed_form(out)
    assert relerr(pinv, g["pinv_auto"]) <= 1e-6
    assert residual_error(pinv, K) <= 1e-14


def test_known_answers_update_sequence():
    # test_solver.py:134-149: (1,0)->(1,0)->(1,1) with targets 2, 4, 5
    out = oracle.ingest(np.array([[[1.0, 0], [1, 0], [1, 1]]]), np.array([[2.0, 4, 5]]))
    assert list(out["branch"][0]) == [1, 0, 1]
    assert np.allclose(oracle.solution(out)[0, :, 0], [3, 2])
    assert int(out["rank"][0]) == 2 and int(out["nobs"][0]) == 3
    # a-priori residuals: 2 - 0, 4 - 2, 5 - 3
    assert np.allclose(out["resid"][0, :, 0], [2, 2, 2])


def test_known_answers_zero_rows_and_duplicates():
    # test_solver.py:166-176: a zero row is a dependent no-op
    out = oracle.ingest(np.array([[[0.0, 0], [1, 0], [0, 0]]]), np.array([[7.0, 2, -3]]))
    assert list(out["branch"][0]) == [0, 1, 0]
    assert np.array_equal(oracle.solution(out)[0, :, 0], [2, 0])
    # test_solver.py:202-204: duplicated inconsistent rows average
    out = oracle.ingest(np.array([[[1.0, 0], [1, 0]]]), np.array([[0.0, 2]]))
    assert np.allclose(oracle.solution(out)[0, :, 0], [1, 0]) and out["rank"][0] == 1
    # test_tracking.py:18-21, 62-66: A+ of (1,1) and of [[1,1],[1,1]]
    assert np.allclose(oracle.pinv_tracker([[1.0, 1.0]]), [[0.5], [0.5]])
    assert np.allclose(oracle.pinv_tracker([[1.0, 1], [1, 1]]), 0.25 * np.ones((2, 2)))
    assert np.array_equal(oracle.pinv_tracker(np.zeros((2, 3))), np.zeros((3, 2)))


def test_rank_cap_overflow_freezes_stream():
    A = np.eye(4)[None]
    out = oracle.ingest(A, np.ones((1, 4)), r_cap=2)
    assert out["status"][0] & oracle.ST_RANK_CAP
    assert int(out["rank"][0]) == 2 and int(out["nobs"][0]) == 2


def test_multi_rhs_equals_separate_runs(golden):
    g = golden("c5_sample.npz")
    rows, tg = g["rows"][:2], g["targets"][:2]
    full = oracle.ingest(rows, tg, r_cap=16)
    for c in range(tg.shape[2]):
        one = oracle.ingest(rows, tg[:, :, c], r_cap=16)
        assert np.array_equal(oracle.solution(one)[:, :, 0], oracle.solution(full)[:, :, c])


def test_fp32_mode_runs_and_tracks_fp64_on_integer_stream(golden):
    g = golden("c5_sample.npz")
    rows, tg = g["rows"][1:2], g["targets"][1:2]   # odd stream: integer factors
    o64 = oracle.ingest(rows, tg, r_cap=16)
    o32 = oracle.ingest(rows.astype(np.float32), tg.astype(np.float32), r_cap=16, dtype=np.float32)
    assert int(o32["rank"][0]) == int(o64["rank"][0]) == 16
    assert relerr(oracle.solution(o32), oracle.solution(o64)) <= 1e-3
