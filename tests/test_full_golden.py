"""Full-length parity fixtures made by the REFERENCE itself
(tests/golden/make_golden.py `full`): config 2 (4 096 rows), config 4
(8 192 rows), 68 config-5 streams with all 8 right-hand sides (including
streams on which the reference runs away past the construction rank) and 64
config-3 streams.  The fixtures store only outputs (branch log, the
reference's rank-test margin rho per row, rank, x) plus a sha256 of the
inputs, which are regenerated from the seeds with a fixed-order product
(workloads.ordered_product) so they have the same bits on any machine.

CPU half: the input pins and the C oracle against the reference.  The GPU
half (librgb.so against the same fixtures) is tests/test_gpu_full_length.py."""

import numpy as np
import pytest

from oracle import oracle
from paper_2106_11594_b200 import workloads
from rgb_testutil import compare_branches, relerr


def test_input_digests_regenerate(golden):
    g = golden("full_c5.npz")
    for i in (0, 1, 2, 3, len(g["streams"]) - 1):
        A, Y = workloads.c5_stream(int(g["streams"][i]), ordered=True)
        assert workloads.input_digest(A, Y) == str(g["digest"][i])
    g = golden("full_c3.npz")
    for i in (0, 1, 63):
        A, y, _ = workloads.c3_stream(int(g["streams"][i]), ordered=True)
        assert workloads.input_digest(A, y) == str(g["digest"][i])
    A, y = workloads.c2(ordered=True)
    assert workloads.input_digest(A, y) == str(golden("full_c2.npz")["digest"])


def test_ordered_product_is_cpu_independent_arithmetic():
    """The fixed-order product equals a plain Python loop with separate
    multiply / add roundings (what any IEEE machine computes)."""
    rng = np.random.default_rng(7)
    L, R = rng.standard_normal((5, 9)), rng.standard_normal((9, 4))
    A = workloads.ordered_product(L, R)
    for i in range(5):
        for j in range(4):
            acc = 0.0
            for t in range(9):
                acc = acc + L[i, t] * R[t, j]
            assert A[i, j] == acc


def _oracle_vs_reference(g, rows, tg, r_cap, x_tol=1e-9):
    o = oracle.ingest(rows, tg, r_cap=r_cap, nthreads=8)
    S = rows.shape[0]
    cmp = compare_branches(o["branch"], o["nobs"], g["branch"], g["rho"], got_rho=o["rho"])
    assert cmp["outside_disagree"] == 0, cmp["disagreements"]
    X = oracle.solution(o)
    xr = g["x"].reshape(S, rows.shape[2], -1)
    same = [b for b in range(S) if o["status"][b] == 0 and np.array_equal(o["branch"][b], g["branch"][b])]
    for b in same:
        assert int(o["rank"][b]) == int(np.atleast_1d(g["rank"])[b])
        assert relerr(X[b], xr[b]) <= x_tol, b
    return cmp, o


def test_oracle_c5_full_length_against_reference(golden):
    g = golden("full_c5.npz")
    rows, tg = workloads.host_batch("c5", [int(b) for b in g["streams"]], ordered=True)
    cmp, o = _oracle_vs_reference(g, rows, tg, r_cap=1024)
    runaway = np.nonzero(g["rank"] > 16)[0]
    assert len(runaway) >= 1  # the fixture holds at least one reference runaway
    # the first 60 streams are well conditioned: identical branch logs; the
    # last 8 were picked because the oracle runs away on them (the reference
    # does on 2): they are where the two sequential fp64 codes part
    assert cmp["exact"] >= 60
    assert all(b >= 60 for b, *_ in cmp["disagreements"])


def test_oracle_c3_full_length_against_reference(golden):
    g = golden("full_c3.npz")
    rows, tg = workloads.host_batch("c3", [int(b) for b in g["streams"]], ordered=True)
    cmp, _ = _oracle_vs_reference(g, rows, tg, r_cap=32)
    assert cmp["exact"] == 64


def test_oracle_c2_full_length_against_reference(golden):
    g = golden("full_c2.npz")
    A, y = workloads.c2(ordered=True)
    cmp, _ = _oracle_vs_reference({"branch": g["branch"][None], "rho": g["rho"][None], "rank": g["rank"],
                                   "x": g["x"][None]}, A[None], y[None, :, None], r_cap=64)
    assert cmp["exact"] == 1


def test_oracle_c4_prefix_against_reference(golden):
    """Config 4: the oracle's branch log over the first 640 rows (the 512 growth
    rows plus 128 dependent rows at full rank) -- the full-length run is on the
    GPU side, where it takes milliseconds instead of a minute."""
    g = golden("full_c4.npz")
    assert int(g["rank"]) == 512
    A, y = workloads.c4(ordered=True)
    assert workloads.input_digest(A, y) == str(g["digest"])
    n = 640
    o = oracle.ingest(np.ascontiguousarray(A[None, :n]), np.ascontiguousarray(y[None, :n, None]), r_cap=512)
    assert np.array_equal(o["branch"][0], g["branch"][:n])
