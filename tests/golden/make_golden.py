"""Generate the golden parity fixtures by running the REFERENCE itself.

Run in the build container only (it imports rankrls from /root/reference,
which does not exist on the GPU box):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Every fixture records the reference's own outputs on seeded inputs:
per-row branch sequence (``RecursiveSolver.update().branch``, solver.py:231-250),
final rank, the solution of ``solve_batch`` (the ``ingest`` fast path,
solver.py:406-422; one call per right-hand side, since the reference has no
multi-RHS API) and, where noted, ``pinv_from_scratch`` (tracking.py:128-142).
The tests compare the C oracle and the CUDA path against these files.
"""

from __future__ import annotations

import os
import sys

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", ".."))

from rankrls import matrices, solver, tracking  # noqa: E402  (the reference)
from rankrls.solver import EpsPolicy  # noqa: E402

from paper_2106_11594_b200 import workloads  # noqa: E402  (input recipes only)

OUT = os.path.dirname(os.path.abspath(__file__))


def ref_stream(A, Y, variant="general", eps=None):
    """Reference branch log (update fold, RHS 0) and per-RHS solve_batch."""
    Y = np.asarray(Y, dtype=np.float64).reshape(A.shape[0], -1)
    s = solver.RecursiveSolver(A.shape[1], variant=variant, eps=eps)
    branch = np.array([s.update(row, t).branch == "independent" for row, t in zip(A, Y[:, 0])],
                      dtype=np.uint8)
    xs, rank = [], None
    for c in range(Y.shape[1]):
        x, rank = solver.solve_batch(A, Y[:, c], variant=variant, eps=eps)
        xs.append(x)
    return branch, np.stack(xs, axis=1), rank, s.solution.copy()


def conditioned_stream(rng, n, m, r):
    """Rank-r rows: r orthogonal rows scaled in [0.5, 2] then random
    combinations of them (the construction of test_solver.py:12-27)."""
    q, _ = np.linalg.qr(rng.standard_normal((m, r)))
    head = rng.uniform(0.5, 2.0, r)[:, None] * q.T
    if n > r:
        return np.vstack([head, rng.standard_normal((n - r, r)) @ head])
    return head[:n]


def main():
    # -- config 1, full size: x, branches, rank and A+ -----------------------
    A, y = workloads.c1()
    branch, X, rank, x_fold = ref_stream(A, y)
    np.savez_compressed(os.path.join(OUT, "c1.npz"), A=A, y=y, branch=branch, x=X[:, 0],
                        x_fold=x_fold, rank=rank, pinv=tracking.pinv_from_scratch(A))

    # -- config 5 sample: 3 Gaussian + 3 integer streams, first 192 rows -----
    streams = [0, 1, 2, 3, 4, 5]
    rows, tg = workloads.host_batch("c5", streams, n=192)
    br, xs, ranks = [], [], []
    for i in range(len(streams)):
        b_, X_, r_, _ = ref_stream(rows[i], tg[i])
        br.append(b_); xs.append(X_); ranks.append(r_)
    np.savez_compressed(os.path.join(OUT, "c5_sample.npz"), streams=np.array(streams),
                        rows=rows, targets=tg, branch=np.stack(br), x=np.stack(xs),
                        rank=np.array(ranks))

    # -- config 3 sample: 2 streams, first 256 rows ---------------------------
    streams = [0, 1]
    rows, tg = workloads.host_batch("c3", streams, n=256)
    br, xs, ranks = [], [], []
    for i in range(len(streams)):
        b_, X_, r_, _ = ref_stream(rows[i], tg[i])
        br.append(b_); xs.append(X_); ranks.append(r_)
    np.savez_compressed(os.path.join(OUT, "c3_sample.npz"), streams=np.array(streams),
                        rows=rows, targets=tg, branch=np.stack(br), x=np.stack(xs),
                        rank=np.array(ranks))

    # -- all three variants on well-conditioned small streams, with A+ --------
    rng = np.random.default_rng(2106)
    cases = {}
    for case in range(12):
        n = int(rng.integers(1, 30)); m = int(rng.integers(1, 24))
        r = int(rng.integers(1, min(n, m) + 1))
        A = conditioned_stream(rng, n, m, r)
        y = rng.standard_normal(n)
        cases[f"A{case}"] = A; cases[f"y{case}"] = y
        for v in solver.VARIANTS:
            branch, X, rank, _ = ref_stream(A, y, variant=v)
            cases[f"{v}_branch{case}"] = branch
            cases[f"{v}_x{case}"] = X[:, 0]
            cases[f"{v}_rank{case}"] = np.array(rank)
            cases[f"{v}_pinv{case}"] = tracking.pinv_from_scratch(A, variant=v)
    np.savez_compressed(os.path.join(OUT, "variants.npz"), **cases)

    # -- Kahan(100, 0.2): the absolute clause of the rank test ---------------
    # (test_stability_harness.py:32-45: fixed eps 1e-8 truncates to rank 99)
    K, _ = matrices.kahan(100, 0.2)
    s = solver.RecursiveSolver(100, eps=EpsPolicy.fixed(1e-8))
    s.ingest(K, np.zeros(100))
    np.savez_compressed(os.path.join(OUT, "kahan.npz"), K=K, rank_fixed=s.rank,
                        rank_auto=solver.solve_batch(K, np.zeros(100))[1],
                        pinv_auto=tracking.pinv_from_scratch(K))

    # -- Pascal(10) in float64 (stability band anchor, test_acceptance.py:159-178)
    P10 = matrices.pascal(10).astype(np.float64)
    np.savez_compressed(os.path.join(OUT, "pascal10.npz"), P=P10,
                        pinv=tracking.pinv_from_scratch(P10))
    for f in sorted(os.listdir(OUT)):
        if f.endswith(".npz"):
            print(f, os.path.getsize(os.path.join(OUT, f)))


def bench_cells():
    """Inputs of the reference's bench cells (bench.py:166-211) for two small
    plans, plus the reference's solve_batch of each solve cell: pins the
    cell-seeding of paper_2106_11594_b200.experiments."""
    from rankrls import bench

    out = {}
    plan = bench.make_plan("rank-fixed-r", [16, 32], fixed_r=4, seed=7)
    for i, (n, m, r) in enumerate(plan.grid):
        A = matrices.random_standardized(n, m, r, bench._cell_seed(plan, i, 0))
        y = np.random.default_rng(bench._cell_seed(plan, i, 1)).standard_normal(n)
        x, rank = solver.solve_batch(A, y)
        out.update({f"solve{i}_A": A, f"solve{i}_y": y, f"solve{i}_x": x, f"solve{i}_rank": rank})
    plan = bench.make_plan("update-cost", [4, 8], fixed_m=32, seed=1)
    for i, (r, m, _) in enumerate(plan.grid):
        rng = np.random.default_rng(bench._cell_seed(plan, i, 0))
        basis = rng.standard_normal((r, m))
        yb = rng.standard_normal(r)
        probes = rng.standard_normal((32, r)) @ basis
        out.update({f"upd{i}_basis": basis, f"upd{i}_y": yb, f"upd{i}_probes": probes,
                    f"upd{i}_targets": rng.standard_normal(32)})
    np.savez_compressed(os.path.join(OUT, "bench_cells.npz"), **out)


# -- full-length fixtures (outputs only; inputs regenerated from the seeds) ------

def ref_trace(A, Y):
    """The reference's ingest fast path (solver.py:252-319) one row at a time on
    one RecursiveSolver: branch per row (rank change), the rank-test margin
    rho = |rej| / (eps max(1, |a|)) from the reference's own `project`
    (solver.py:210-219) at the current rank, and x for every right-hand side
    from `solve_batch` (one call per RHS; the reference has no multi-RHS API).
    The one-row ingests must reproduce solve_batch's x bit for bit."""
    Y = np.asarray(Y, dtype=np.float64).reshape(A.shape[0], -1)
    n, m = A.shape
    s = solver.RecursiveSolver(m)
    eps_m = np.finfo(np.float64).eps
    branch = np.zeros(n, np.uint8)
    rho = np.zeros(n, np.float64)
    for i in range(n):
        r0 = s.rank
        p = s.project(A[i])
        eps = (m * m * r0 + m * r0 + m) * eps_m
        rho[i] = np.sqrt(float(p.rejection_sq_norm) / (eps * eps * max(1.0, float(np.dot(A[i], A[i])))))
        s.ingest(A[i:i + 1], Y[i:i + 1, 0])
        branch[i] = s.rank > r0
    xs = []
    rank = None
    for c in range(Y.shape[1]):
        x, rank = solver.solve_batch(A, Y[:, c])
        xs.append(x)
    assert rank == s.rank and np.array_equal(xs[0], s.solution), "one-row ingests != solve_batch"
    return branch, rho.astype(np.float32), rank, np.stack(xs, axis=1)


def _c5_trace(b):
    A, Y = workloads.c5_stream(b, ordered=True)
    return (b,) + ref_trace(A, Y) + (workloads.input_digest(A, Y),)


def _c3_trace(b):
    A, y, r = workloads.c3_stream(b, ordered=True)
    return (b,) + ref_trace(A, y) + (workloads.input_digest(A, y),)


def runaway_scan(count):
    """Host-seeded config-5 streams [0, count) whose C-oracle run leaves the
    construction rank (SURVEY.md finding 0.3): candidates for the golden's
    runaway streams (the reference itself decides which really run away)."""
    sys.path.insert(0, os.path.join(OUT, "..", ".."))
    from oracle import oracle

    found = []
    for c0 in range(0, count, 1024):
        rows, tg = workloads.host_batch("c5", range(c0, c0 + 1024), ordered=True)
        o = oracle.ingest(rows, tg, r_cap=17, nthreads=os.cpu_count() or 8, logs=False)
        found += [c0 + int(i) for i in np.nonzero(o["status"] & 1)[0]]
    return found


def full_length():
    """Reference-run full-length fixtures for every config:
    C2 (4 096 rows), C4 (8 192 rows), 64 C5 streams with all 8 RHS plus streams
    on which the reference runs away, 64 C3 streams."""
    from multiprocessing import Pool

    os.environ["OPENBLAS_NUM_THREADS"] = "1"
    for name, fn in (("c2", workloads.c2), ("c4", workloads.c4)):
        A, y = fn(ordered=True)
        branch, rho, rank, X = ref_trace(A, y)
        np.savez_compressed(os.path.join(OUT, f"full_{name}.npz"), digest=workloads.input_digest(A, y),
                            branch=branch, rho=rho, rank=rank, x=X[:, 0])
        print(name, "rank", rank, "max dependent rho", float(rho[branch == 0].max()))
    runaway = runaway_scan(8192)
    print("oracle runaway candidates", runaway)
    streams = list(range(60)) + runaway[:8]
    with Pool(os.cpu_count() or 8) as p:
        res = p.map(_c5_trace, streams, chunksize=1)
    np.savez_compressed(os.path.join(OUT, "full_c5.npz"), streams=np.array([t[0] for t in res]),
                        branch=np.stack([t[1] for t in res]), rho=np.stack([t[2] for t in res]),
                        rank=np.array([t[3] for t in res]), x=np.stack([t[4] for t in res]),
                        digest=np.array([t[5] for t in res]))
    print("c5 ranks", [t[3] for t in res])
    with Pool(os.cpu_count() or 8) as p:
        res = p.map(_c3_trace, list(range(64)), chunksize=1)
    np.savez_compressed(os.path.join(OUT, "full_c3.npz"), streams=np.array([t[0] for t in res]),
                        branch=np.stack([t[1] for t in res]), rho=np.stack([t[2] for t in res]),
                        rank=np.array([t[3] for t in res]), x=np.stack([t[4] for t in res]),
                        digest=np.array([t[5] for t in res]))


if __name__ == "__main__":
    if sys.argv[1:] == ["bench"]:
        bench_cells()
    elif sys.argv[1:] == ["full"]:
        full_length()
    else:
        main()
        bench_cells()
