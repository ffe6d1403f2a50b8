"""CPU check of the algebra behind the kernels' deferred fold: on the C
oracle's coords log B of config-3 / config-5 streams, P = (B^T B)^-1 and x = C~^T P B^T y
reproduce the oracle's sequential Sherman-Morrison result (solver.py:297-304) to well inside
the 1e-9 bar whenever kappa_F(B^T B) <= 1e6 -- the certificate the kernels apply -- and the
two forms drift apart beyond it, which is why the kernels keep the chain as the fallback."""
import numpy as np
import pytest

from oracle import oracle
from paper_2106_11594_b200 import workloads


def relerr(a, b):
    return float(np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-300))


@pytest.mark.parametrize("cfg,r_cap", [("c5", 16), ("c3", 32)])
def test_normal_equations_in_the_coords_match_the_recursion_under_the_certificate(cfg, r_cap):
    streams = list(range(96))
    rows, tg = workloads.host_batch(cfg, streams)
    o = oracle.ingest(rows, tg, r_cap=r_cap, nthreads=8)
    X = oracle.solution(o)
    checked = 0
    for i in range(len(streams)):
        if o["status"][i]:
            continue
        r = int(o["rank"][i])
        B = o["coords"][i][:, :r]
        y = tg[i].reshape(B.shape[0], -1)
        Q = B.T @ B
        P = np.linalg.inv(Q)
        # growth rows are unit rows of B and the basis never shrinks: Q >= I
        assert np.linalg.eigvalsh(Q).min() >= 1.0 - 1e-9
        kappa = np.linalg.norm(Q) * np.linalg.norm(P)
        if kappa > 1e6:
            continue
        x = o["D"][i][:r].T @ (P @ (B.T @ y))
        assert relerr(x, X[i]) <= 1e-10, (i, kappa)
        assert relerr(P, o["P"][i][:r, :r]) <= 1e-9, (i, kappa)
        checked += 1
    assert checked >= 80
