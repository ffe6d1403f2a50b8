"""Numerical study behind the deferred fold: numpy restatement on the C
oracle's coords log (CPU only; the oracle is the checker here, not a product path).

For config-3 / config-5 streams: x from the deferred form  W = (B^T B)^-1 B^T y,  x = C~^T W
against the oracle's sequential x and against an SVD solve of the stream ("truth"); the same
by the kappa_F(B^T B) bound; and how well kappa_F a few rows into the stream predicts the final
one (the early check of the one-warp kernel).

    python scripts/deferred_fold_sim.py [streams]
"""
import os
import sys

import numpy as np
import scipy.linalg as sl

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import oracle  # noqa: E402  (checker)
from paper_2106_11594_b200 import workloads  # noqa: E402


def relerr(a, b):
    return float(np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-300))


def kappa_f(Q):
    return float(np.linalg.norm(Q) * np.linalg.norm(np.linalg.inv(Q)))


def main():
    B = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
    for name, rc in (("c3", 32), ("c5", 16)):
        streams = list(range(B))
        rows, tg = workloads.host_batch(name, streams)
        o = oracle.ingest(rows, tg, r_cap=rc, nthreads=os.cpu_count() or 8)
        X = oracle.solution(o)
        rec = []
        for i in range(B):
            if o["status"][i]:
                continue
            r = int(o["rank"][i])
            Bf = o["coords"][i][:, :r]
            y = tg[i].reshape(Bf.shape[0], -1)
            Q = Bf.T @ Bf
            c = sl.cho_factor(Q)
            x = o["D"][i][:r].T @ sl.cho_solve(c, Bf.T @ y)
            U, s, Vt = np.linalg.svd(rows[i], full_matrices=False)
            xt = Vt[:r].T @ ((U[:, :r].T @ y) / s[:r, None])
            tc = rc + 32
            rec.append((relerr(x, X[i]), relerr(X[i], xt), relerr(x, xt), kappa_f(Q),
                        kappa_f(Bf[:tc].T @ Bf[:tc])))
        rec = np.array(rec)
        print(f"{name}: {len(rec)} streams")
        print("  deferred vs oracle max %.2e | oracle vs svd max %.2e | deferred vs svd max %.2e"
              % (rec[:, 0].max(), rec[:, 1].max(), rec[:, 2].max()))
        for thr in (1e4, 1e5, 1e6, 1e7):
            sel = rec[:, 3] <= thr
            print("  kappa_F <= %.0e: %5.1f %% of the streams, deferred vs oracle max %.2e"
                  % (thr, 100 * sel.mean(), rec[sel, 0].max()))
        fail = rec[:, 3] > 1e6
        for thr in (3e5, 5e5, 1e6):
            pred = rec[:, 4] > thr
            print("  early check at row %d, kappa_F > %.0e: catches %.3f of the streams past 1e6, "
                  "false positives %.4f of all" % (rc + 32, thr, (pred & fail).sum() / max(fail.sum(), 1),
                                                   (pred & ~fail).mean()))


if __name__ == "__main__":
    main()
