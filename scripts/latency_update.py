"""Per-call latency of the drop-in API (RecursiveSolver.update / ingest of one row)."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2106_11594_b200 as p  # noqa: E402

for m in [int(v) for v in os.environ.get("RGB_LAT_M", "16,64,256,1024").split(",")]:
    rng = np.random.default_rng(0)
    A = rng.standard_normal((40, m))
    r = min(20, m)
    s = p.RecursiveSolver(m)
    s.ingest(A[:r], rng.standard_normal(r))
    rows = rng.standard_normal((400, r)) @ A[:r]
    ys = rng.standard_normal(400)
    for i in range(20):
        s.update(rows[i], ys[i])
    t0 = time.perf_counter()
    for i in range(20, 400):
        s.update(rows[i], ys[i])
    t_upd = (time.perf_counter() - t0) / 380
    t0 = time.perf_counter()
    for i in range(20, 400):
        s.ingest(rows[i:i + 1], ys[i:i + 1])
    t_ing = (time.perf_counter() - t0) / 380
    t0 = time.perf_counter()
    for i in range(20, 400):
        s.project(rows[i])
    t_prj = (time.perf_counter() - t0) / 380
    print(f"m={m}: update {t_upd * 1e6:.1f} us/call, ingest(1 row) {t_ing * 1e6:.1f} us/call, "
          f"project {t_prj * 1e6:.1f} us/call", flush=True)
