"""Where the wall time of a drop-in solve_batch goes (one rank-fixed-r cell)."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2106_11594_b200 as p  # noqa: E402
from paper_2106_11594_b200 import experiments as ex  # noqa: E402
from paper_2106_11594_b200.solver import RecursiveSolver  # noqa: E402

plan = ex.make_plan("rank-fixed-r", [1024, 2048], fixed_r=20, repetitions=3, seed=11)
for idx, cell in enumerate(plan.grid):
    A, y = ex.solve_inputs(plan, idx, cell)
    n, m, _ = cell
    for _ in range(3):
        p.solve_batch(A, y)
    torch.cuda.synchronize()

    def t(f, reps=5):
        ts = []
        for _ in range(reps):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            f()
            torch.cuda.synchronize()
            ts.append(time.perf_counter() - t0)
        return 1e3 * sorted(ts)[len(ts) // 2]

    out = {"solve_batch": t(lambda: p.solve_batch(A, y)),
           "new_solver": t(lambda: RecursiveSolver(m)),
           "pinned_copy": None, "h2d": None}
    s = RecursiveSolver(m)
    buf = s._buffers(n)
    out["pinned_copy"] = t(lambda: buf["rows_h_np"].__setitem__(slice(0, n), A))
    out["h2d"] = t(lambda: buf["t"]["rows_d"][:n].copy_(buf["t"]["rows_h"][:n], non_blocking=True))

    def ing():
        s2 = RecursiveSolver(m)
        s2.ingest(A, y)
    out["new+ingest"] = t(ing)
    s3 = RecursiveSolver(m, r_cap=32)
    s3._buffers(n)

    def ing_warm():
        s3._bs.reset()
        s3._host["nobs"] = 0
        s3.ingest(A, y)
    out["warm_ingest"] = t(ing_warm)
    print(cell, {k: round(v, 3) for k, v in out.items()}, flush=True)

from torch.profiler import ProfilerActivity, profile  # noqa: E402

with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
    for _ in range(3):
        ing_warm()
    torch.cuda.synchronize()
print(prof.key_averages().table(sort_by="cuda_time_total", row_limit=12))
print(prof.key_averages().table(sort_by="cpu_time_total", row_limit=12))
