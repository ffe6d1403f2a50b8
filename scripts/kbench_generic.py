"""Back-to-back one-row generic-kernel launches (update() shape): device time per launch."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2106_11594_b200.batched import BatchedSolver  # noqa: E402

for m, r in ((16, 8), (64, 20), (256, 20), (1024, 20), (256, 100)):
    rng = np.random.default_rng(0)
    basis = rng.standard_normal((r, m))
    rows = torch.as_tensor((rng.standard_normal((2000, r)) @ basis)[None], device="cuda")
    tg = torch.as_tensor(rng.standard_normal((1, 2000, 1)), device="cuda")
    cap = 1 << max(5, (r - 1).bit_length())
    bs = BatchedSolver(1, m, k=1, r_cap=cap)
    bs.ingest(torch.as_tensor(basis[None], device="cuda"), torch.as_tensor(rng.standard_normal((1, r, 1)), device="cuda"))
    res = torch.zeros((1, 1, 1), dtype=torch.float64, device="cuda")
    br = torch.zeros((1, 1), dtype=torch.uint8, device="cuda")
    for t in range(20):
        bs.ingest(rows[:, t:t + 1], tg[:, t:t + 1], resid_log=res, branch_log=br)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for t in range(20, 1020):
        bs.ingest(rows[:, t:t + 1], tg[:, t:t + 1], resid_log=res, branch_log=br)
    e1.record()
    torch.cuda.synchronize()
    one = e0.elapsed_time(e1)
    e0.record()
    bs.ingest(rows[:, 1020:2000], tg[:, 1020:2000], resid_log=torch.zeros((1, 980, 1), dtype=torch.float64, device="cuda"))
    e1.record()
    torch.cuda.synchronize()
    print(f"m={m} r={r}: one-row launches {one:.3f} us each (1000 back to back); "
          f"980 rows in one launch {e0.elapsed_time(e1) * 1e3 / 980:.3f} us/row, rank {int(bs.rank[0])}", flush=True)
