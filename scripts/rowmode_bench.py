"""Row-mode cost of the panel kernel: streams whose first 32 rows are all
independent (Gaussian m = 128), timed per row for one and two CTAs per SM."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2106_11594_b200.batched import BatchedSolver  # noqa: E402

g = torch.Generator(device="cuda").manual_seed(0)
out = {}
for B, T in ((148, 32), (296, 32), (296, 24), (4096, 32)):
    rows = torch.randn((B, T, 128), device="cuda", dtype=torch.float64, generator=g)
    tg = torch.randn((B, T, 1), device="cuda", dtype=torch.float64, generator=g)
    bs = BatchedSolver(B, 128, k=1, r_cap=32)
    ts = []
    for i in range(4):
        bs.reset()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        bs.ingest(rows, tg)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ms = min(ts[1:])
    waves = max(1.0, B / 296)
    out[f"B{B}_T{T}"] = {"ms": ms, "us_per_row_per_wave": 1e3 * ms / T / waves, "rank": int(bs.rank.max())}
print(json.dumps(out))
