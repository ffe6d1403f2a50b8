"""One long generic-kernel launch (m 64, r 20, 980 dependent rows, resid log) for ncu."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2106_11594_b200.batched import BatchedSolver  # noqa: E402

m, r = 64, 20
rng = np.random.default_rng(0)
basis = rng.standard_normal((r, m))
rows = torch.as_tensor((rng.standard_normal((980, r)) @ basis)[None], device="cuda")
tg = torch.as_tensor(rng.standard_normal((1, 980, 1)), device="cuda")
bs = BatchedSolver(1, m, k=1, r_cap=32)
res0 = torch.zeros((1, r, 1), dtype=torch.float64, device="cuda")
bs.ingest(torch.as_tensor(basis[None], device="cuda"), torch.as_tensor(rng.standard_normal((1, r, 1)), device="cuda"),
          resid_log=res0)
res = torch.zeros((1, 980, 1), dtype=torch.float64, device="cuda")
bs.ingest(rows, tg, resid_log=res)
torch.cuda.synchronize()
print("rank", int(bs.rank[0]))
