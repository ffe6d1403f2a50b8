"""Debug: config-3 streams where a kernel's rank/branches differ from the oracle."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import oracle  # noqa: E402
from paper_2106_11594_b200 import workloads  # noqa: E402
from paper_2106_11594_b200.batched import BatchedSolver  # noqa: E402

rows_d, tg_d = workloads.device_batch("c3", 0, 1024, "cuda")
S, n, _ = rows_d.shape
bs = BatchedSolver(S, 128, k=1, r_cap=32)
br = torch.zeros((S, n), dtype=torch.uint8, device="cuda")
bs.ingest(rows_d, tg_d, branch_log=br)
torch.cuda.synchronize()
rows, tg = rows_d.cpu().numpy(), tg_d.cpu().numpy()
o = oracle.ingest(rows, tg, r_cap=32, nthreads=16)
rk = bs.rank.cpu().numpy()
bl = br.cpu().numpy()
st = bs.status.cpu().numpy() if hasattr(bs, "status") else None
bad = np.nonzero((rk != o["rank"]) | (bl != o["branch"]).any(axis=1))[0]
print("mismatching streams:", bad.tolist()[:20], "of", S)
for b in bad[:6]:
    d = np.nonzero(bl[b] != o["branch"][b])[0]
    print(f"stream {b}: rank dev {rk[b]} oracle {o['rank'][b]} status {None if st is None else st[b]} "
          f"first diff rows {d[:8].tolist()} dev {bl[b][d[:8]].tolist()} oracle {o['branch'][b][d[:8]].tolist()} "
          f"rho {o['rho'][b][d[:4]].tolist()} oracle indep rows {np.nonzero(o['branch'][b])[0][:40].tolist()}")
