"""Quick parity probe of the m = 128 kernels against the C oracle (config-3 streams)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import oracle  # noqa: E402
from paper_2106_11594_b200 import workloads  # noqa: E402
from paper_2106_11594_b200.batched import BatchedSolver  # noqa: E402

for nstreams, n in ((4, 64), (16, 512)):
    rows, tg = workloads.host_batch("c3", list(range(nstreams)), n=n)
    B, T, m = rows.shape
    bs = BatchedSolver(B, m, k=1, r_cap=32, device="cuda:0")
    br = torch.zeros((B, T), dtype=torch.uint8, device="cuda:0")
    bs.ingest(torch.as_tensor(rows, device="cuda:0"), torch.as_tensor(tg, device="cuda:0"), branch_log=br)
    torch.cuda.synchronize()
    o = oracle.ingest(rows, tg, r_cap=32, nthreads=8)
    x = bs.solution.cpu().numpy()
    xo = oracle.solution(o)
    err = np.abs(x - xo).max(axis=(1, 2)) / np.maximum(1.0, np.abs(xo).max(axis=(1, 2)))
    print("B", B, "T", T, "rank dev", bs.rank.cpu().numpy().tolist(), "oracle", o["rank"].tolist())
    print("  branch equal per stream", (br.cpu().numpy() == o["branch"]).all(axis=1).tolist())
    print("  x err", err.tolist())
