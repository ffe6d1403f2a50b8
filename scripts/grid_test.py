import os, sys, time, numpy as np, torch
sys.path.insert(0, os.getcwd())
from oracle import oracle
from paper_2106_11594_b200 import workloads
from paper_2106_11594_b200.batched import BatchedSolver
cfg = sys.argv[1]; n = int(sys.argv[2])
A, y = getattr(workloads, cfg)()
A, y = A[:n], y[:n]
m = A.shape[1]; rc = workloads.CONFIGS[cfg].r_cap
bs = BatchedSolver(1, m, k=1, r_cap=rc)
rows = torch.as_tensor(A[None], device="cuda"); tg = torch.as_tensor(y[None, :, None], device="cuda")
br = torch.zeros((1, n), dtype=torch.uint8, device="cuda")
torch.cuda.synchronize(); t = time.time()
bs.ingest(rows, tg, branch_log=br); torch.cuda.synchronize(); dt = time.time() - t
bs.reset(); torch.cuda.synchronize(); t = time.time()
bs.ingest(rows, tg); torch.cuda.synchronize(); dt2 = time.time() - t
bs.reset(); bs.ingest(rows, tg, branch_log=br); torch.cuda.synchronize()
t = time.time(); o = oracle.ingest(A[None], y[None], r_cap=rc); to = time.time() - t
x = bs.solution.cpu().numpy()[0, :, 0]; xo = oracle.solution(o)[0, :, 0]
print(cfg, n, "gpu s", round(dt, 4), round(dt2, 4), "us/row %.2f" % (dt2 / n * 1e6), "oracle s", round(to, 2),
      "rank", int(bs.rank.item()), int(o["rank"][0]), "status", int(bs.status.item()),
      "branch eq", bool(np.array_equal(br.cpu().numpy()[0], o["branch"][0])),
      "x relerr %.2e" % (np.abs(x - xo).max() / max(1, np.abs(xo).max())), "max rho dep", float(o["rho"][0][o["branch"][0] == 0].max()))
