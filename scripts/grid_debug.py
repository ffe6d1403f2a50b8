import os, sys, numpy as np, torch
sys.path.insert(0, os.getcwd())
from oracle import oracle
from paper_2106_11594_b200 import workloads
from paper_2106_11594_b200.batched import BatchedSolver
A, y = workloads.c4()
for n in (64, 256, 512, 520, 600):
    bs = BatchedSolver(1, 2048, k=1, r_cap=512)
    bs.ingest(torch.as_tensor(A[None, :n], device="cuda"), torch.as_tensor(y[None, :n, None], device="cuda"))
    torch.cuda.synchronize()
    r = int(bs.rank.item())
    C = bs.basis_t[0, :r].cpu().numpy(); D = bs.dual_t[0, :r].cpu().numpy(); P = bs.gram_t[0, :r, :r].cpu().numpy()
    o = oracle.ingest(A[None, :n], y[None, :n], r_cap=512)
    ro = int(o["rank"][0])
    Co = o["C"][0, :ro]; Do = o["D"][0, :ro]; Po = o["P"][0, :ro, :ro]
    print(n, "rank", r, ro, "status", int(bs.status.item()), int(o["status"][0]),
          "dual inv %.2e" % np.abs(D @ C.T - np.eye(r)).max(), "oracle dual inv %.2e" % np.abs(Do @ Co.T - np.eye(ro)).max(),
          "C diff %.2e" % (np.abs(C - Co[:r]).max() if r == ro else -1), "D diff %.2e" % (np.abs(D - Do).max() / np.abs(Do).max() if r == ro else -1),
          "P diff %.2e" % (np.abs(P - Po).max() / np.abs(Po).max() if r == ro else -1),
          "x diff %.2e" % np.abs(bs.solution.cpu().numpy()[0, :, 0] - oracle.solution(o)[0, :, 0]).max())
