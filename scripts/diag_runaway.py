"""Diagnose device/oracle branch disagreements on device-generated C5 streams."""
import json, os, sys
import numpy as np, torch
sys.path.insert(0, os.getcwd())
from oracle import oracle
from paper_2106_11594_b200 import workloads
from paper_2106_11594_b200.batched import BatchedSolver

B0, B1 = int(sys.argv[1]), int(sys.argv[2])
rows, tg = workloads.device_batch("c5", B0, B1, "cuda")
S, n, m = rows.shape
bs = BatchedSolver(S, 64, k=8, r_cap=16)
br = torch.zeros((S, n), dtype=torch.uint8, device="cuda")
bs.ingest(rows, tg, branch_log=br)
torch.cuda.synchronize()
st = bs.status.cpu().numpy(); rk = bs.rank.cpu().numpy(); brn = br.cpu().numpy()
R, Y = rows.cpu().numpy(), tg.cpu().numpy()
o = oracle.ingest(R, Y, r_cap=16, nthreads=16)
mism = np.nonzero((o["rank"] != rk) | (o["status"] != st) | np.any(o["branch"] != brn, axis=1))[0]
out = {"streams": int(S), "gpu_rank_cap": int((st & 1).sum()), "oracle_rank_cap": int((o["status"] & 1).sum()),
       "mismatched_streams": int(len(mism)), "details": []}
for b in mism[:40]:
    d = np.nonzero(o["branch"][b] != brn[b])[0]
    t = int(d[0]) if len(d) else -1
    # margin of the oracle's rank test at the first disagreement (rho<1: dependent)
    out["details"].append({"stream": int(B0 + b), "first_row": t, "oracle_rho": float(o["rho"][b][t]) if t >= 0 else None,
                           "gpu_branch": int(brn[b][t]) if t >= 0 else None, "gpu_status": int(st[b]),
                           "oracle_status": int(o["status"][b]), "max_dep_rho_before": float(o["rho"][b][:max(t,1)][o["branch"][b][:max(t,1)] == 0].max()) if t > 0 and (o["branch"][b][:t] == 0).any() else None})
print(json.dumps(out))
