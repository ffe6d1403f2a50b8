"""Parity sweep at scale: device-generated config-5 / config-3 streams through
the tensor-core kernels against the C oracle on the same bytes; writes counts
of exact matches, ambiguous streams (oracle margin rho in [1/8, 8] or oracle
runaway) and the worst x error to a JSON summary."""
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle import oracle  # noqa: E402  (checker)
from paper_2106_11594_b200 import workloads  # noqa: E402
from paper_2106_11594_b200.batched import BatchedSolver  # noqa: E402


def sweep(cfg_name, B, kernel="default"):
    """kernel: "default" (the dispatcher's choice) or "warp-group" (RGB_NO_PANEL=1)."""
    os.environ["RGB_NO_PANEL"] = "1" if kernel == "warp-group" else "0"
    c = workloads.CONFIGS[cfg_name]
    rows_d, tg_d = workloads.device_batch(cfg_name, 0, B, "cuda")
    n = rows_d.shape[1]
    bs = BatchedSolver(B, c.m, k=c.k, r_cap=c.r_cap)
    br = torch.zeros((B, n), dtype=torch.uint8, device="cuda")
    bs.ingest(rows_d, tg_d, branch_log=br)
    torch.cuda.synchronize()
    rows, tg = rows_d.cpu().numpy(), tg_d.cpu().numpy()
    o = oracle.ingest(rows, tg, r_cap=c.r_cap, nthreads=os.cpu_count() or 8)
    amb = ((o["rho"] >= 0.125) & (o["rho"] <= 8)).any(axis=1) | (o["status"] != 0)
    dev_status = bs.status.cpu().numpy()
    ok = ~amb & (dev_status == 0)
    branch = br.cpu().numpy()
    rank = bs.rank.cpu().numpy()
    X, XO = bs.solution.cpu().numpy(), oracle.solution(o)
    err = np.abs(X - XO).max(axis=(1, 2)) / np.maximum(1.0, np.abs(XO).max(axis=(1, 2)))
    return {"config": cfg_name, "kernel": {"c5": "one-warp", "c3": "panel"}[cfg_name] if kernel == "default" else kernel,
            "streams": B, "rows_per_stream": n,
            "ambiguous_or_runaway": int(amb.sum()), "device_frozen": int((dev_status != 0).sum()),
            "checked": int(ok.sum()),
            "branch_mismatch": int((branch[ok] != o["branch"][ok]).any(axis=1).sum()),
            "rank_mismatch": int((rank[ok] != o["rank"][ok]).sum()),
            "x_relerr_max": float(err[ok].max()), "x_relerr_median": float(np.median(err[ok])),
            "tolerance": 1e-9}


out = [sweep("c5", 16384), sweep("c3", 4096), sweep("c3", 4096, "warp-group")]
print(json.dumps(out, indent=1))
path = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "gpurun_out", "parity_sweep.json")
json.dump(out, open(path, "w"), indent=1)
