"""Parity sweep at scale: device-generated config-5 / config-3 streams through
the tensor-core kernels against the C oracle on the same bytes.  Per stream the
first branch disagreement (if any) is located and classified by the oracle's
rank-test margin rho at that row: inside the noise band (tests/rgb_testutil.py
BAND, [1/16, 16]) or outside it (a parity failure).  Writes the counts, every
disagreement as (stream, row, rho), the distribution of the largest dependent
margin per stream, and the worst x error over exactly matching streams."""
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
from oracle import oracle  # noqa: E402  (checker)
from rgb_testutil import BAND, compare_branches  # noqa: E402
from paper_2106_11594_b200 import workloads  # noqa: E402
from paper_2106_11594_b200.batched import BatchedSolver  # noqa: E402


def sweep(cfg_name, B, kernel="default"):
    """kernel: "default" (the dispatcher's choice: deferred fold with the sequential
    chain as its fallback), "sequential" (RGB_BLOCKED_SEQ / RGB_PANEL_SEQ: the chain
    for every stream) or "warp-group" (RGB_NO_PANEL=1)."""
    os.environ["RGB_NO_PANEL"] = "1" if kernel == "warp-group" else "0"
    os.environ["RGB_BLOCKED_SEQ"] = os.environ["RGB_PANEL_SEQ"] = "1" if kernel == "sequential" else "0"
    c = workloads.CONFIGS[cfg_name]
    rows_d, tg_d = workloads.device_batch(cfg_name, 0, B, "cuda")
    n = rows_d.shape[1]
    bs = BatchedSolver(B, c.m, k=c.k, r_cap=c.r_cap)
    br = torch.zeros((B, n), dtype=torch.uint8, device="cuda")
    bs.ingest(rows_d, tg_d, branch_log=br)
    torch.cuda.synchronize()
    rows, tg = rows_d.cpu().numpy(), tg_d.cpu().numpy()
    o = oracle.ingest(rows, tg, r_cap=c.r_cap, nthreads=os.cpu_count() or 8)
    dev_status = bs.status.cpu().numpy()
    branch = br.cpu().numpy()
    nobs = bs.nobs_t.cpu().numpy()
    cmp = compare_branches(branch, nobs, o["branch"], o["rho"])
    ok = np.array([dev_status[b] == 0 and o["status"][b] == 0 and np.array_equal(branch[b], o["branch"][b])
                   for b in range(B)])
    rank = bs.rank.cpu().numpy()
    X, XO = bs.solution.cpu().numpy(), oracle.solution(o)
    err = np.abs(X - XO).max(axis=(1, 2)) / np.maximum(1.0, np.abs(XO).max(axis=(1, 2)))
    dep_rho = np.where(o["branch"] == 0, o["rho"], 0.0).max(axis=1)
    name = {"c5": "one-warp", "c3": "panel"}[cfg_name]
    return {"config": cfg_name,
            "kernel": {"default": name + " (deferred fold)", "sequential": name + " (sequential chain)"}.get(kernel, kernel),
            "streams": B, "rows_per_stream": n, "band": list(BAND),
            "exact_branch_logs": cmp["exact"], "first_disagreement_in_band": cmp["band_disagree"],
            "first_disagreement_outside_band": cmp["outside_disagree"],
            "disagreements": [(int(b), int(i), float(r)) for b, i, r, _ in cmp["disagreements"]],
            "streams_with_band_rows": cmp["streams_with_band_rows"],
            "oracle_runaway": int((o["status"] != 0).sum()), "device_frozen": int((dev_status != 0).sum()),
            "x_checked": int(ok.sum()), "rank_mismatch_on_exact": int((rank[ok] != o["rank"][ok]).sum()),
            "x_relerr_max": float(err[ok].max()), "x_relerr_median": float(np.median(err[ok])),
            "x_relerr_q999": float(np.quantile(err[ok], 0.999)),
            "max_dependent_rho_quantiles": {q: float(np.quantile(dep_rho, float(q))) for q in
                                            ("0.5", "0.99", "0.999", "1.0")},
            "tolerance": 1e-9}


out = [sweep("c5", 16384), sweep("c5", 16384, "sequential"), sweep("c3", 4096), sweep("c3", 4096, "sequential"),
       sweep("c3", 4096, "warp-group")]
print(json.dumps(out, indent=1))
path = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "gpurun_out", "parity_sweep.json")
json.dump(out, open(path, "w"), indent=1)
