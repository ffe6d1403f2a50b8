"""Tuning probe: blocked-kernel time for C5-shaped streams of n rows (n varies),
separating the rank-growth phase (first r rows) from the steady state."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2106_11594_b200.batched import BatchedSolver  # noqa: E402


def run(S, n, reps=3):
    g = torch.Generator(device="cuda").manual_seed(5)
    A = torch.bmm(torch.randn(S, n, 16, generator=g, device="cuda", dtype=torch.float64),
                  torch.randn(S, 16, 64, generator=g, device="cuda", dtype=torch.float64))
    Y = torch.randn(S, n, 8, generator=g, device="cuda", dtype=torch.float64)
    bs = BatchedSolver(S, 64, k=8, r_cap=16)
    ts = []
    for i in range(reps + 1):
        bs.reset()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        bs.ingest(A, Y)
        e1.record()
        torch.cuda.synchronize()
        if i:
            ts.append(e0.elapsed_time(e1))
    return min(ts)


if __name__ == "__main__":
    S = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
    out = {}
    for n in (16, 64, 256, 1024, 2048):
        out[n] = run(S, n)
    steady = (out[2048] - out[1024]) / 1024
    print(json.dumps({"lib": os.environ.get("RGB_LIB_PATH", "default"), "S": S, "ms": out,
                      "steady_ms_per_row": steady, "growth_ms_16rows": out[16],
                      "growth_rows_equiv": out[16] / steady,
                      "rows_per_s_steady": S / (steady * 1e-3)}))
