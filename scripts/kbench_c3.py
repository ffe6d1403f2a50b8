"""Tuning probe: warp-group kernel time on the config-3 batch (device-generated)."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2106_11594_b200 import workloads  # noqa: E402
from paper_2106_11594_b200.batched import BatchedSolver  # noqa: E402

rows, tg = workloads.device_batch("c3", 0, 4096, "cuda")
bs = BatchedSolver(4096, 128, k=1, r_cap=32)
ts = []
for i in range(6):
    bs.reset()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    bs.ingest(rows, tg)
    e1.record()
    torch.cuda.synchronize()
    if i:
        ts.append(e0.elapsed_time(e1))
print(json.dumps({"c3_ms_min": min(ts), "c3_ms": ts}))
