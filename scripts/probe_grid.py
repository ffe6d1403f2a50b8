"""Phase timing of the grid kernel on config 4 or 2 (probe build in scratch/gprobe)."""
import ctypes
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ.setdefault("RGB_LIB_PATH", os.path.join(ROOT, "scratch", "gprobe", "librgb.so"))
from paper_2106_11594_b200 import _lib, workloads  # noqa: E402
from paper_2106_11594_b200.batched import BatchedSolver  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c4"
lib = _lib.load()
lib.rgb_grid_probe.argtypes = [ctypes.c_void_p, ctypes.c_int]
A, y = getattr(workloads, cfg)()
c = workloads.CONFIGS[cfg]
rows = torch.as_tensor(A[None], device="cuda")
tg = torch.as_tensor(y[None, :, None], device="cuda")
bs = BatchedSolver(1, c.m, k=1, r_cap=c.r_cap)
buf = np.zeros((2, 16), np.uint64)
for i in range(2):
    bs.reset()
    lib.rgb_grid_probe(buf.ctypes.data, 1)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    bs.ingest(rows, tg)
    e1.record()
    torch.cuda.synchronize()
lib.rgb_grid_probe(buf.ctypes.data, 0)
names = ["P6+grow+P1", "bar1", "P2 reduce", "bar2", "P3", "bar3", "P4+U/S", "bar4", "P5 LDL/Y", "bar5", "grow-ng", "bar-ng",
         "t(first R rows)"]
print(cfg, "kernel ms", e0.elapsed_time(e1))
for k in range(2):
    print("CTA", k, {n: round(buf[k][i] / 1e6, 3) for i, n in enumerate(names)})
