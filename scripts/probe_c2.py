"""Phase timing of the cluster kernel on config 2 (probe build in scratch/probe)."""
import ctypes
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ.setdefault("RGB_LIB_PATH", os.path.join(ROOT, "scratch", "probe", "librgb.so"))
from paper_2106_11594_b200 import _lib, workloads  # noqa: E402
from paper_2106_11594_b200.batched import BatchedSolver  # noqa: E402

lib = _lib.load()
lib.rgb_cluster_probe.argtypes = [ctypes.c_void_p, ctypes.c_int]
A, y = workloads.c2()
rows = torch.as_tensor(A[None], device="cuda")
tg = torch.as_tensor(y[None, :, None], device="cuda")
bs = BatchedSolver(1, 1024, k=1, r_cap=64)
buf = np.zeros((2, 16), np.uint64)
for i in range(3):
    bs.reset()
    lib.rgb_cluster_probe(buf.ctypes.data, 1)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    bs.ingest(rows, tg)
    e1.record()
    torch.cuda.synchronize()
lib.rgb_cluster_probe(buf.ctypes.data, 0)
names = ["P1", "barA", "P2", "barB", "P3+norms", "barC", "P4", "-", "grow", "panel-load", "dep:U", "dep:S+LDL", "dep:Y+W", "dep:P", "wait-slot"]
print("kernel ms", e0.elapsed_time(e1))
for c in range(2):
    print(["column 0", "home"][c], {n: round(buf[c][i] / 1e6, 3) for i, n in enumerate(names)})
