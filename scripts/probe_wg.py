"""Per-phase cycles of the warp-group kernel: warp 0 of every CTA, summed,
printed per tile.  Needs the probe build:

    nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -shared -Xcompiler -fPIC \
        -DRGB_WG_PROBE -Iinclude -o scratch/wgp/librgb.so paper_2106_11594_b200/csrc/*.cu
"""
import ctypes
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ.setdefault("RGB_LIB_PATH", os.path.join(ROOT, "scratch", "wgp", "librgb.so"))
from paper_2106_11594_b200 import _lib, workloads  # noqa: E402
from paper_2106_11594_b200.batched import BatchedSolver  # noqa: E402

lib = _lib.load()
lib.rgb_wg_probe.argtypes = [ctypes.c_void_p, ctypes.c_int]
rows, tg = workloads.device_batch("c3", 0, 4096, "cuda")
bs = BatchedSolver(4096, 128, k=1, r_cap=32)
buf = np.zeros(16, np.uint64)
for i in range(3):
    bs.reset()
    lib.rgb_wg_probe(buf.ctypes.data, 1)
    bs.ingest(rows, tg)
    torch.cuda.synchronize()
lib.rgb_wg_probe(buf.ctypes.data, 0)
tiles = 4096 * 64
names = ["pre-front", "front1", "sync1", "front2", "sync2", "front3", "pre-scan", "scan1", "syncS1", "scan2",
         "syncS2", "-", "scan3+tail", "sync-tile"]
tot = buf.sum()
for i, nme in enumerate(names):
    print(f"{nme:11s} {buf[i] / tiles:8.0f} cycles/tile  {100 * buf[i] / tot:5.1f}%")
