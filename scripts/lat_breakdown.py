"""Host-side breakdown of one RecursiveSolver.update() (perf_counter around each API call)."""
import ctypes
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2106_11594_b200 as p  # noqa: E402
from paper_2106_11594_b200 import _lib  # noqa: E402

m = 64
rng = np.random.default_rng(0)
A = rng.standard_normal((20, m))
s = p.RecursiveSolver(m)
s.ingest(A, rng.standard_normal(20))
rows = rng.standard_normal((400, 20)) @ A
for i in range(20):
    s.update(rows[i], 1.0)
bs = s._bs
buf = s._buffers(1)
lib = bs.lib
acc = np.zeros(8)
N = 300
for i in range(N):
    t = [time.perf_counter()]
    row = s._kind.vector(rows[i], m)
    buf["in_np"][:m] = row
    buf["in_np"][m] = 1.0
    t.append(time.perf_counter())
    stream = torch.cuda.current_stream(bs.device)
    h = ctypes.c_void_p(stream.cuda_stream)
    t.append(time.perf_counter())
    lib.rgb_memcpy_async(buf["in_d_p"], buf["in_h_p"], (m + 1) * 8, h)
    t.append(time.perf_counter())
    logs = _lib.Logs(buf["io_d_p"] + buf["off_branch"], None, buf["io_d_p"] + buf["off_resid"],
                     buf["io_d_p"] + buf["off_gain"])
    cfg, st = s._structs()
    t.append(time.perf_counter())
    lib.rgb_ingest(ctypes.byref(cfg), ctypes.byref(st), buf["in_d_p"], m, buf["in_d_p"] + m * 8, 1, 1,
                   ctypes.byref(logs), h)
    t.append(time.perf_counter())
    lib.rgb_memcpy_async(buf["io_h_p"], buf["io_d_p"], buf["off_resid"] + 8, h)
    t.append(time.perf_counter())
    stream.synchronize()
    t.append(time.perf_counter())
    acc[:7] += np.diff(t)
names = ["host prep", "stream handle", "H2D call", "logs+structs", "ingest call", "D2H call", "sync"]
print({k: round(v / N * 1e6, 2) for k, v in zip(names, acc)}, "total", round(acc.sum() / N * 1e6, 2))
# empty-stream round trip for reference
t0 = time.perf_counter()
for i in range(N):
    lib.rgb_memcpy_async(buf["io_h_p"], buf["io_d_p"], 16, h)
    stream.synchronize()
print("D2H 16 B + sync", round((time.perf_counter() - t0) / N * 1e6, 2))
t0 = time.perf_counter()
for i in range(N):
    stream.synchronize()
print("sync only", round((time.perf_counter() - t0) / N * 1e6, 2))
