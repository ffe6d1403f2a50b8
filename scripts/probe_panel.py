"""Per-phase cycles of the panel kernel on config 3: projection warp 0 and the
home warp of every CTA, summed, per stream.  Needs the probe build:
    python scripts/build_variant.py scratch/pp -DRGB_PANEL_PROBE
"""
import ctypes
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ.setdefault("RGB_LIB_PATH", os.path.join(ROOT, "scratch", "pp", "librgb.so"))
from paper_2106_11594_b200 import _lib, workloads  # noqa: E402
from paper_2106_11594_b200.batched import BatchedSolver  # noqa: E402

lib = _lib.load()
lib.rgb_panel_probe.argtypes = [ctypes.c_void_p, ctypes.c_int]
rows, tg = workloads.device_batch("c3", 0, 4096, "cuda")
bs = BatchedSolver(4096, 128, k=1, r_cap=32)
buf = np.zeros(32, np.uint64)
for i in range(3):
    bs.reset()
    lib.rgb_panel_probe(buf.ctypes.data, 1)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    bs.ingest(rows, tg)
    e1.record()
    torch.cuda.synchronize()
lib.rgb_panel_probe(buf.ctypes.data, 0)
print("ms", e0.elapsed_time(e1))
names = {0: "P setup", 1: "P row mode", 2: "P stage wait", 3: "P projection", 4: "P proj barrier",
         5: "P wait EMPTY", 6: "P growth", 7: "P end", 8: "H setup", 9: "H wait FULL", 10: "H scan",
         11: "H end", 12: "end sync wait", 13: "x+writeback+sync", 16: " bulk: warp-0 solve", 17: " bulk: barrier", 18: " bulk: C~ update", 19: " bulk: new rows", 20: " bulk: between tiles", 21: " scan: pre-LDL", 22: " scan: LDL", 23: " scan: post-LDL", 24: "defer: invert", 25: "defer: W", 31: "defer: redo count x4096"}
ws = np.zeros(8192, np.uint32)
lib.rgb_panel_wslot.argtypes = [ctypes.c_void_p]
lib.rgb_panel_wslot(ws.ctypes.data)
for cta in range(4):
    v = ws[cta * 8: cta * 8 + 5]
    print("cta", cta, "sm", (v >> 16).tolist(), "warpid", (v & 0xffff).tolist())
for i, nme in names.items():
    print(f"{nme:15s} {buf[i] / 4096:10.0f} cycles/stream")
