import ctypes, os, sys, numpy as np, torch
sys.path.insert(0, os.getcwd())
os.environ["RGB_LIB_PATH"] = os.path.join(os.getcwd(), "scratch/probe/librgb_probe.so")
from paper_2106_11594_b200.batched import BatchedSolver
from paper_2106_11594_b200 import _lib
S, n = int(sys.argv[1]), 64
g = torch.Generator(device="cuda").manual_seed(5)
A = torch.bmm(torch.randn(S, n, 16, generator=g, device="cuda", dtype=torch.float64), torch.randn(S, 16, 64, generator=g, device="cuda", dtype=torch.float64))
Y = torch.randn(S, n, 8, generator=g, device="cuda", dtype=torch.float64)
bs = BatchedSolver(S, 64, k=8, r_cap=16)
for _ in range(2):
    bs.reset(); bs.ingest(A, Y); torch.cuda.synchronize()
lib = _lib.load()
buf = (ctypes.c_longlong * 4096)()
lib.rgb_probe_read(buf, 4096)
a = np.array(buf[:16], dtype=np.int64)
print("S=%d load %d | tiles %s | after-loop->wb %d | writeback %d" % (S, a[1]-a[0], [int(a[i+1]-a[i]) for i in range(2, 9)], a[10]-a[9], a[11]-a[10]))
