import ctypes, os, sys, numpy as np, torch
sys.path.insert(0, os.getcwd())
os.environ["RGB_LIB_PATH"] = os.path.join(os.getcwd(), "scratch/probe/librgb_probe.so")
from paper_2106_11594_b200.batched import BatchedSolver
from paper_2106_11594_b200 import _lib
S, n = int(sys.argv[1]), 256
g = torch.Generator(device="cuda").manual_seed(5)
A = torch.bmm(torch.randn(S, n, 16, generator=g, device="cuda", dtype=torch.float64), torch.randn(S, 16, 64, generator=g, device="cuda", dtype=torch.float64))
Y = torch.randn(S, n, 8, generator=g, device="cuda", dtype=torch.float64)
bs = BatchedSolver(S, 64, k=8, r_cap=16)
for _ in range(2):
    bs.reset(); bs.ingest(A, Y); torch.cuda.synchronize()
lib = _lib.load()
buf = (ctypes.c_longlong * 4096)()
lib.rgb_probe_read(buf, 4096)
a = np.array(buf[:], dtype=np.int64)
for t in range(4):
    p = a[t*16:t*16+4]
    print("S=%d tile %d: wait %d  scan %d  front %d  -> next" % (S, t + 4, p[1]-p[0], p[2]-p[1], p[3]-p[2]),
          " total to next tile", (a[(t+1)*16] - p[0]) if t < 3 else -1)
for t in range(5, 9):
    s0, s1, s2 = a[1000+t], a[2000+t], a[3000+t]
    print(" scan tile %d: pre-S %s, elimination %d, rd+yt+dh %d" % (t, "-", s1 - s0, s2 - s1))
