import ctypes, os, sys, numpy as np, torch
sys.path.insert(0, os.getcwd())
os.environ["RGB_LIB_PATH"] = os.path.join(os.getcwd(), "scratch/gprobe/librgb_gp.so")
from paper_2106_11594_b200 import workloads, _lib
from paper_2106_11594_b200.batched import BatchedSolver
for cfg in ("c2", "c4"):
    A, y = getattr(workloads, cfg)()
    rc = workloads.CONFIGS[cfg].r_cap
    bs = BatchedSolver(1, A.shape[1], k=1, r_cap=rc)
    rows = torch.as_tensor(A[None], device="cuda"); tg = torch.as_tensor(y[None, :, None], device="cuda")
    for _ in range(2):
        bs.reset(); bs.ingest(rows, tg); torch.cuda.synchronize()
    buf = (ctypes.c_ulonglong * 64)()
    _lib.load().rgb_gprobe_read(buf)
    a = np.array(buf[:11], dtype=np.int64)
    names = ["P1", "sync1", "P2+sync2", "Gs load", "P3+sync3", "P4 test", "scanU", "sync4", "P5", "sync5", "P6"]
    print(cfg, " ".join("%s=%.2fus" % (names[i], (a[i + 1] - a[i]) / 1e3) for i in range(10)), "total %.2fus" % ((a[10] - a[0]) / 1e3))
    b2 = (ctypes.c_ulonglong * 640)()
    _lib.load().rgb_gprobe2_read(b2)
    g = np.array(b2[:], dtype=np.int64).reshape(160, 4)[:128]
    t0 = g[:, 0].min()
    print(cfg, "P1 start spread %.2fus" % ((g[:, 0].max() - t0) / 1e3), "P1 dur min/med/max %.2f/%.2f/%.2f us" % tuple(np.percentile((g[:, 1] - g[:, 0]) / 1e3, [0, 50, 100])),
          "P1 end spread %.2fus" % ((g[:, 1].max() - g[:, 1].min()) / 1e3),
          "P3 dur (incl sync3 wait excluded) min/med/max %.2f/%.2f/%.2f" % tuple(np.percentile((g[:, 3] - g[:, 2]) / 1e3, [0, 50, 100])),
          "slowest P1-start CTAs", list(np.argsort(g[:, 0])[-5:]), "owners start med %.2f non-owners %.2f" % (np.median(g[:64, 0] - t0) / 1e3, np.median(g[64:, 0] - t0) / 1e3))
