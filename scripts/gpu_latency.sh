python scripts/latency_update.py > gpurun_out/lat.log 2>&1
python - >> gpurun_out/lat.log 2>&1 <<'PY'
import sys, numpy as np, torch
sys.path.insert(0, '.')
import paper_2106_11594_b200 as p
from torch.profiler import profile, ProfilerActivity
rng = np.random.default_rng(0)
A = rng.standard_normal((20, 64)); s = p.RecursiveSolver(64); s.ingest(A, rng.standard_normal(20))
rows = rng.standard_normal((50, 20)) @ A
for i in range(10): s.update(rows[i], 1.0)
with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
    for i in range(10, 50): s.update(rows[i], 1.0)
print(prof.key_averages().table(sort_by="cpu_time_total", row_limit=25))
PY
