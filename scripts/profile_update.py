"""cProfile of the drop-in update() path (host-side overhead per call)."""
import cProfile
import os
import pstats
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2106_11594_b200 as p  # noqa: E402

rng = np.random.default_rng(0)
m = 64
A = rng.standard_normal((20, m))
s = p.RecursiveSolver(m)
s.ingest(A, rng.standard_normal(20))
rows = rng.standard_normal((600, 20)) @ A
ys = rng.standard_normal(600)
for i in range(50):
    s.update(rows[i], ys[i])
pr = cProfile.Profile()
pr.enable()
for i in range(50, 550):
    s.update(rows[i], ys[i])
pr.disable()
st = pstats.Stats(pr)
st.sort_stats("tottime").print_stats(18)
