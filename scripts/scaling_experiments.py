"""Regenerate the reference's scaling experiments (its acceptance criteria
5-7, test_acceptance.py:127-156) on the GPU through the device-backed
harness; writes one CSV per experiment and prints the fitted exponents."""
import json
import os
import sys
import time
import warnings

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2106_11594_b200 import experiments as ex  # noqa: E402

out_dir = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "gpurun_out")
plans = {
    "rank-fixed-r": ex.make_plan("rank-fixed-r", [256, 512, 1024, 2048], fixed_r=20, repetitions=5, seed=11),
    "square": ex.make_plan("square", [64, 128, 256, 512], repetitions=9, seed=13),
    "update-cost": ex.make_plan("update-cost", [50, 100, 200, 400], fixed_m=2000, repetitions=5, seed=17),
}
res = {}
for (name, plan), clock in [(kv, c) for c in ("wall", "device") for kv in plans.items()]:
    t0 = time.perf_counter()
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        samples, fit = ex.run_plan(plan, clock=clock)
    name = f"{name}_{clock}"
    ex.write_csv(samples, os.path.join(out_dir, f"scaling_{name}.csv"))
    med = {}
    for s in samples:
        med.setdefault(plan.swept_size((s.n, s.m, s.r)), []).append(s.seconds)
    res[name] = {"exponent": fit.exponent, "r_squared": fit.r_squared, "elapsed_s": time.perf_counter() - t0,
                 "median_s": {k: sorted(v)[len(v) // 2] for k, v in med.items()}}
print(json.dumps(res, indent=1))
