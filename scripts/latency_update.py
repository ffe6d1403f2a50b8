"""Per-call latency of the drop-in per-row API (RecursiveSolver.update, and
ingest / project of one row) against the reference's own update
and project (baseline/_ref, the unmodified rankrls, one core), with the distribution
(median / p90 / p99) and a breakdown of one update() call: the graph replay +
synchronisation alone, and the device time of the captured work.

    python scripts/latency_update.py [out.json]
"""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2106_11594_b200 as p  # noqa: E402


def dist(ts):
    ts = np.asarray(ts) * 1e6
    return {"median_us": float(np.median(ts)), "p90_us": float(np.quantile(ts, 0.9)),
            "p99_us": float(np.quantile(ts, 0.99)), "min_us": float(ts.min())}


def reference_update(m, A, rows, ys, r):
    ref = os.path.join(ROOT, "baseline", "_ref")
    if not os.path.isdir(os.path.join(ref, "rankrls")):
        return None
    sys.path.insert(0, ref)
    from rankrls import solver as rs

    s = rs.RecursiveSolver(m)
    s.ingest(A[:r], np.zeros(r))
    ts, tp = [], []
    for i in range(len(rows)):
        t0 = time.perf_counter()
        s.update(rows[i], ys[i])
        ts.append(time.perf_counter() - t0)
    for i in range(len(rows)):
        t0 = time.perf_counter()
        s.project(rows[i])
        tp.append(time.perf_counter() - t0)
    sys.path.remove(ref)
    return dist(ts[20:]), dist(tp[20:])


def main():
    import torch

    out = {}
    for m in [int(v) for v in os.environ.get("RGB_LAT_M", "16,64,128,256,1024").split(",")]:
        rng = np.random.default_rng(0)
        A = rng.standard_normal((40, m))
        r = min(20, m)
        rows = rng.standard_normal((600, r)) @ A[:r]
        ys = rng.standard_normal(600)
        s = p.RecursiveSolver(m)
        s.ingest(A[:r], np.zeros(r))
        res = {}
        for name, fn in (("update", lambda i: s.update(rows[i], ys[i])),
                         ("ingest_1row", lambda i: s.ingest(rows[i:i + 1], ys[i:i + 1])),
                         ("project", lambda i: s.project(rows[i]))):
            ts = []
            for i in range(len(rows)):
                t0 = time.perf_counter()
                fn(i)
                ts.append(time.perf_counter() - t0)
            res[name] = dist(ts[20:])
        # breakdown: the row pipe alone (rgb_rowpipe_run: graph launch + spin), no Python work
        pipe = next(iter(s._pipes.values())) if s._pipes else None
        if pipe is not None:
            import ctypes

            lib = s._bs.lib
            h = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
            ts = []
            for _ in range(300):
                t0 = time.perf_counter()
                lib.rgb_rowpipe_run(pipe["h"], h)
                ts.append(time.perf_counter() - t0)
            res["rowpipe_run"] = dist(ts[20:])
        ref = reference_update(m, A, rows[:200], ys[:200], r)
        res["reference_update"], res["reference_project"] = ref if ref else (None, None)
        out[f"m={m}"] = res
        print(f"m={m}", json.dumps(res), flush=True)
    if len(sys.argv) > 1:
        json.dump(out, open(sys.argv[1], "w"), indent=1)


if __name__ == "__main__":
    main()
