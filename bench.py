#!/usr/bin/env python
"""Rank-Greville RLS on B200: observation updates/s (rows x streams) and % of roofline.

Workload (BASELINE.json configs[4], "C5"): B = 65536 independent streams,
n = 1024 rows each, m = 64 regressors, rank 16 (A_b = G1_b G2_b; even b
Gaussian factors, odd b integer factors in {-3..3}), k = 8 right-hand sides,
fp64.  One step = solve every stream from scratch (state reset + one pass of
the hot path over all n rows of all streams).  Weak scaling: each of N GPUs
folds its own 65 536 streams -- contiguous blocks of one global set of
N x 65 536, no collective on the data path; the single-stream configs (rows
strictly sequential) run one replica per GPU.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config c5|c3|c1|c2|c4]
                  [--dtype fp64|fp32|fp32-state] [--impl ours|reference]

`--impl reference` times the CPU oracle port (oracle/rgb_oracle.c, the C
restatement of rankrls' ingest) on the host cores on a bounded sample of the
same workload -- the reference itself is pure Python and cannot travel to the
GPU box.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from paper_2106_11594_b200 import sharding, workloads  # noqa: E402

METRIC = "observation updates/sec (rows x streams, fp64) and % of fp64/HBM roofline"
UNIT = "rows*streams/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", default="c5", choices=sorted(workloads.CONFIGS))
    # fp32: float32 rows/targets widened exactly into a float64 state (fp64
    # arithmetic, fp64 parity; half the input bytes); fp32-state: float32 state
    # and arithmetic (generic kernel, 1e-3 parity)
    ap.add_argument("--dtype", default="fp64", choices=["fp64", "fp32", "fp32-state"])
    ap.add_argument("--eps", type=float, default=None,
                    help="fixed eps policy (EpsPolicy.fixed); default auto for fp64, 1e-5 for fp32 inputs")
    ap.add_argument("--streams", type=int, default=None, help="override B (debug only)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--e2e-chunk", type=int, default=4096)
    ap.add_argument("--dist-backend", default="nccl", choices=["nccl", "gloo"])
    ap.add_argument("--op", default="ingest", choices=["ingest", "pinv", "covariance"],
                    help="pinv / covariance: time the A+ / covariance extraction (rgb_pinv / rgb_covariance) "
                         "from the factors of the config's ingested streams instead of the ingest")
    ap.add_argument("--dump", default=None,
                    help="rank 0 writes the per-stream ranks / status / x of the untimed pass (npz), for tests")
    args = ap.parse_args()
    if args.eps is None and args.dtype == "fp32":
        # float32 inputs carry ~6e-8 relative rounding: the auto policy's fp64
        # threshold would read it as rank, so the fp32 workload runs with a
        # fixed threshold above that noise (the reference's EpsPolicy.fixed)
        args.eps = 1e-5
    return args


# -- algorithmic work --------------------------------------------

def flops_per_row(dep, r, m, k):
    """Reference op count per row, general variant, r = rank before the row:
    dependent r>=1: 6mr + 4r^2 + 3r + 5m + 4mk; dependent r=0: 5m;
    independent: 6mr + 6m + 4mk."""
    if dep:
        return 5 * m if r == 0 else 6 * m * r + 4 * r * r + 3 * r + 5 * m + 4 * m * k
    return 6 * m * r + 6 * m + 4 * m * k


def algorithmic_flops(branch, m, k):
    """Sum of flops_per_row over a branch log [S, T] (uint8, 1 = independent)."""
    import torch

    b = branch.to(torch.int64)
    r_before = torch.cumsum(b, dim=1) - b
    r = r_before.to(torch.float64)
    dep = (b == 0)
    f_dep = torch.where(r == 0, torch.full_like(r, 5.0 * m), 6 * m * r + 4 * r * r + 3 * r + 5 * m + 4 * m * k)
    f_ind = 6 * m * r + 6 * m + 4 * m * k
    return float(torch.where(dep, f_dep, f_ind).sum().item())


def alg_bytes(S, n, m, k, s, sx=None):
    """Compulsory HBM bytes: rows + targets read (s bytes per value), solutions
    written (sx bytes per value, default s), 4 B of rank."""
    sx = s if sx is None else sx
    return s * S * n * (m + k) + sx * S * m * k + 4 * S


# -- clocks ------------------------------------------------------------------------

class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled every 50 ms during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap,timestamp")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.path = None

    def start(self):
        fd, self.path = tempfile.mkstemp(suffix=".csv")
        os.close(fd)
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "50"], stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except OSError:
            self.proc = None
            return
        # wait for the first sample so that the timed region is covered
        t0 = time.time()
        while time.time() - t0 < 5 and os.path.getsize(self.path) == 0:
            time.sleep(0.05)

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        sm, smax, reasons = [], None, set()
        names = ["active", "hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in open(self.path):
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                smax = float(parts[2])
            except ValueError:
                continue
            for nm, v in zip(names[1:], parts[5:9]):
                if v.lower() == "active":
                    reasons.add(nm)
        os.unlink(self.path)
        load = [v for v in sm if smax and v > 0.3 * smax] or sm
        return {"sm_mhz": statistics.median(load) if load else None, "sm_max_mhz": smax,
                "reasons": sorted(reasons), "samples": len(sm)}


def fp64_peak():
    """Live peaks of this GPU (tools/libfp64peak.so), TFLOP/s: fp64 DFMA and DMMA,
    fp32 FFMA (the fp32-state kernel's pipe) and tf32 mma.sync (its G projection)."""
    import ctypes

    from paper_2106_11594_b200 import _build

    try:
        lib = ctypes.CDLL(_build.build_peak_probe())
        lib.rgb_probe_fp64_peak.restype = ctypes.c_double
        return {"dfma": lib.rgb_probe_fp64_peak(0), "dmma": lib.rgb_probe_fp64_peak(1),
                "ffma": lib.rgb_probe_fp64_peak(2), "tf32_mma": lib.rgb_probe_fp64_peak(3)}
    except Exception as e:  # noqa: BLE001
        return {"error": str(e)}


def measured_peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except OSError:
        return {}


def ncu_entry(cfg_name, dtype):
    """The ingest kernel's entry of the committed ncu summary (profiles/ncu_summary.json)."""
    try:
        d = json.load(open(os.path.join(ROOT, "profiles", "ncu_summary.json")))
        return d.get(f"{cfg_name}_{dtype}") or {}
    except (OSError, ValueError):
        return {}


def ncu_traffic(cfg_name, dtype):
    """dram bytes per launch of the ingest kernel from the committed ncu summary."""
    return ncu_entry(cfg_name, dtype).get("dram_bytes_per_launch")


def ncu_pipe_pct(cfg_name, dtype):
    """DMMA pipe utilisation (%) of the ingest kernel from the committed ncu capture."""
    try:
        return float(ncu_entry(cfg_name, dtype).get("dmma_pipe_pct"))
    except (TypeError, ValueError):
        return None


# -- CPU baseline (oracle port, host cores) ------------------------------------------

def _gen_sample(args):
    cfg_name, b = args
    if cfg_name == "c5":
        return workloads.c5_stream(b)
    A, y, _ = workloads.c3_stream(b)
    return A, y[:, None]


def cpu_sample_inputs(cfg_name, count, rows_dev=None, tg_dev=None):
    """The bounded CPU sample: the first `count` streams of the workload (exact
    device bytes when given, else regenerated on the host)."""
    cfg = workloads.CONFIGS[cfg_name]
    if rows_dev is not None:
        return rows_dev[:count].cpu().numpy(), tg_dev[:count].cpu().numpy()
    if cfg_name in ("c5", "c3"):
        try:
            import torch

            if torch.cuda.is_available():  # the GPU arm's bytes (input generation only, no kernel of ours)
                r, t = workloads.device_batch(cfg_name, 0, max(count, 2048), "cuda", chunk=2048)
                out = r[:count].cpu().numpy(), t[:count].cpu().numpy()
                del r, t
                torch.cuda.empty_cache()
                return out
        except Exception:  # noqa: BLE001  (no usable GPU: regenerate on the host)
            pass
        from multiprocessing import Pool

        with Pool(min(16, os.cpu_count() or 1)) as p:
            res = p.map(_gen_sample, [(cfg_name, b) for b in range(count)])
        return np.stack([a for a, _ in res]), np.stack([y for _, y in res])
    A, y = getattr(workloads, cfg_name)()
    return A[None], y[None, :, None]


def cpu_baseline(cfg_name, dtype, rows, tg, reps=1, eps=None):
    from oracle import oracle

    cores = len(os.sched_getaffinity(0))
    cfg = workloads.CONFIGS[cfg_name]
    npdt = np.float32 if dtype == "fp32-state" else np.float64
    if dtype != "fp64":  # float32 data (widened exactly for the fp64-state mode)
        rows, tg = rows.astype(np.float32), tg.astype(np.float32)
    rows = rows.astype(npdt, copy=False)
    tg = tg.astype(npdt, copy=False)
    if rows.shape[0] == 1 and cfg.m * cfg.r > 100000:
        # single large stream: a bounded prefix (the growth rows plus steady-state
        # rows at the full rank) keeps the sample to ~10-30 s of CPU work
        keep = min(rows.shape[1], 2 * cfg.r + 1024)
        rows, tg = rows[:, :keep], tg[:, :keep]
    S, T, _ = rows.shape
    best = None
    for _ in range(reps):
        t0 = time.perf_counter()
        oracle.ingest(rows, tg, r_cap=cfg.r_cap, dtype=npdt, eps=eps,
                      nthreads=cores, logs=False)
        dt = time.perf_counter() - t0
        best = dt if best is None else min(best, dt)
    return {"value": S * T / best, "unit": UNIT, "cores": min(cores, S), "kind": "port",
            "sample": f"{S} streams x {T} rows of {cfg_name} (m={cfg.m}, k={cfg.k}, {dtype}), "
                      f"C oracle oracle/rgb_oracle.c, {min(cores, S)} pthreads, {best:.2f} s"}


# -- reference arm ---------------------------------------------------------------------

def _py_ref_stream(args):
    """One stream through the reference's own solve_batch (baseline/_ref), one
    call per right-hand side (the reference has no multi-RHS API)."""
    rows, tg = args
    from rankrls import solver as ref_solver

    for c in range(tg.shape[1]):
        ref_solver.solve_batch(rows, tg[:, c])
    return rows.shape[0]


def python_reference(rows, tg, cores):
    """The reference package itself (pip-installed into baseline/_ref, the
    unmodified rankrls 0.1.0 `solve_batch`, general variant, auto eps) on a
    small sample of the same streams: multiprocessing.Pool(cores), one stream
    per task, OPENBLAS_NUM_THREADS=1 per worker."""
    ref_dir = os.path.join(ROOT, "baseline", "_ref")
    if not os.path.isdir(os.path.join(ref_dir, "rankrls")):
        return {"unavailable": "baseline/_ref not installed (pip install --target baseline/_ref /root/reference/pkg)"}
    import multiprocessing as mproc

    env_old = os.environ.get("OPENBLAS_NUM_THREADS")
    os.environ["OPENBLAS_NUM_THREADS"] = "1"
    sys.path.insert(0, ref_dir)
    try:
        ctx = mproc.get_context("fork")
        with ctx.Pool(cores) as pool:
            pool.map(_py_ref_stream, [(rows[0, :8], tg[0, :8])] * cores)  # warm-up (imports)
            t0 = time.perf_counter()
            done = sum(pool.map(_py_ref_stream, [(rows[i], tg[i]) for i in range(rows.shape[0])], chunksize=1))
            dt = time.perf_counter() - t0
    finally:
        sys.path.remove(ref_dir)
        if env_old is None:
            os.environ.pop("OPENBLAS_NUM_THREADS", None)
        else:
            os.environ["OPENBLAS_NUM_THREADS"] = env_old
    return {"value": done / dt, "unit": UNIT, "cores": cores, "kind": "reference (Python, baseline/_ref)",
            "sample": f"{rows.shape[0]} streams x {rows.shape[1]} rows, {tg.shape[2] if tg.ndim == 3 else 1} "
                      f"solve_batch calls per stream (one per RHS), {dt:.2f} s measured"}


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    cfg = workloads.CONFIGS[args.config]
    count = {"c5": 2048, "c3": 2048}.get(args.config, 1)
    rows, tg = cpu_sample_inputs(args.config, count)
    for _ in range(args.warmup):
        cpu_baseline(args.config, args.dtype, rows[: min(64, len(rows))], tg[: min(64, len(rows))], eps=args.eps)
    vals = [cpu_baseline(args.config, args.dtype, rows, tg, eps=args.eps) for _ in range(args.steps)]
    v = statistics.median([c["value"] for c in vals])
    cb = dict(vals[0])
    cb["value"] = v
    sample_rows = rows.shape[0] * rows.shape[1]
    n_total = cfg.streams * cfg.n
    py = None
    if cfg.streams > 1 and args.dtype == "fp64" and args.eps is None:
        cores = len(os.sched_getaffinity(0))
        ns = min(len(rows), 8 * cores)
        py = python_reference(rows[:ns], tg[:ns], cores)
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup,
        # each step is the bounded sample, measured; the full-workload time is
        # an extrapolation at the same per-row rate and is labelled as such
        "ms_per_step": 1e3 * sample_rows / v,
        "ms_per_full_workload_extrapolated": 1e3 * n_total / v,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f32" if args.dtype == "fp32-state" else "f64",
        "data": "synthetic (seeded A = G1 G2, SURVEY.md 8(d)); the sample's bytes are the GPU arm's device-generated "
                "streams when a GPU is present",
        "config": {"workload": args.config, "streams": cfg.streams, "streams_per_gpu": cfg.streams, "n": cfg.n,
                   "m": cfg.m, "k": cfg.k, "rank": cfg.r, "sampled_streams": rows.shape[0],
                   "sampled_rows_per_step": sample_rows},
        "cpu_baseline": cb,
        "python_reference": py,
        "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# -- our arm ----------------------------------------------------------------------------

def run_ours(args):
    import torch
    import torch.distributed as dist

    from paper_2106_11594_b200.batched import BatchedSolver

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # one process per GPU; --dist-backend gloo lets a 1-GPU box exercise the
    # multi-rank host logic (ranks share the device, no kernel waits on another)
    local_dev = local % max(1, torch.cuda.device_count())
    torch.cuda.set_device(local_dev)
    device = torch.device("cuda", local_dev)
    if world > 1:
        if args.dist_backend == "nccl":
            dist.init_process_group("nccl", device_id=device)
        else:
            dist.init_process_group("gloo")
    cfg = workloads.CONFIGS[args.config]
    # weak scaling: every GPU folds its own per_gpu streams of one global set of
    # world * per_gpu (ranks take contiguous blocks of global stream ids, no
    # collective on the data path); single-stream configs run one replica per GPU
    per_gpu = args.streams or cfg.streams
    B = per_gpu * world
    b0, b1 = sharding.shard_range(B, world, rank)
    S = b1 - b0
    tdtype = torch.float64 if args.dtype == "fp64" else torch.float32   # inputs
    sdtype = torch.float32 if args.dtype == "fp32-state" else torch.float64  # state / arithmetic
    esize = 4 if args.dtype != "fp64" else 8

    # inputs resident in HBM before timing (generation is not timed)
    if cfg.streams > 1:
        rows, tg = workloads.device_batch(args.config, b0, b1, device, dtype=tdtype)
    else:
        A, y = getattr(workloads, args.config)()
        rows = torch.as_tensor(A[None], dtype=tdtype, device=device)
        tg = torch.as_tensor(y[None, :, None], dtype=tdtype, device=device)
    n = rows.shape[1]
    bs = BatchedSolver(S, cfg.m, k=cfg.k, r_cap=cfg.r_cap, dtype=sdtype, eps=args.eps, device=device)
    stream = torch.cuda.current_stream(device)

    # one untimed pass with the branch log: exact algorithmic work + status census
    branch = torch.zeros((S, n), dtype=torch.uint8, device=device)
    bs.reset()
    bs.ingest(rows, tg, branch_log=branch)
    torch.cuda.synchronize()
    flops = algorithmic_flops(branch, cfg.m, cfg.k)
    status = bs.status.cpu().numpy()
    ranks = bs.rank.cpu().numpy()
    # rows actually folded per step (a stream frozen at the rank capacity or on a
    # non-finite row stops counting observations)
    nobs_local = int(bs.nobs_t.sum().item())
    if args.dump:
        dump = {"rank": sharding.gather_streams(bs.rank_t.cpu(), device).cpu().numpy(),
                "status": sharding.gather_streams(bs.status_t.cpu(), device).cpu().numpy(),
                "nobs": sharding.gather_streams(bs.nobs_t.cpu(), device).cpu().numpy(),
                "x": sharding.gather_streams(bs.x_t.cpu(), device).cpu().numpy(),
                "branch": sharding.gather_streams(branch.cpu(), device).cpu().numpy()}
        if rank == 0:
            np.savez_compressed(args.dump, **dump)
        del dump
    del branch

    def barrier():
        if world > 1:
            if args.dist_backend == "nccl":
                dist.barrier(device_ids=[local_dev])
            else:
                dist.barrier()

    def step(ev=None):
        bs.reset()
        if ev is not None:
            ev[0].record(stream)
        bs.ingest(rows, tg)
        if ev is not None:
            ev[1].record(stream)

    for _ in range(args.warmup):
        step()
    kev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    # inputs smaller than twice L2 (the single-stream configs): flush L2 between
    # steps by writing a 512 MB buffer, outside per-step CUDA events
    in_bytes = (rows.numel() + tg.numel()) * esize
    flush = in_bytes * world < 2 * 126e6
    flush_buf = torch.empty(64 * 1024 * 1024, dtype=torch.float64, device=device) if flush else None
    sev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    clocks = ClockSampler(local_dev)
    barrier()
    torch.cuda.synchronize()
    clocks.start()
    t0.record(stream)
    for i in range(args.steps):
        if flush:
            flush_buf.fill_(float(i))
            sev[i][0].record(stream)
            step(kev[i])
            sev[i][1].record(stream)
        else:
            step(kev[i])
    t1.record(stream)
    torch.cuda.synchronize()
    clk = clocks.stop()
    barrier()
    # device time, max over ranks (sharding.py: no collective inside the timed region)
    local_ms = sum(a.elapsed_time(b) for a, b in sev) if flush else t0.elapsed_time(t1)
    elapsed_ms = sharding.max_over_ranks(local_ms, device)
    kern_ms = sharding.max_over_ranks(statistics.mean(a.elapsed_time(b) for a, b in kev), device)
    flops_total = sharding.sum_over_ranks(flops, device)
    n_cap = int(sharding.sum_over_ranks(int((status & 1).astype(bool).sum()), device))
    n_nonfinite = int(sharding.sum_over_ranks(int((status & 2).astype(bool).sum()), device))

    total_rows = int(sharding.sum_over_ranks(nobs_local, device))
    value = total_rows * args.steps / (elapsed_ms * 1e-3)

    # parity spot check outside the timed region: oracle on this rank's first streams
    parity = None
    if rank == 0:
        from oracle import oracle

        ns = min(16, S)
        r_np, t_np = rows[:ns].cpu().numpy(), tg[:ns].cpu().numpy()
        o = oracle.ingest(r_np.astype(np.float64), t_np.astype(np.float64), r_cap=cfg.r_cap, eps=args.eps,
                          nthreads=8, logs=False)
        x = bs.solution[:ns].cpu().numpy().astype(np.float64)
        xo = oracle.solution(o)
        ok = (o["status"] == 0) & (status[:ns] == 0)
        rank_ref = o["rank"]
        if args.dtype == "fp32-state":
            # fp32 policy: ranks against the oracle's fp32 mode on the
            # same float32 bytes; x against the fp64 oracle within 1e-3 where the
            # fp32 and fp64 oracle ranks agree
            o32 = oracle.ingest(r_np, t_np, r_cap=cfg.r_cap, eps=args.eps, dtype=np.float32, nthreads=8, logs=False)
            ok &= (o32["status"] == 0) & (o32["rank"] == o["rank"])
            rank_ref = o32["rank"]
        errs = [float(np.abs(x[b] - xo[b]).max() / max(1.0, np.abs(xo[b]).max())) for b in range(ns) if ok[b]]
        parity = {"streams": ns, "rank_match": bool(np.array_equal(ranks[:ns][ok], rank_ref[ok])),
                  "x_relerr_max": max(errs) if errs else None,
                  "tolerance": 1e-3 if args.dtype == "fp32-state" else 1e-9}
        # streams the device froze at the rank capacity: the oracle, given room
        # to grow, must run away past the construction rank too (SURVEY.md
        # finding 0.3: the reference itself does on ~1 in 2048 C5 streams)
        capped = np.nonzero(status & 1)[0][:6]
        if len(capped):
            rc_ = torch.tensor(capped, device=device, dtype=torch.long)
            o2 = oracle.ingest(rows[rc_].cpu().numpy().astype(np.float64), tg[rc_].cpu().numpy().astype(np.float64),
                               r_cap=n, eps=args.eps, nthreads=8, logs=False)
            parity["rank_cap_streams_checked"] = int(len(capped))
            parity["rank_cap_oracle_ranks"] = [int(v) for v in o2["rank"]]
            parity["rank_cap_oracle_runaway"] = bool((o2["rank"] > cfg.r).all())

    # end-to-end through the public API from pinned host buffers
    e2e = None
    if not args.no_e2e:
        e2e = run_e2e(args, bs, rows, tg, stream, world, local, device, esize)
        ms = sharding.max_over_ranks(e2e.pop("_ms"), device)
        e2e["value"] = total_rows * e2e.pop("_steps") / (ms * 1e-3)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        count = {"c5": 2048, "c3": 2048}.get(args.config, 1)
        r_s, t_s = cpu_sample_inputs(args.config, min(count, S), rows, tg)
        cpu = cpu_baseline(args.config, args.dtype, r_s, t_s, eps=args.eps)

    if rank == 0:
        peaks = fp64_peak()
        mp = measured_peaks()
        peak_tf = peaks.get("dmma")
        peak_src = "live fp64 DMMA m8n8k4 probe (tools/fp64_peak.cu), this GPU, this run"
        if args.dtype == "fp32-state":
            peak_tf, peak_src = peaks.get("ffma"), "live fp32 FFMA probe (tools/fp64_peak.cu), this GPU, this run"
        achieved = flops_total / world / (kern_ms * 1e-3) / 1e12
        byt = alg_bytes(S, n, cfg.m, cfg.k, esize, 4 if args.dtype == "fp32-state" else 8)
        hbm_gbs = byt / (kern_ms * 1e-3) / 1e9
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": elapsed_ms / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f32" if args.dtype == "fp32-state" else "f64",
            "data": "synthetic: seeded A = G1 G2 per stream generated on device (SURVEY.md 8(d)); inputs resident in HBM",
            "config": {"workload": args.config, "streams": B, "streams_per_gpu": per_gpu, "n": n, "m": cfg.m,
                       "rank": cfg.r, "k": cfg.k,
                       "r_cap": cfg.r_cap, "variant": "general",
                       "eps": "auto" if args.eps is None else f"fixed {args.eps:g}",
                       "inputs": {"fp64": "fp64", "fp32": "fp32, widened exactly into the fp64 state on load",
                                  "fp32-state": "fp32 (fp32 state and arithmetic)"}[args.dtype],
                       "l2": (f"inputs {in_bytes * world / 1e6:.0f} MB < 2x L2: L2 flushed (512 MB write) between "
                              "steps, outside the per-step events" if flush else
                              f"inputs {byt * world / 1e9:.1f} GB >> L2 126 MB (no flush needed)"),
                       "sharding": (f"{S} contiguous streams per GPU of {B}, no collective" if cfg.streams > 1 else
                                    "single stream: one replica per GPU (rows are sequential; replicas only)")},
            "roofline": {"bound": "compute" if args.dtype == "fp32-state" else "tensor", "achieved": achieved, "peak": peak_tf, "unit": "TFLOP/s",
                         "frac": achieved / peak_tf if peak_tf else None,
                         "traffic": ncu_traffic(args.config, args.dtype),
                         "algorithmic_flops_per_launch": flops_total / world,
                         "kernel_ms": kern_ms, "peak_source": peak_src,
                         "note": (("bound by the fp32 CUDA-core pipe (FFMA; the fp32-state kernel rgb_f32.cu, whose "
                                   "G = A C~^T runs as 3-pass tf32 on mma.sync: fp64_peaks_tflops.tf32_mma / 3 is that "
                                   "path's fp32-accurate ceiling); "
                                   if args.dtype == "fp32-state" else
                                   "bound by the fp64 tensor pipe (mma.sync DMMA; tcgen05 has no f64 kind); ") +
                                  "achieved counts the reference's per-row op count (SURVEY.md 8(d)) over the branch "
                                  "log; the kernels execute less: the blocked algebra ~65% of it, and the deferred "
                                  "fold of fresh streams (Q = B^T B accumulated, one inversion per call, DESIGN.md 3) "
                                  "~50%, so frac -- algorithmic flops over the measured peak -- can exceed 1 on "
                                  "config 5; dmma_pipe_pct_ncu (the committed ncu capture, profiles/) is the "
                                  "hardware-side utilisation of the same kernel"),
                         "dmma_pipe_pct_ncu": None if args.dtype == "fp32-state" else ncu_pipe_pct(args.config, args.dtype),
                         "hbm": {"achieved_gbs": hbm_gbs, "peak_gbs": mp.get("hbm_gbs"),
                                 "frac": hbm_gbs / mp["hbm_gbs"] if mp.get("hbm_gbs") else None,
                                 "algorithmic_bytes_per_launch": byt}},
            "fp64_peaks_tflops": peaks,
            "gpu_launches": args.steps,
            "clocks": clk,
            "status": {"rank_cap_streams": n_cap, "nonfinite_streams": n_nonfinite},
            "parity": parity,
            "e2e": e2e,
            "cpu_baseline": cpu,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def run_e2e(args, bs, rows, tg, stream, world, local, device, esize):
    """Same metric through BatchedSolver.ingest_host: every step copies that
    step's rows/targets from pinned host memory (chunked, overlapped with the
    kernel) and reads the solutions and ranks back to pinned host memory."""
    import torch

    S, n, m = rows.shape
    k = tg.shape[2]
    need = (rows.numel() + tg.numel()) * esize
    avail = 0
    try:
        for line in open("/proc/meminfo"):
            if line.startswith("MemAvailable"):
                avail = int(line.split()[1]) * 1024
    except OSError:
        pass
    S_e = S
    if avail and need * world > 0.6 * avail:
        S_e = max(args.e2e_chunk, int(S * 0.6 * avail / (need * world)) // args.e2e_chunk * args.e2e_chunk)
        S_e = min(S_e, S)
    rows_h = torch.empty((S_e, n, m), dtype=rows.dtype, pin_memory=True)
    tg_h = torch.empty((S_e, n, k), dtype=tg.dtype, pin_memory=True)
    rows_h.copy_(rows[:S_e])
    tg_h.copy_(tg[:S_e])
    x_h = torch.empty((S_e, k, m), dtype=bs.dtype, pin_memory=True)
    r_h = torch.empty(S_e, dtype=torch.int32, pin_memory=True)
    from paper_2106_11594_b200.batched import BatchedSolver

    sub = bs if S_e == S else BatchedSolver(S_e, m, k=k, r_cap=bs.r_cap, dtype=bs.dtype, device=device)

    def step():
        sub.reset()
        launches = sub.ingest_host(rows_h, tg_h, chunk=args.e2e_chunk)
        x_h.copy_(sub.x_t, non_blocking=True)
        r_h.copy_(sub.rank_t, non_blocking=True)
        return launches

    step()
    torch.cuda.synchronize()
    steps = max(1, min(args.steps, 3))
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0.record(stream)
    for _ in range(steps):
        step()
    t1.record(stream)
    torch.cuda.synchronize()
    ms = t0.elapsed_time(t1)
    scale = S / S_e
    return {"_ms": ms * scale, "_steps": steps, "unit": UNIT,
            "h2d_bytes_per_step": int((rows_h.numel() + tg_h.numel()) * esize),
            "d2h_bytes_per_step": int(x_h.numel() * x_h.element_size() + r_h.numel() * 4),
            "streams_measured": S_e, "chunk_streams": args.e2e_chunk,
            "note": "pinned host -> device copies overlapped with ingest; value scaled to the full batch"
                    if S_e != S else "pinned host -> device copies overlapped with ingest (BatchedSolver.ingest_host)"}


# -- process launch -------------------------------------------------------------------

# -- extraction (A+ / covariance) ------------------------------------------------------

def run_extract(args):
    """rgb_pinv / rgb_covariance timed on the device: the config's streams are
    ingested once (with the coords log, untimed), then each step extracts A+
    (m x n per stream, PseudoinverseTracker.pinv / pinv_from_scratch,
    tracking.py:19-85, 128-142) or the covariance (m x m, CovarianceTracker,
    tracking.py:88-119).  L2 is flushed between steps when the data fits in it."""
    import torch

    from paper_2106_11594_b200.batched import BatchedSolver

    torch.cuda.set_device(0)
    device = torch.device("cuda", 0)
    cfg = workloads.CONFIGS[args.config]
    S = args.streams or cfg.streams
    if cfg.streams > 1:
        rows, tg = workloads.device_batch(args.config, 0, S, device)
    else:
        A, y = getattr(workloads, args.config)()
        rows = torch.as_tensor(A[None], device=device)
        tg = torch.as_tensor(y[None, :, None], device=device)
    n, m = rows.shape[1], cfg.m
    bs = BatchedSolver(S, m, k=cfg.k, r_cap=cfg.r_cap, device=device)
    coords = torch.zeros((S, n, cfg.r_cap), dtype=torch.float64, device=device)
    bs.ingest(rows, tg, coords_log=coords)
    torch.cuda.synchronize()
    del rows, tg
    ranks = bs.rank.to(torch.float64)
    ncols = n if args.op == "pinv" else m
    # algorithmic work (closed form C~^T P^-1 F, F = B^T or C~): the m x r x ncols
    # contraction plus V = P^-1 C~ (r x r x m), r the stream's rank
    flops = float((2 * m * ncols * ranks + 2 * ranks * ranks * m).sum().item())
    # compulsory bytes: the output, the coords log (pinv), C~ and P^-1 at the rank
    byt = float((8 * (m * ncols + (n * ranks if args.op == "pinv" else 0) + ranks * m + ranks * ranks)).sum().item())
    run = (lambda: bs.pinv(coords)) if args.op == "pinv" else bs.covariance
    flush = byt < 2 * 126e6
    flush_buf = torch.empty(64 * 1024 * 1024, dtype=torch.float64, device=device) if flush else None
    for _ in range(args.warmup):
        out = run()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    torch.cuda.synchronize()
    clocks = ClockSampler(0)
    clocks.start()
    for i in range(args.steps):
        if flush:
            flush_buf.fill_(float(i))
        ev[i][0].record()
        out = run()
        ev[i][1].record()
    torch.cuda.synchronize()
    clk = clocks.stop()
    ms = statistics.median(a.elapsed_time(b) for a, b in ev)
    peaks = fp64_peak()
    mp = measured_peaks()
    tf = flops / (ms * 1e-3) / 1e12
    gbs = byt / (ms * 1e-3) / 1e9
    line = {
        "metric": f"{args.op} extraction time", "value": ms, "unit": "ms", "higher_is_better": False,
        "n_gpus": 1, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "dtype": "f64",
        "data": "synthetic (seeded A = G1 G2, SURVEY.md 8(d))",
        "config": {"workload": args.config, "op": args.op, "streams": S, "n": n, "m": m, "r_cap": cfg.r_cap,
                   "output": f"[{S}, {m}, {ncols}] fp64", "l2": "flushed between steps" if flush else "data >> L2"},
        "roofline": {"bound": "tensor", "achieved": tf, "peak": peaks.get("dmma"), "unit": "TFLOP/s",
                     "frac": tf / peaks["dmma"] if peaks.get("dmma") else None,
                     "algorithmic_flops_per_launch": flops,
                     "hbm": {"achieved_gbs": gbs, "peak_gbs": mp.get("hbm_gbs"),
                             "frac": gbs / mp["hbm_gbs"] if mp.get("hbm_gbs") else None,
                             "algorithmic_bytes_per_launch": byt}},
        "gpu_launches": args.steps * 2,
        "clocks": clk,
        "out_checksum": float(out.abs().sum().item()),
    }
    print(json.dumps(line), flush=True)
    return 0


def _free_port():
    import socket

    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        return sk.getsockname()[1]


def launch_ranks(n, argv, env=None):
    """One process per GPU without torchrun: start `argv` n times with RANK /
    LOCAL_RANK / WORLD_SIZE / MASTER_ADDR / MASTER_PORT set (the same env
    torchrun gives each rank), wait for all, return the first non-zero exit
    code.  If one rank fails the others are stopped by PID (a rank stuck in a
    collective would otherwise wait forever)."""
    port = _free_port()
    procs = []
    for r in range(n):
        e = dict(os.environ if env is None else env, RANK=str(r), LOCAL_RANK=str(r), WORLD_SIZE=str(n),
                 LOCAL_WORLD_SIZE=str(n), MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        procs.append(subprocess.Popen(argv, env=e))
    rc = 0
    live = list(procs)
    while live:
        for p in list(live):
            code = p.poll()
            if code is None:
                continue
            live.remove(p)
            if code != 0 and rc == 0:
                rc = code
                for q in live:
                    q.terminate()
        time.sleep(0.05)
    return rc


def main():
    args = parse()
    world_env = os.environ.get("WORLD_SIZE")
    if args.impl == "reference":
        return run_reference(args)
    if world_env is None and args.gpus > 1:
        # `python bench.py --gpus N`: spawn the N ranks ourselves
        return launch_ranks(args.gpus, [sys.executable, os.path.abspath(__file__)] + sys.argv[1:])
    if world_env is not None and int(world_env) != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world_env}; launch one rank per GPU "
                         "with matching counts")
    if args.op != "ingest":
        return run_extract(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
