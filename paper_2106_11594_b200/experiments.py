"""Scaling experiments on the device: the reference's bench backend (SURVEY.md
section 8(f), rank 4) driven through this package's solvers.

Mirrors ``rankrls.bench`` (bench.py:1-215): the same four experiments, grid
builder, plan validation, log-log fit over the largest half of the grid,
interleaved repetitions after one discarded warm-up per cell, seeded cell
inputs and CSV layout -- so the paper's scaling figures can be regenerated on
a B200 with the reference's own methodology.  Cells call ``solve_batch`` /
``RecursiveSolver.ingest`` of this package (librgb.so kernels); each timed
quantum is bracketed by ``torch.cuda.synchronize()`` so it measures the whole
call as the user sees it (host arrays in, host solution out), like the
reference's ``time.perf_counter`` cells.
"""

from __future__ import annotations

import csv
import math
import time
import warnings
from dataclasses import dataclass

import numpy as np

from .scalars import FLOAT64
from .workloads import random_standardized

EXPERIMENTS = ("square", "rect-fixed-n", "rank-fixed-r", "update-cost")

# quanta shorter than this are at the mercy of timer resolution (bench.py:31-33)
MIN_TIMED_SECONDS = 1e-3


@dataclass(frozen=True)
class FitResult:
    """t = prefactor * size ** exponent (bench.py:36-42)."""

    exponent: float
    prefactor: float
    r_squared: float


@dataclass(frozen=True)
class BenchSample:
    experiment: str
    n: int
    m: int
    r: int
    rep: int
    seconds: float


@dataclass(frozen=True)
class BenchPlan:
    """A size grid and its measurement settings (bench.py:55-87)."""

    experiment: str
    grid: tuple
    repetitions: int = 5
    variant: str = "general"
    scalar: object = FLOAT64
    seed: int = 0

    def __post_init__(self):
        _validate(self)

    def swept_size(self, cell):
        """The grid coordinate an experiment varies: m, r, or n."""
        return {"rect-fixed-n": cell[1], "update-cost": cell[2]}.get(self.experiment, cell[0])


def _validate(plan):
    """ValueError for a malformed plan (the reference's checks, bench.py:65-78)."""
    problems = []
    if plan.experiment not in EXPERIMENTS:
        problems.append(f"experiment must be one of {EXPERIMENTS}, got {plan.experiment!r}")
    elif plan.repetitions < 3:
        problems.append(f"at least 3 repetitions are required, got {plan.repetitions}")
    elif len(plan.grid) < 2:
        problems.append("a plan needs two or more grid cells")
    else:
        sizes = np.array([plan.swept_size(c) for c in plan.grid])
        if (np.diff(sizes) <= 0).any():
            problems.append(f"swept sizes must increase strictly, got {sizes.tolist()}")
        bad = [c for c in plan.grid if not (1 <= c[2] <= min(c[0], c[1]))]
        if bad:
            problems.append(f"cells need 1 <= r <= min(n, m): {bad}")
    if problems:
        raise ValueError(problems[0])


def make_plan(experiment, sizes, *, fixed_n=100, fixed_r=100, fixed_m=2000, repetitions=5,
              variant="general", scalar=FLOAT64, seed=0):
    """Grid of (n, m, r) cells for an experiment (bench.py:89-104)."""
    sizes = [int(v) for v in sizes]
    cells = {
        "square": lambda v: (v, v, v),
        "rect-fixed-n": lambda v: (fixed_n, v, fixed_n),
        "rank-fixed-r": lambda v: (v, v, fixed_r),
        "update-cost": lambda v: (v, fixed_m, v),
    }
    if experiment not in cells:
        raise ValueError(f"experiment must be one of {EXPERIMENTS}, got {experiment!r}")
    grid = tuple(cells[experiment](v) for v in sizes)
    return BenchPlan(experiment, grid, repetitions=repetitions, variant=variant, scalar=scalar, seed=seed)


def fit_loglog(sizes, seconds):
    """Least-squares line through (log size, log t) (bench.py:107-118)."""
    x = np.log(np.asarray(sizes, dtype=np.float64))
    t = np.log(np.asarray(seconds, dtype=np.float64))
    if len(x) < 2:
        raise ValueError("a power-law fit needs two or more points")
    slope, icpt = np.polyfit(x, t, 1)
    resid = t - (slope * x + icpt)
    ss_res = float(resid @ resid)
    ss_tot = float(((t - t.mean()) ** 2).sum())
    r2 = 1.0 if ss_tot == 0.0 else max(0.0, 1.0 - ss_res / ss_tot)
    return FitResult(float(slope), math.exp(float(icpt)), r2)


def fit_tail(sizes, seconds):
    """Fit over the largest half of the grid, at least two points (bench.py:121-125)."""
    order = np.argsort(sizes)
    tail = order[len(order) // 2:] if len(order) > 3 else order[-2:]
    return fit_loglog(np.asarray(sizes)[tail], np.asarray(seconds)[tail])


def _sync():
    import torch

    if torch.cuda.is_available():
        torch.cuda.synchronize()


def _cell_seed(plan, index, stream):
    """Per-cell generator seed (bench.py:166-168), so cells match the reference's inputs."""
    seq = np.random.SeedSequence([plan.seed, index, stream])
    return int(seq.generate_state(1, dtype=np.uint64)[0])


def solve_inputs(plan, index, cell):
    """(A, y) of a solve cell: seeded exactly as the reference's (bench.py:176-178)."""
    rows, cols, rank = cell
    matrix = random_standardized(rows, cols, rank, _cell_seed(plan, index, 0))
    targets = np.random.default_rng(_cell_seed(plan, index, 1)).standard_normal(rows)
    return matrix, targets


def update_inputs(plan, index, cell, block=32):
    """(basis rows, their targets, dependent probes, probe targets) of an
    update-cost cell, drawn in the reference's order (bench.py:189-201)."""
    rank, width = cell[0], cell[1]
    gen = np.random.default_rng(_cell_seed(plan, index, 0))
    basis = gen.standard_normal((rank, width))
    basis_y = gen.standard_normal(rank)
    probes = gen.standard_normal((block, rank)) @ basis
    return basis, basis_y, probes, gen.standard_normal(block)


def _solve_cell(plan, index, cell):
    from .solver import solve_batch

    matrix, targets = solve_inputs(plan, index, cell)

    def timed():
        _sync()
        t0 = time.perf_counter()
        solve_batch(matrix, targets, variant=plan.variant, scalar=plan.scalar)
        _sync()
        return time.perf_counter() - t0

    return timed


def _update_cell(plan, index, cell):
    """Per-update cost of dependent rows at rank r, width m (bench.py:187-211)."""
    from .solver import RecursiveSolver

    rank, width = cell[0], cell[1]
    block = 32  # probes per timed quantum
    basis, basis_y, probes, probe_y = update_inputs(plan, index, cell, block)
    s = RecursiveSolver(width, variant=plan.variant, scalar=plan.scalar)
    s.ingest(basis, basis_y)
    if s.rank != rank:
        raise RuntimeError(f"the basis prefix reached rank {s.rank}, expected {rank}")

    def timed():
        _sync()
        t0 = time.perf_counter()
        s.ingest(probes, probe_y)
        _sync()
        dt = time.perf_counter() - t0
        if s.rank != rank:
            raise RuntimeError("a dependent probe changed the rank")
        return dt / block

    return timed


def _device_solve_cell(plan, index, cell):
    """Device time (CUDA events) of a solve from scratch on inputs already in
    HBM: the state reset and the ingest kernel(s), without the host round trip."""
    import torch

    from .batched import BatchedSolver

    matrix, targets = solve_inputs(plan, index, cell)
    n, m, r = cell
    rows = torch.as_tensor(matrix[None], device="cuda")
    tg = torch.as_tensor(targets[None, :, None], device="cuda")
    # the capacity the drop-in solver reaches for a rank-r stream (it doubles from 32)
    cap = min(m, 1 << max(5, (r - 1).bit_length()))
    bs = BatchedSolver(1, m, k=1, r_cap=cap, variant=plan.variant)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)

    def timed():
        bs.reset()
        e0.record()
        bs.ingest(rows, tg)
        e1.record()
        e1.synchronize()
        if int(bs.status[0]) != 0:
            raise RuntimeError(f"cell {cell}: device status {int(bs.status[0])}")
        return e0.elapsed_time(e1) * 1e-3

    return timed


def _device_update_cell(plan, index, cell):
    """Device time per dependent update: a block of probes folded into a
    rank-r state (inputs in HBM)."""
    import torch

    from .batched import BatchedSolver

    rank, width = cell[0], cell[1]
    block = 32
    basis, basis_y, probes, probe_y = update_inputs(plan, index, cell, block)
    cap = 1 << max(3, (rank - 1).bit_length())
    bs = BatchedSolver(1, width, k=1, r_cap=cap, variant=plan.variant)
    bs.ingest(torch.as_tensor(basis[None], device="cuda"), torch.as_tensor(basis_y[None, :, None], device="cuda"))
    if int(bs.rank[0]) != rank:
        raise RuntimeError(f"the basis prefix reached rank {int(bs.rank[0])}, expected {rank}")
    rows = torch.as_tensor(probes[None], device="cuda")
    tg = torch.as_tensor(probe_y[None, :, None], device="cuda")
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)

    def timed():
        e0.record()
        bs.ingest(rows, tg)
        e1.record()
        e1.synchronize()
        return e0.elapsed_time(e1) * 1e-3 / block

    return timed


def run_plan(plan, progress=None, clock="wall"):
    """Run a plan: (samples, fit over per-cell medians) (bench.py:128-163).

    One discarded warm-up per cell, then repetitions interleaved round-robin
    across cells so that drift hits every cell alike.  clock="wall" times the
    drop-in call as the reference does (host arrays in, host results out);
    clock="device" times the device work alone with CUDA events on inputs
    already in HBM (the B200-side scaling of the same cells).
    """
    if clock not in ("wall", "device"):
        raise ValueError(f"clock must be 'wall' or 'device', got {clock!r}")
    if clock == "device":
        build = _device_update_cell if plan.experiment == "update-cost" else _device_solve_cell
    else:
        build = _update_cell if plan.experiment == "update-cost" else _solve_cell
    cells = list(plan.grid)
    runners = [build(plan, i, cell) for i, cell in enumerate(cells)]
    for run in runners:  # warm-up, discarded
        run()
    # rounds[rep][i]: repetition rep of cell i
    rounds = [[run() for run in runners] for _ in range(plan.repetitions)]
    per_cell = np.array(rounds).T
    samples = [BenchSample(plan.experiment, *cell, rep, float(sec))
               for cell, row in zip(cells, per_cell) for rep, sec in enumerate(row)]
    medians = np.median(per_cell, axis=1)
    for cell, med in zip(cells, medians):
        if med < MIN_TIMED_SECONDS:
            warnings.warn(f"cell {cell} of {plan.experiment} ran in {med:.2e}s; "
                          "timer resolution may dominate", stacklevel=2)
        if progress is not None:
            progress(cell, float(med))
    return samples, fit_tail([plan.swept_size(c) for c in cells], medians.tolist())


def write_csv(samples, path):
    """experiment, n, m, r, rep, seconds (17 significant digits) (bench.py:214-220)."""
    with open(path, "w", newline="", encoding="ascii") as fh:
        out = csv.writer(fh)
        out.writerow(["experiment", "n", "m", "r", "rep", "seconds"])
        out.writerows([b.experiment, b.n, b.m, b.r, b.rep, f"{b.seconds:.17g}"] for b in samples)
