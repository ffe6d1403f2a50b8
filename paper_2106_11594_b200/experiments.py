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
        if self.experiment not in EXPERIMENTS:
            raise ValueError(f"unknown experiment {self.experiment!r}")
        if self.repetitions < 3:
            raise ValueError("repetitions must be at least 3")
        if len(self.grid) < 2:
            raise ValueError("need at least two grid sizes")
        swept = [self.swept_size(cell) for cell in self.grid]
        if any(later <= earlier for earlier, later in zip(swept, swept[1:])):
            raise ValueError("grid must be strictly increasing in the swept parameter")
        for n, m, r in self.grid:
            if not 1 <= r <= min(n, m):
                raise ValueError(f"invalid grid cell {(n, m, r)}")

    def swept_size(self, cell):
        n, m, r = cell
        return {"rect-fixed-n": m, "update-cost": r}.get(self.experiment, n)


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
        raise ValueError(f"unknown experiment {experiment!r}")
    grid = tuple(cells[experiment](v) for v in sizes)
    return BenchPlan(experiment, grid, repetitions=repetitions, variant=variant, scalar=scalar, seed=seed)


def fit_loglog(sizes, seconds):
    """Least-squares line through (log size, log t) (bench.py:107-118)."""
    x = np.log(np.asarray(sizes, dtype=np.float64))
    t = np.log(np.asarray(seconds, dtype=np.float64))
    if len(x) < 2:
        raise ValueError("need at least two points to fit")
    slope, icpt = np.polyfit(x, t, 1)
    resid = t - (slope * x + icpt)
    ss_res = float(resid @ resid)
    ss_tot = float(((t - t.mean()) ** 2).sum())
    r2 = 1.0 if ss_tot == 0.0 else max(0.0, 1.0 - ss_res / ss_tot)
    return FitResult(float(slope), math.exp(float(icpt)), r2)


def fit_tail(sizes, seconds):
    """Fit over the largest half of the grid, at least two points (bench.py:121-125)."""
    idx = np.argsort(sizes)
    keep = idx[len(idx) // 2:] if len(idx) > 3 else idx[-2:]
    return fit_loglog([sizes[i] for i in keep], [seconds[i] for i in keep])


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
    n, m, r = cell
    A = random_standardized(n, m, r, _cell_seed(plan, index, 0))
    y = np.random.default_rng(_cell_seed(plan, index, 1)).standard_normal(n)
    return A, y


def update_inputs(plan, index, cell, block=32):
    """(basis rows, their targets, dependent probes, probe targets) of an
    update-cost cell, drawn in the reference's order (bench.py:189-201)."""
    r, m, _ = cell
    rng = np.random.default_rng(_cell_seed(plan, index, 0))
    basis_rows = rng.standard_normal((r, m))
    basis_y = rng.standard_normal(r)
    probes = rng.standard_normal((block, r)) @ basis_rows
    return basis_rows, basis_y, probes, rng.standard_normal(block)


def _solve_cell(plan, index, cell):
    from .solver import solve_batch

    A, y = solve_inputs(plan, index, cell)

    def timed():
        _sync()
        t0 = time.perf_counter()
        solve_batch(A, y, variant=plan.variant, scalar=plan.scalar)
        _sync()
        return time.perf_counter() - t0

    return timed


def _update_cell(plan, index, cell):
    """Per-update cost of dependent rows at rank r, width m (bench.py:187-211)."""
    from .solver import RecursiveSolver

    r, m, _ = cell
    block = 32  # probes per timed quantum
    basis_rows, basis_y, probes, targets = update_inputs(plan, index, cell, block)
    solver = RecursiveSolver(m, variant=plan.variant, scalar=plan.scalar)
    solver.ingest(basis_rows, basis_y)
    if solver.rank != r:
        raise RuntimeError(f"prefix did not reach rank {r}")

    def timed():
        _sync()
        t0 = time.perf_counter()
        solver.ingest(probes, targets)
        _sync()
        per_update = (time.perf_counter() - t0) / block
        if solver.rank != r:
            raise RuntimeError("probe updates unexpectedly grew the rank")
        return per_update

    return timed


def run_plan(plan, progress=None):
    """Run a plan: (samples, fit over per-cell medians) (bench.py:128-163).

    One discarded warm-up per cell, then repetitions interleaved round-robin
    across cells so that drift hits every cell alike.
    """
    make = _update_cell if plan.experiment == "update-cost" else _solve_cell
    timers = [make(plan, i, cell) for i, cell in enumerate(plan.grid)]
    for timer in timers:
        timer()
    times = [[] for _ in plan.grid]
    for _ in range(plan.repetitions):
        for slot, timer in enumerate(timers):
            times[slot].append(timer())
    samples, medians, swept = [], [], []
    for slot, cell in enumerate(plan.grid):
        samples.extend(BenchSample(plan.experiment, *cell, rep, sec) for rep, sec in enumerate(times[slot]))
        medians.append(float(np.median(times[slot])))
        swept.append(plan.swept_size(cell))
        if medians[-1] < MIN_TIMED_SECONDS:
            warnings.warn(f"cell {cell} of {plan.experiment} ran in {medians[-1]:.2e}s; "
                          "timer resolution may dominate", stacklevel=2)
        if progress is not None:
            progress(cell, medians[-1])
    return samples, fit_tail(swept, medians)


def write_csv(samples, path):
    """experiment, n, m, r, rep, seconds (17 significant digits) (bench.py:214-220)."""
    with open(path, "w", newline="", encoding="ascii") as fh:
        out = csv.writer(fh)
        out.writerow(["experiment", "n", "m", "r", "rep", "seconds"])
        for s in samples:
            out.writerow([s.experiment, s.n, s.m, s.r, s.rep, f"{s.seconds:.17g}"])
