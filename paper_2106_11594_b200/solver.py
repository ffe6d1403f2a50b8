"""Drop-in ``RecursiveSolver`` / ``solve_batch`` over the CUDA library.

Same names, arguments, return types and exceptions as rankrls.solver
(/root/reference/pkg/src/rankrls/solver.py), with the factors resident on the
GPU and every update running in librgb.so (a one-stream ``BatchedSolver``):

  RecursiveSolver(num_regressors, *, variant, eps, scalar, alpha)  solver.py:140-171
  .update(row, target) -> UpdateReport                             solver.py:231-250
  .ingest(rows, targets)                                           solver.py:252-319
  .project(row) -> ProjectionResult / .is_dependent(proj, row)     solver.py:210-229
  .solution .rank .num_observations .variant .scalar .eps_policy .basis()
  solve_batch(matrix, targets, ...) -> (x, rank)                   solver.py:406-422

Differences, all deliberate and documented in DESIGN.md:
  * ``solution`` and ``basis()`` return read-only host copies, not live views;
  * RATIONAL (exact mode) and callable ``alpha`` are CPU-only features of the
    reference and raise CapabilityError here;
  * the stored rank has a device capacity that doubles on demand, so streams
    behave as if unbounded (the reference reallocates per row, solver.py:112-117).
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _lib
from .scalars import FLOAT32, FLOAT64, CapabilityError, ScalarKind

VARIANTS = ("general", "orthogonal", "orthonormal")


@dataclass(frozen=True)
class EpsPolicy:
    """Threshold policy (solver.py:32-72): auto / fixed / exact."""

    mode: str
    value: float | None = None

    def __post_init__(self):
        if self.mode not in ("auto", "fixed", "exact"):
            raise ValueError(f"unknown eps mode {self.mode!r}")
        if self.mode == "fixed":
            if self.value is None or self.value < 0:
                raise ValueError("fixed eps requires a nonnegative value")
        elif self.value is not None:
            raise ValueError(f"eps mode {self.mode!r} takes no value")

    @classmethod
    def auto(cls):
        return cls("auto")

    @classmethod
    def fixed(cls, value):
        return cls("fixed", float(value))

    @classmethod
    def exact_zero(cls):
        return cls("exact")

    def threshold(self, num_regressors, rank, machine_epsilon):
        if self.mode == "fixed":
            return self.value
        if self.mode == "exact":
            return 0.0
        m, r = num_regressors, rank
        return (m * m * r + m * r + m) * machine_epsilon


@dataclass(frozen=True)
class ProjectionResult:
    coords: np.ndarray
    rejection: np.ndarray
    rejection_sq_norm: object


@dataclass(frozen=True)
class UpdateReport:
    branch: str
    gain: np.ndarray
    predicted_residual: object
    new_rank: int


def _readonly(a):
    a = np.array(a, copy=True)
    a.flags.writeable = False
    return a


class RecursiveSolver:
    """Online minimum-norm least squares on the GPU (drop-in for rankrls)."""

    def __init__(self, num_regressors, *, variant="general", eps=None, scalar=FLOAT64, alpha=1,
                 device=None, r_cap=None):
        if not isinstance(num_regressors, (int, np.integer)) or num_regressors < 1:
            raise ValueError(f"num_regressors must be a positive integer, got {num_regressors!r}")
        if variant not in VARIANTS:
            raise ValueError(f"unknown variant {variant!r}; expected one of {VARIANTS}")
        if not isinstance(scalar, ScalarKind):
            raise TypeError(f"scalar must be a ScalarKind, got {scalar!r}")
        if variant == "orthonormal" and not scalar.has_sqrt:
            raise CapabilityError(
                "the orthonormal variant needs square roots, which the "
                f"{scalar.name!r} scalar kind does not provide")
        if eps is None:
            eps = EpsPolicy.exact_zero() if scalar.exact else EpsPolicy.auto()
        if scalar.exact and eps.mode != "exact":
            raise ValueError("exact rational scalars require the exact-zero eps policy")
        if not scalar.exact and eps.mode == "exact":
            raise ValueError("the exact-zero eps policy requires rational scalars")
        if scalar.exact:
            raise CapabilityError("exact rational arithmetic is CPU-only (use the reference rankrls)")
        if callable(alpha):
            raise CapabilityError("a callable orthogonal rescaling factor is not supported on the GPU")
        import torch

        from .batched import BatchedSolver

        self._kind = scalar
        self._variant = variant
        self._eps = eps
        self._alpha = alpha
        self._m = int(num_regressors)
        self._trackers = []
        self._coords_chunks = []
        tdtype = torch.float32 if scalar is FLOAT32 else torch.float64
        cap = int(r_cap) if r_cap is not None else min(self._m, 32)
        self._bs = BatchedSolver(1, self._m, k=1, r_cap=cap, variant=variant,
                                 eps=None if eps.mode == "auto" else eps.value,
                                 alpha=float(alpha), dtype=tdtype, device=device)
        self._torch = torch
        self._f32in = False
        self._host = {"rank": 0, "nobs": 0}

    # -- read-only access ---------------------------------------------------
    @property
    def num_regressors(self):
        return self._m

    @property
    def rank(self):
        return self._host["rank"]

    @property
    def num_observations(self):
        return self._host["nobs"]

    @property
    def variant(self):
        return self._variant

    @property
    def scalar(self):
        return self._kind

    @property
    def eps_policy(self):
        return self._eps

    @property
    def solution(self):
        """Read-only host copy of the current minimum-norm solution."""
        return _readonly(self._bs.x_t[0, 0].cpu().numpy())

    def basis(self):
        """Read-only host copies of (C, C_tilde, P_inv)."""
        r = self.rank
        C = self._bs.basis_t[0, :r].cpu().numpy()
        D = C if self._variant == "orthonormal" else self._bs.dual_t[0, :r].cpu().numpy()
        P = self._bs.gram_t[0, :r, :r].cpu().numpy()
        return _readonly(C), _readonly(D), _readonly(P)

    # -- core operations ------------------------------------------------------
    def project(self, row):
        """Coordinates of ``row`` in the stored basis plus its rejection."""
        row = self._kind.vector(row, self._m)
        t = self._torch.as_tensor(row, device=self._bs.device).view(1, self._m)
        coords, rej, rsq, _ = self._bs.project(t)
        r = self.rank
        return ProjectionResult(coords[0, :r].cpu().numpy(), rej[0].cpu().numpy(),
                                float(rsq[0].item()))

    def is_dependent(self, proj, row):
        """Rank test of solver.py:221-229 (a scalar decision, done on the host)."""
        eps = self._eps.threshold(self._m, self.rank, self._kind.machine_epsilon)
        eps_sq = eps * eps
        rej_sq = float(proj.rejection_sq_norm)
        row = np.asarray(row, dtype=np.float64)
        row_sq = float(np.dot(row, row))
        return rej_sq < eps_sq or rej_sq < eps_sq * row_sq

    def update(self, row, target):
        """Ingest one observation; returns an UpdateReport (solver.py:231-250)."""
        row = self._kind.vector(row, self._m)
        target = self._kind.coerce(target)
        out = self._run(row[None, :], np.array([target], dtype=self._kind.dtype), want_report=True)
        branch = "independent" if out["branch"][0] else "dependent"
        return UpdateReport(branch, out["gain"], float(out["resid"][0]), self.rank)

    def ingest(self, rows, targets):
        """Fold a block of observations (solver.py:252-319); validated up front."""
        A = self._kind.matrix(rows)
        if A.shape[1] != self._m:
            raise ValueError(f"rows have {A.shape[1]} columns, expected {self._m}")
        y = self._kind.vector(targets, A.shape[0])
        if A.shape[0]:
            self._run(A, y, want_report=False)

    # -- device plumbing --------------------------------------------------------
    def _buffers(self, n):
        """Pinned host staging and device buffers for calls of up to n rows,
        reused across calls.  A per-row update() is latency bound, so a call is
        one host-to-device copy per input, one ingest, asynchronous copies of
        the counters and the report into pinned memory and one synchronisation,
        all through raw pointers (librgb's rgb_memcpy_async)."""
        torch = self._torch
        buf = getattr(self, "_buf", None)
        if buf is not None and buf["cap"] >= n:
            return buf
        cap = 1 << max(0, (n - 1).bit_length())
        dev, dt, m = self._bs.device, self._bs.dtype, self._m
        t = {
            "rows_h": torch.empty((cap, m), dtype=dt, pin_memory=True),
            "y_h": torch.empty((cap,), dtype=dt, pin_memory=True),
            "rows_d": torch.empty((cap, m), dtype=dt, device=dev),
            "y_d": torch.empty((cap,), dtype=dt, device=dev),
            "branch_d": torch.empty((1, cap), dtype=torch.uint8, device=dev),
            "resid_d": torch.empty((1, cap, 1), dtype=dt, device=dev),
            "gain_d": torch.empty((1, m), dtype=dt, device=dev),
            "branch_h": torch.empty((cap,), dtype=torch.uint8, pin_memory=True),
            "resid_h": torch.empty((cap,), dtype=dt, pin_memory=True),
            "gain_h": torch.empty((m,), dtype=dt, pin_memory=True),
            "nobs_h": torch.empty((1,), dtype=torch.int64, pin_memory=True),
            "cnt_h": torch.empty((2,), dtype=torch.int32, pin_memory=True),
        }
        buf = {"cap": cap, "t": t, "esz": t["y_h"].element_size()}
        buf.update({k + "_np": v.numpy() for k, v in t.items() if not k.endswith("_d")})
        buf.update({k + "_p": v.data_ptr() for k, v in t.items()})
        self._buf = buf
        return buf

    def _structs(self):
        """rgb_config / rgb_state of the single stream, rebuilt when the capacity grows."""
        bs = self._bs
        key = (bs.r_cap, bs.basis_t.data_ptr())
        if getattr(self, "_st_key", None) != key:
            self._st = (bs.config(), bs.state())
            self._st_key = key
        return self._st

    # rows staged per device call: bounds the pinned and device staging buffers
    # (a continuation call is equivalent to one long call)
    _CHUNK_ROWS = 8192
    # bytes per pipelined slice of a large call (0 disables the pipeline)
    _SLICE_BYTES = 4 << 20

    def _pipeline_rows(self, n):
        """Rows per staging slice for a call of n rows, or 0 when one copy is
        cheaper (a few slices at least, each a multiple of 32 rows)."""
        if not self._SLICE_BYTES:
            return 0
        row_bytes = self._m * self._bs.dtype.itemsize
        sub = max(32, (self._SLICE_BYTES // row_bytes) // 32 * 32)
        return sub if n >= 2 * sub else 0

    def _copy_stream(self):
        cs = getattr(self, "_cs", None)
        if cs is None:
            cs = self._cs = self._torch.cuda.Stream(self._bs.device)
        return cs

    def _run(self, A, y, want_report):
        n = A.shape[0]
        res = {}
        for s0 in range(0, n, self._CHUNK_ROWS):
            res = self._run_block(A[s0:s0 + self._CHUNK_ROWS], y[s0:s0 + self._CHUNK_ROWS], want_report)
        return res

    def _run_block(self, A, y, want_report):
        torch = self._torch
        bs = self._bs
        lib = bs.lib
        n = A.shape[0]
        m = self._m
        buf = self._buffers(n)
        esz = buf["esz"]
        stream = torch.cuda.current_stream(bs.device)
        h = ctypes.c_void_p(stream.cuda_stream)
        cp = lib.rgb_memcpy_async
        ingest = lib.rgb_ingest_f32in if self._f32in else lib.rgb_ingest
        done = 0
        res = {}
        sub = self._pipeline_rows(n)
        if sub and not want_report and not self._trackers:
            # a large plain ingest: stage it in slices -- the host copy of
            # slice i+1 into pinned memory and its host-to-device copy (on a
            # side stream) overlap the ingest of slice i; a stream that stops
            # early (rank cap) skips the later slices and is resumed below
            # from the rows already on the device
            cs = self._copy_stream()
            hc = ctypes.c_void_p(cs.cuda_stream)
            cfg, st = self._structs()
            for s0 in range(0, n, sub):
                s1 = min(n, s0 + sub)
                buf["rows_h_np"][s0:s1] = A[s0:s1]
                buf["y_h_np"][s0:s1] = y[s0:s1]
                _lib.check(cp(buf["rows_d_p"] + s0 * m * esz, buf["rows_h_p"] + s0 * m * esz,
                              (s1 - s0) * m * esz, hc), "rgb_memcpy_async")
                _lib.check(cp(buf["y_d_p"] + s0 * esz, buf["y_h_p"] + s0 * esz, (s1 - s0) * esz, hc),
                           "rgb_memcpy_async")
                ev = torch.cuda.Event()
                ev.record(cs)
                stream.wait_event(ev)
                _lib.check(ingest(ctypes.byref(cfg), ctypes.byref(st), buf["rows_d_p"] + s0 * m * esz, 0,
                                  buf["y_d_p"] + s0 * esz, 0, s1 - s0, None, h), "rgb_ingest")
            _lib.check(cp(buf["nobs_h_p"], bs.nobs_t.data_ptr(), 8, h), "rgb_memcpy_async")
            _lib.check(cp(buf["cnt_h_p"], bs.rank_t.data_ptr(), 4, h), "rgb_memcpy_async")
            _lib.check(cp(buf["cnt_h_p"] + 4, bs.status_t.data_ptr(), 4, h), "rgb_memcpy_async")
            stream.synchronize()
            nobs = int(buf["nobs_h_np"][0])
            done = nobs - self._host["nobs"]
            self._host["nobs"] = nobs
            self._host["rank"] = int(buf["cnt_h_np"][0])
            status = int(buf["cnt_h_np"][1])
            if status & _lib.ST_RANK_CAP:
                bs.grow(2 * bs.r_cap)
                bs.status_t.zero_()
            elif status:
                bs.status_t.zero_()
                raise ValueError(f"device status {status}: non-finite input or invalid rescaling factor")
        else:
            buf["rows_h_np"][:n] = A
            buf["y_h_np"][:n] = y
            _lib.check(cp(buf["rows_d_p"], buf["rows_h_p"], n * m * esz, h), "rgb_memcpy_async")
            _lib.check(cp(buf["y_d_p"], buf["y_h_p"], n * esz, h), "rgb_memcpy_async")
        while done < n:
            T = n - done
            log_coords = bool(self._trackers)
            # per-row residuals only for update() reports: requesting them
            # routes the call to the generic kernel (the tensor-core kernels
            # do not log them); every log entry of a consumed row is written
            coords = torch.zeros((1, T, bs.r_cap), dtype=bs.dtype, device=bs.device) if log_coords else None
            logs = _lib.Logs(buf["branch_d_p"] if want_report else None,
                             coords.data_ptr() if log_coords else None,
                             buf["resid_d_p"] if want_report else None,
                             buf["gain_d_p"] if want_report else None)
            cfg, st = self._structs()
            _lib.check(ingest(ctypes.byref(cfg), ctypes.byref(st), buf["rows_d_p"] + done * m * esz, T * m,
                              buf["y_d_p"] + done * esz, T, T, ctypes.byref(logs), h), "rgb_ingest")
            # counters and report: asynchronous copies into pinned memory, one sync
            _lib.check(cp(buf["nobs_h_p"], bs.nobs_t.data_ptr(), 8, h), "rgb_memcpy_async")
            _lib.check(cp(buf["cnt_h_p"], bs.rank_t.data_ptr(), 4, h), "rgb_memcpy_async")
            _lib.check(cp(buf["cnt_h_p"] + 4, bs.status_t.data_ptr(), 4, h), "rgb_memcpy_async")
            if want_report:
                _lib.check(cp(buf["branch_h_p"], buf["branch_d_p"], T, h), "rgb_memcpy_async")
                _lib.check(cp(buf["resid_h_p"], buf["resid_d_p"], T * esz, h), "rgb_memcpy_async")
                _lib.check(cp(buf["gain_h_p"], buf["gain_d_p"], m * esz, h), "rgb_memcpy_async")
            stream.synchronize()
            nobs = int(buf["nobs_h_np"][0])
            rank, status = int(buf["cnt_h_np"][0]), int(buf["cnt_h_np"][1])
            consumed = nobs - self._host["nobs"]
            self._host["nobs"] = nobs
            self._host["rank"] = rank
            if log_coords and consumed:
                self._coords_chunks.append(coords[0, :consumed].cpu().numpy())
            if want_report:
                res = {"branch": buf["branch_h_np"][:consumed].copy(),
                       "resid": buf["resid_h_np"][:consumed].copy(),
                       "gain": buf["gain_h_np"].copy()}
            done += consumed
            if status & _lib.ST_RANK_CAP:
                bs.grow(2 * bs.r_cap)
                bs.status_t.zero_()
            elif status:
                bs.status_t.zero_()
                raise ValueError(f"device status {status}: non-finite input or invalid rescaling factor")
        return res


def solve_batch(matrix, targets, *, variant="general", eps=None, scalar=FLOAT64, alpha=1):
    """Fold all rows of a system through the solver; returns (x, rank) (solver.py:406-422)."""
    A = scalar.matrix(matrix)
    y = scalar.vector(targets)
    if A.shape[0] != y.shape[0]:
        raise ValueError(f"row count mismatch: matrix has {A.shape[0]} rows, targets {y.shape[0]}")
    solver = RecursiveSolver(A.shape[1], variant=variant, eps=eps, scalar=scalar, alpha=alpha)
    solver.ingest(A, y)
    return np.array(solver.solution, copy=True), solver.rank
