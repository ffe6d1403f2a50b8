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
  * ``solution`` is a live read-only view as in the reference, but of a pinned
    host mirror that each call refreshes; ``basis()`` returns read-only copies;
  * RATIONAL (exact mode) and callable ``alpha`` are CPU-only features of the
    reference and raise CapabilityError here;
  * the stored rank has a device capacity that doubles on demand, so streams
    behave as if unbounded (the reference reallocates per row, solver.py:112-117);
  * ``update`` and ``ingest`` are not bitwise interchangeable.  The reference
    guarantees that folding ``update`` row by row equals ``ingest`` bit for bit
    (test_solver.py:212-222).  Here ``update`` runs on the shape-generic kernel
    (the only one that reports the per-row a-priori residual), while ``ingest``
    runs on the tensor-core kernels (m 64 / 128 / 256 / up to 1 080 / up to
    4 736), whose summation orders differ.  The two agree on rank and on every
    branch outside the rank test's noise band, and x agrees to ~1e-13
    (tests/test_gpu_parity.py::test_update_fold_matches_ingest).
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
        # pinned host mirror of x (first right-hand side): the live `solution` view
        self._xh = torch.zeros(self._m, dtype=tdtype, pin_memory=True)
        self._x_np = self._xh.numpy()
        self._pipes = {}  # one-row pipes (librgb rgb_rowpipe), by layout; None: unsupported
        self._fast = {}   # want_report -> the current pipe's handles, unpacked for update() / ingest()

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
        """Live read-only view of the current minimum-norm solution
        (solver.py:200-202): a view of a pinned host mirror that every call
        refreshes (the row pipe's kernel writes it directly), so a view taken
        earlier follows later updates, as the reference's does."""
        v = self._x_np.view()
        v.flags.writeable = False
        return v

    def basis(self):
        """Read-only host copies of (C, C_tilde, P_inv)."""
        r = self.rank
        C = self._bs.basis_t[0, :r].cpu().numpy()
        D = C if self._variant == "orthonormal" else self._bs.dual_t[0, :r].cpu().numpy()
        P = self._bs.gram_t[0, :r, :r].cpu().numpy()
        return _readonly(C), _readonly(D), _readonly(P)

    # -- core operations ------------------------------------------------------
    def project(self, row):
        """Coordinates of ``row`` in the stored basis plus its rejection
        (solver.py:210-219): through the row server when the solver has one (the
        state is already in its shared memory), else one projection kernel."""
        row = self._kind.vector(row, self._m)
        if not self._trackers and self._pipes is not None:
            pipe = self._row_pipe(True)
            if pipe is not None and pipe.get("proj") is not None:
                m = self._m
                pipe["in"][:m] = row
                rc = self._bs.lib.rgb_rowpipe_project(pipe["h"], pipe["stream"])
                if rc == _lib.OK:
                    pc, pr, ps = pipe["proj"]
                    return ProjectionResult(pc[:self.rank].copy(), pr.copy(), float(ps[0]))
                if rc != _lib.E_UNSUPPORTED:
                    _lib.check(rc, "rgb_rowpipe_project")
        torch = self._torch
        bs = self._bs
        m, rc = self._m, bs.r_cap
        buf = self._buffers(1)
        esz = buf["esz"]
        pb = getattr(self, "_pbuf", None)
        if pb is None or pb[0] != rc:
            # device block: coords [r_cap] | rejection [m] | rej_sq | dependent flag
            nbytes = esz * (rc + m + 1) + 8
            pd = torch.empty((nbytes,), dtype=torch.uint8, device=bs.device)
            ph = torch.empty((nbytes,), dtype=torch.uint8, pin_memory=True)
            npdt = np.float32 if bs.dtype == torch.float32 else np.float64
            pb = self._pbuf = (rc, pd, ph, ph.numpy()[:esz * (rc + m + 1)].view(npdt))
        _, pd, ph, pv = pb
        buf["in_np"][:m] = row
        stream = torch.cuda.current_stream(bs.device)
        h = ctypes.c_void_p(stream.cuda_stream)
        cp = bs.lib.rgb_memcpy_async
        _lib.check(cp(buf["in_d_p"], buf["in_h_p"], m * esz, h), "rgb_memcpy_async")
        cfg, st = self._structs()
        base = pd.data_ptr()
        _lib.check(bs.lib.rgb_project(ctypes.byref(cfg), ctypes.byref(st), buf["in_d_p"], base,
                                      base + esz * rc, base + esz * (rc + m), base + esz * (rc + m + 1), h),
                   "rgb_project")
        _lib.check(cp(ph.data_ptr(), base, esz * (rc + m + 1), h), "rgb_memcpy_async")
        stream.synchronize()
        r = self.rank
        return ProjectionResult(pv[:r].copy(), pv[rc:rc + m].copy(), float(pv[rc + m]))

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
        fast = self._fast.get(True) if self._fast else None
        if fast is not None and fast[0] == self._st_key:
            # the steady-state per-row path: stage, one row-pipe run, read the report
            _, pin, run, h, s, hdr_n, hdr_c, hdr_b, resid, gain = fast
            m = self._m
            pin[:m] = row
            pin[m] = target
            rc = run(h, s)
            if rc:
                _lib.check(rc, "rgb_rowpipe_run")
            nobs = int(hdr_n[0])
            host = self._host
            if nobs != host["nobs"] and not hdr_c[1]:
                host["nobs"] = nobs
                rank = host["rank"] = int(hdr_c[0])
                return UpdateReport("independent" if hdr_b[0] else "dependent", gain.copy(), float(resid[0]), rank)
            # a stop (rank capacity, bad rescaling): the general path handles it
            consumed = nobs - host["nobs"]
            host["nobs"], host["rank"] = nobs, int(hdr_c[0])
            self._on_status(int(hdr_c[1]))
            if consumed:
                return UpdateReport("independent" if hdr_b[0] else "dependent", gain.copy(), float(resid[0]),
                                    self.rank)
        out = self._run(row[None, :], np.array([target], dtype=self._kind.dtype), want_report=True)
        branch = "independent" if out["branch"][0] else "dependent"
        return UpdateReport(branch, out["gain"], float(out["resid"][0]), self.rank)

    def ingest(self, rows, targets):
        """Fold a block of observations (solver.py:252-319); validated up front."""
        A = self._kind.matrix(rows)
        if A.shape[1] != self._m:
            raise ValueError(f"rows have {A.shape[1]} columns, expected {self._m}")
        y = self._kind.vector(targets, A.shape[0])
        fast = self._fast.get(True) if self._fast else None  # the one pipe (its report goes unread)
        if A.shape[0] == 1 and fast is not None and fast[0] == self._st_key:
            _, pin, run, h, s, hdr_n, hdr_c = fast[:7]
            m = self._m
            pin[:m] = A[0]
            pin[m] = y[0]
            rc = run(h, s)
            if rc:
                _lib.check(rc, "rgb_rowpipe_run")
            nobs = int(hdr_n[0])
            consumed = nobs - self._host["nobs"]
            self._host["nobs"], self._host["rank"] = nobs, int(hdr_c[0])
            if consumed and not hdr_c[1]:
                return
            self._on_status(int(hdr_c[1]))
            if consumed:
                return
        if A.shape[0]:
            self._run(A, y, want_report=False)

    # -- device plumbing --------------------------------------------------------
    def _buffers(self, n):
        """Pinned host staging and device buffers for calls of up to n rows,
        reused across calls.  A per-row update() is latency bound, so a call is
        one host-to-device copy (rows and targets packed in one block), one
        ingest, one device-to-host copy of a packed report block and one
        synchronisation, all through raw pointers (librgb's rgb_memcpy_async).

        Report block (bytes): nobs int64 | rank int32 | status int32 | gain
        [m] | branch [cap, padded to 8] | resid [cap].  The solver's counters
        live at its head (rebound on every reallocation), so the one copy
        brings back the counters with the report."""
        torch = self._torch
        buf = getattr(self, "_buf", None)
        if buf is not None and buf["cap"] >= n:
            return buf
        cap = 1 << max(0, (n - 1).bit_length())
        bs = self._bs
        dev, dt, m = bs.device, bs.dtype, self._m
        esz = torch.empty((), dtype=dt).element_size()
        off_gain = 16
        off_branch = off_gain + esz * m
        off_resid = off_branch + (cap + 7) // 8 * 8
        nbytes = off_resid + esz * cap
        t = {
            "in_h": torch.empty((cap * (m + 1),), dtype=dt, pin_memory=True),
            "in_d": torch.empty((cap * (m + 1),), dtype=dt, device=dev),
            "io_h": torch.zeros((nbytes,), dtype=torch.uint8, pin_memory=True),
            "io_d": torch.zeros((nbytes,), dtype=torch.uint8, device=dev),
        }
        io = t["io_d"]
        if buf is not None:
            io[:16].copy_(buf["t"]["io_d"][:16])
        else:
            io[0:8].view(torch.int64).copy_(bs.nobs_t)
            io[8:12].view(torch.int32).copy_(bs.rank_t)
            io[12:16].view(torch.int32).copy_(bs.status_t)
        bs.nobs_t = io[0:8].view(torch.int64)
        bs.rank_t = io[8:12].view(torch.int32)
        bs.status_t = io[12:16].view(torch.int32)
        ioh = t["io_h"].numpy()
        npdt = np.dtype(np.float32 if dt == torch.float32 else np.float64)
        buf = {"cap": cap, "t": t, "esz": esz, "off_gain": off_gain, "off_branch": off_branch,
               "off_resid": off_resid, "in_np": t["in_h"].numpy(),
               "nobs_np": ioh[0:8].view(np.int64), "cnt_np": ioh[8:16].view(np.int32),
               "gain_np": ioh[off_gain:off_branch].view(npdt), "branch_np": ioh[off_branch:off_branch + cap],
               "resid_np": ioh[off_resid:].view(npdt)}
        buf.update({k + "_p": v.data_ptr() for k, v in t.items()})
        self._buf = buf
        return buf

    def _structs(self):
        """rgb_config / rgb_state of the single stream, rebuilt when the capacity
        grows or the counters move."""
        bs = self._bs
        key = (bs.r_cap, bs.basis_t.data_ptr(), bs.nobs_t.data_ptr())
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
        in_h, in_d = buf["in_h_p"], buf["in_d_p"]
        io_h, io_d = buf["io_h_p"], buf["io_d_p"]
        y_off = n * m  # the targets follow the rows in the staging block
        if n == 1 and not self._trackers and self._pipes is not None:
            # a per-row call: the row pipe (one graph launch; the kernel reads the
            # row from mapped host memory and writes the report back into it)
            pipe = self._row_pipe(True)  # one pipe per layout (one row server per state)
            if pipe is not None:
                pipe["in"][:m] = A[0]
                pipe["in"][m] = y[0]
                _lib.check(lib.rgb_rowpipe_run(pipe["h"], pipe["stream"]), "rgb_rowpipe_run")
                hdr = pipe["hdr"]
                nobs, status = int(hdr["nobs"][0]), int(hdr["cnt"][1])
                consumed = nobs - self._host["nobs"]
                self._host["nobs"] = nobs
                self._host["rank"] = int(hdr["cnt"][0])
                if consumed:
                    self._on_status(status)
                    if want_report:
                        return {"branch": hdr["branch"].copy(), "resid": pipe["resid"].copy(),
                                "gain": pipe["gain"].copy()}
                    return {}
                self._on_status(status)  # rank cap: grown; the row runs again below
        self._quiesce()  # other kernels write the state: the row server stops first
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
                buf["in_np"][s0 * m:s1 * m] = A[s0:s1].reshape(-1)
                buf["in_np"][y_off + s0:y_off + s1] = y[s0:s1]
                _lib.check(cp(in_d + s0 * m * esz, in_h + s0 * m * esz, (s1 - s0) * m * esz, hc),
                           "rgb_memcpy_async")
                _lib.check(cp(in_d + (y_off + s0) * esz, in_h + (y_off + s0) * esz, (s1 - s0) * esz, hc),
                           "rgb_memcpy_async")
                ev = torch.cuda.Event()
                ev.record(cs)
                stream.wait_event(ev)
                _lib.check(ingest(ctypes.byref(cfg), ctypes.byref(st), in_d + s0 * m * esz, 0,
                                  in_d + (y_off + s0) * esz, 0, s1 - s0, None, h), "rgb_ingest")
            _lib.check(cp(io_h, io_d, 16, h), "rgb_memcpy_async")
            _lib.check(cp(self._xh.data_ptr(), bs.x_t.data_ptr(), m * esz, h), "rgb_memcpy_async")  # live view
            stream.synchronize()
            done, status = self._take_counters(buf)
            self._on_status(status)
        else:
            buf["in_np"][:y_off] = A.reshape(-1)
            buf["in_np"][y_off:y_off + n] = y
            _lib.check(cp(in_d, in_h, (y_off + n) * esz, h), "rgb_memcpy_async")
        while done < n:
            T = n - done
            log_coords = bool(self._trackers)
            # per-row residuals only for update() reports: requesting them
            # routes the call to the generic kernel (the tensor-core kernels
            # do not log them); every log entry of a consumed row is written
            coords = torch.zeros((1, T, bs.r_cap), dtype=bs.dtype, device=bs.device) if log_coords else None
            logs = _lib.Logs(io_d + buf["off_branch"] if want_report else None,
                             coords.data_ptr() if log_coords else None,
                             io_d + buf["off_resid"] if want_report else None,
                             io_d + buf["off_gain"] if want_report else None)
            cfg, st = self._structs()
            _lib.check(ingest(ctypes.byref(cfg), ctypes.byref(st), in_d + done * m * esz, T * m,
                              in_d + (y_off + done) * esz, T, T, ctypes.byref(logs), h), "rgb_ingest")
            # counters (and the report): one asynchronous copy into pinned memory, one sync
            nb = buf["off_resid"] + T * esz if want_report else 16
            _lib.check(cp(io_h, io_d, nb, h), "rgb_memcpy_async")
            _lib.check(cp(self._xh.data_ptr(), bs.x_t.data_ptr(), m * esz, h), "rgb_memcpy_async")  # live view
            stream.synchronize()
            consumed, status = self._take_counters(buf)
            if log_coords and consumed:
                self._coords_chunks.append(coords[0, :consumed].cpu().numpy())
            if want_report:
                res = {"branch": buf["branch_np"][:consumed].copy(),
                       "resid": buf["resid_np"][:consumed].copy(),
                       "gain": buf["gain_np"].copy()}
            done += consumed
            self._on_status(status)
        return res

    def _row_pipe(self, want_report):
        """The librgb row pipe of this solver's current layout (include/rgb.h,
        rgb_rowpipe_*): the row goes to a row server -- a one-CTA persistent
        kernel that keeps the state in shared memory, reads the staged row from
        pinned, device-mapped host memory and writes the report and the counters
        back, so update() costs a request word and a spin on a sequence word; it
        exits after RGB_ROWSERVE_IDLE_US (default 500 us) without a row and is
        relaunched on demand (states beyond its shared memory: one graph launch
        per row).  Recreated when the state moves (capacity growth).  None (and
        pipes off) if creation fails."""
        bs = self._bs
        cfg, st = self._structs()
        key = (want_report, self._st_key)
        pipe = self._pipes.get(key)
        if pipe is not None:
            return pipe
        self._drop_pipes(keep=self._st_key)  # pipes of an older layout point at freed buffers
        lib = bs.lib
        h, blk = ctypes.c_void_p(), ctypes.c_void_p()
        # the device counters must be current before the pipe's first run
        self._torch.cuda.current_stream(bs.device).synchronize()
        if lib.rgb_rowpipe_create(ctypes.byref(cfg), ctypes.byref(st), int(want_report), int(self._f32in),
                                  ctypes.c_void_p(self._xh.data_ptr()), ctypes.byref(h), ctypes.byref(blk)) != _lib.OK:
            self._pipes = None
            return None
        off = [ctypes.c_int64() for _ in range(3)]
        nbytes = lib.rgb_rowpipe_layout(ctypes.byref(cfg), int(self._f32in), *[ctypes.byref(o) for o in off])
        raw = np.ctypeslib.as_array((ctypes.c_uint8 * nbytes).from_address(blk.value))
        sdt = np.dtype(np.float32 if bs.dtype == self._torch.float32 else np.float64)
        idt = np.dtype(np.float32) if (self._f32in or sdt == np.float32) else np.dtype(np.float64)
        o_in, o_res, o_gain = (o.value for o in off)
        m = self._m
        off_p = lib.rgb_rowpipe_proj_offset(ctypes.byref(cfg), int(self._f32in))
        rc_, esz = bs.r_cap, sdt.itemsize
        proj = (raw[off_p:off_p + esz * rc_].view(sdt), raw[off_p + esz * rc_:off_p + esz * (rc_ + m)].view(sdt),
                raw[off_p + esz * (rc_ + m):off_p + esz * (rc_ + m + 1)].view(sdt))
        pipe = {"h": h, "raw": raw, "proj": proj,
                # every drop-in call completes before it returns, so one stream
                # handle per pipe is safe
                "stream": ctypes.c_void_p(self._torch.cuda.current_stream(bs.device).cuda_stream),
                "in": raw[o_in:o_in + idt.itemsize * (m + 1)].view(idt),
                "resid": raw[o_res:o_res + sdt.itemsize].view(sdt),
                "gain": raw[o_gain:o_gain + sdt.itemsize * m].view(sdt),
                "hdr": {"nobs": raw[_lib.ROWPIPE_OFF_NOBS:_lib.ROWPIPE_OFF_NOBS + 8].view(np.int64),
                        "cnt": raw[_lib.ROWPIPE_OFF_RANK:_lib.ROWPIPE_OFF_STATUS + 4].view(np.int32),
                        "branch": raw[_lib.ROWPIPE_OFF_BRANCH:_lib.ROWPIPE_OFF_BRANCH + 1]}}
        self._pipes[key] = pipe
        hdr = pipe["hdr"]
        self._fast[want_report] = (self._st_key, pipe["in"], lib.rgb_rowpipe_run, h, pipe["stream"], hdr["nobs"],
                                   hdr["cnt"], hdr["branch"], pipe["resid"], pipe["gain"])
        return pipe

    def _quiesce(self):
        """Stop the row pipe's row server (include/rgb.h, rgb_rowpipe_quiesce),
        which keeps the state in its shared memory between update() calls,
        before another kernel writes the state."""
        if self._pipes:
            lib = self._bs.lib
            for pipe in self._pipes.values():
                _lib.check(lib.rgb_rowpipe_quiesce(pipe["h"]), "rgb_rowpipe_quiesce")

    def _drop_pipes(self, keep=None):
        """Destroy the row pipes (all, or those not of layout `keep`)."""
        if self._fast:
            for wr in [wr for wr, f in self._fast.items() if f[0] != keep]:
                del self._fast[wr]
        if self._pipes:
            lib = self._bs.lib
            for key in [key for key in self._pipes if key[1] != keep]:
                lib.rgb_rowpipe_destroy(self._pipes.pop(key)["h"])

    def __del__(self):
        try:
            self._drop_pipes()
        except Exception:  # noqa: BLE001  (interpreter shutdown)
            pass

    def _take_counters(self, buf):
        """Counters of the last report copy: records nobs and rank; returns
        (rows consumed since the previous read, status bits)."""
        nobs = int(buf["nobs_np"][0])
        rank, status = int(buf["cnt_np"][0]), int(buf["cnt_np"][1])
        consumed = nobs - self._host["nobs"]
        self._host["nobs"] = nobs
        self._host["rank"] = rank
        return consumed, status

    def _on_status(self, status):
        """A rank-cap stop doubles the capacity (the caller resumes); any other
        stop (invalid rescaling factor) raises."""
        bs = self._bs
        if status & _lib.ST_RANK_CAP:
            self._drop_pipes()  # the state moves
            bs.grow(2 * bs.r_cap)
            bs.status_t.zero_()
        elif status:
            bs.status_t.zero_()
            raise ValueError(f"device status {status}: non-finite input or invalid rescaling factor")


def solve_batch(matrix, targets, *, variant="general", eps=None, scalar=FLOAT64, alpha=1):
    """Fold all rows of a system through the solver; returns (x, rank) (solver.py:406-422)."""
    A = scalar.matrix(matrix)
    y = scalar.vector(targets)
    if A.shape[0] != y.shape[0]:
        raise ValueError(f"row count mismatch: matrix has {A.shape[0]} rows, targets {y.shape[0]}")
    solver = RecursiveSolver(A.shape[1], variant=variant, eps=eps, scalar=scalar, alpha=alpha)
    solver.ingest(A, y)
    return np.array(solver.solution, copy=True), solver.rank
