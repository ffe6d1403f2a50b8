"""Batched device API: many independent rank-Greville streams on one GPU.

``BatchedSolver`` owns the device state of B independent solvers of m
regressors, each with k right-hand sides, in the layout of include/rgb.h, and
folds row blocks into all of them with one ``rgb_ingest`` launch.  It is the
batched generalisation of ``RecursiveSolver`` (solver.py:120-397): the
reference's single-writer / independent-instances model is what
makes the streams a data-parallel batch.

torch is used for device memory and streams only; all arithmetic runs in
librgb.so.
"""

from __future__ import annotations

import ctypes

import torch

from . import _lib

_DTYPES = {torch.float64: _lib.F64, torch.float32: _lib.F32}
_VARIANTS = {"general": _lib.GENERAL, "orthogonal": _lib.ORTHOGONAL, "orthonormal": _lib.ORTHONORMAL}


def _ptr(t):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def _stream_handle(device):
    return ctypes.c_void_p(torch.cuda.current_stream(device).cuda_stream)


class BatchedSolver:
    """B independent streams x k right-hand sides on one CUDA device.

    Parameters mirror ``RecursiveSolver`` (solver.py:140-141) plus the batch
    extensions: ``num_streams``, ``k`` (right-hand sides), ``r_cap`` (stored
    rank capacity) and ``dtype`` (torch.float64, or torch.float32 -- a kind
    the reference does not have).  ``eps`` is None (auto policy) or a float
    (fixed policy); ``alpha`` is the orthogonal rescaling constant.
    """

    def __init__(self, num_streams, num_regressors, *, k=1, r_cap=None, variant="general",
                 eps=None, alpha=1.0, dtype=torch.float64, device=None):
        if not torch.cuda.is_available():
            raise _lib.RgbError("no CUDA device: the rank-Greville path is GPU-only")
        if variant not in _VARIANTS:
            raise ValueError(f"unknown variant {variant!r}; expected one of {tuple(_VARIANTS)}")
        if dtype not in _DTYPES:
            raise ValueError(f"dtype must be torch.float64 or torch.float32, got {dtype}")
        if not isinstance(num_regressors, int) or num_regressors < 1:
            raise ValueError(f"num_regressors must be a positive integer, got {num_regressors!r}")
        if eps is not None and not eps >= 0:
            raise ValueError("fixed eps requires a nonnegative value")
        self.lib = _lib.load()
        self.device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        self.B, self.m, self.k = int(num_streams), int(num_regressors), int(k)
        self.r_cap = int(r_cap) if r_cap is not None else self.m
        self.variant, self.eps, self.alpha, self.dtype = variant, eps, float(alpha), dtype
        self._alloc(self.r_cap)
        self.reset()

    # -- state ------------------------------------------------------------
    def _alloc(self, r_cap):
        kw = dict(dtype=self.dtype, device=self.device)
        B, m, k = self.B, self.m, self.k
        self.basis_t = torch.zeros((B, r_cap, m), **kw)
        self.dual_t = self.basis_t if self.variant == "orthonormal" else torch.zeros((B, r_cap, m), **kw)
        self.gram_t = torch.zeros((B, r_cap, r_cap), **kw)
        if not hasattr(self, "x_t"):
            self.x_t = torch.zeros((B, k, m), **kw)
            self.rank_t = torch.zeros(B, dtype=torch.int32, device=self.device)
            self.nobs_t = torch.zeros(B, dtype=torch.int64, device=self.device)
            self.status_t = torch.zeros(B, dtype=torch.int32, device=self.device)
        self.r_cap = r_cap

    def config(self, num_streams=None):
        return _lib.Config(
            self.B if num_streams is None else num_streams, self.m, self.k, self.r_cap,
            _DTYPES[self.dtype], _VARIANTS[self.variant],
            _lib.EPS_AUTO if self.eps is None else _lib.EPS_FIXED,
            0.0 if self.eps is None else float(self.eps), self.alpha)

    def state(self, b=0):
        """rgb_state pointing at stream b onwards (b > 0 for sub-batches)."""
        def at(t):
            return ctypes.c_void_p(t.data_ptr() + b * t.stride(0) * t.element_size())
        return _lib.State(at(self.basis_t), at(self.dual_t), at(self.gram_t), at(self.x_t),
                          at(self.rank_t), at(self.nobs_t), at(self.status_t))

    def reset(self):
        """Empty every stream (RecursiveSolver.__init__, solver.py:160-171)."""
        cfg, st = self.config(), self.state()
        _lib.check(self.lib.rgb_state_reset(ctypes.byref(cfg), ctypes.byref(st), _stream_handle(self.device)),
                   "rgb_state_reset")

    def grow(self, new_cap):
        """Raise the stored-rank capacity, keeping every factor."""
        if new_cap <= self.r_cap:
            return
        old = (self.basis_t, self.dual_t, self.gram_t, self.r_cap)
        self._alloc(new_cap)
        rc = old[3]
        self.basis_t[:, :rc].copy_(old[0])
        if self.variant != "orthonormal":
            self.dual_t[:, :rc].copy_(old[1])
        self.gram_t[:, :rc, :rc].copy_(old[2])

    # -- the hot path -------------------------------------------------------
    def ingest(self, rows, targets, *, branch_log=None, coords_log=None, resid_log=None,
               gain_out=None, stream=None):
        """Fold rows[B, T, m] / targets[B, T, k] (device tensors of this dtype).

        A float64 solver also accepts float32 rows and targets: they are
        widened exactly on load inside the kernel (rgb_ingest_f32in), so the
        result equals ingesting rows.double() while reading half the bytes.

        Optional logs (preallocated device tensors): branch_log uint8 [B, T],
        coords_log [B, T, r_cap], resid_log [B, T, k], gain_out [B, m].
        Asynchronous on the current (or given) CUDA stream.
        """
        B, T, m = rows.shape
        if B != self.B or m != self.m:
            raise ValueError(f"rows have shape {tuple(rows.shape)}, expected ({self.B}, T, {self.m})")
        if targets.dim() == 2:
            targets = targets.unsqueeze(-1)
        if tuple(targets.shape) != (B, T, self.k):
            raise ValueError(f"targets have shape {tuple(targets.shape)}, expected ({B}, {T}, {self.k})")
        f32in = self._f32_inputs(rows, targets)
        for t in (rows, targets):
            if t.device != self.device:
                raise ValueError("rows/targets must be device tensors of the solver dtype")
            if (t.shape[2] > 1 and t.stride(2) != 1) or (t.shape[1] > 1 and t.stride(1) != t.shape[2]):
                raise ValueError("rows/targets must be contiguous within each stream")
        logs = _lib.Logs(_ptr(branch_log), _ptr(coords_log), _ptr(resid_log), _ptr(gain_out))
        cfg, st = self.config(), self.state()
        h = ctypes.c_void_p(stream.cuda_stream) if stream is not None else _stream_handle(self.device)
        fn = self.lib.rgb_ingest_f32in if f32in else self.lib.rgb_ingest
        _lib.check(fn(ctypes.byref(cfg), ctypes.byref(st), _ptr(rows), rows.stride(0),
                      _ptr(targets), targets.stride(0), T, ctypes.byref(logs), h), "rgb_ingest")

    def _f32_inputs(self, rows, targets):
        """True for float32 inputs into a float64 state; raises on any other mismatch."""
        if rows.dtype != targets.dtype:
            raise ValueError("rows and targets must have the same dtype")
        if rows.dtype == self.dtype:
            return False
        if self.dtype == torch.float64 and rows.dtype == torch.float32:
            return True
        raise ValueError(f"rows/targets must be {self.dtype} (or float32 into a float64 solver), got {rows.dtype}")

    def ingest_host(self, rows_h, targets_h, *, chunk=4096):
        """Fold rows/targets that live in (pinned) HOST memory.

        Streams are copied host-to-device in chunks of ``chunk`` streams on a
        side CUDA stream, double-buffered so that the copy of chunk i+1
        overlaps the ingest of chunk i on the current stream.  Returns the
        number of ingest launches issued.
        """
        B, T, m = rows_h.shape
        if targets_h.dim() == 2:
            targets_h = targets_h.unsqueeze(-1)
        if B != self.B or m != self.m or tuple(targets_h.shape) != (B, T, self.k):
            raise ValueError("host rows/targets do not match the solver shape")
        f32in = self._f32_inputs(rows_h, targets_h)
        in_dtype = rows_h.dtype
        fn = self.lib.rgb_ingest_f32in if f32in else self.lib.rgb_ingest
        chunk = max(1, min(chunk, B))
        dev = self.device
        compute = torch.cuda.current_stream(dev)
        copy = torch.cuda.Stream(dev)
        bufs = [(torch.empty((chunk, T, m), dtype=in_dtype, device=dev),
                 torch.empty((chunk, T, self.k), dtype=in_dtype, device=dev)) for _ in range(2)]
        ready = [torch.cuda.Event() for _ in range(2)]
        free = [torch.cuda.Event() for _ in range(2)]
        for e in free:
            e.record(compute)
        launches = 0
        for i, s0 in enumerate(range(0, B, chunk)):
            s1 = min(B, s0 + chunk)
            n = s1 - s0
            rb, tb = bufs[i % 2]
            copy.wait_event(free[i % 2])
            with torch.cuda.stream(copy):
                rb[:n].copy_(rows_h[s0:s1], non_blocking=True)
                tb[:n].copy_(targets_h[s0:s1], non_blocking=True)
                ready[i % 2].record(copy)
            compute.wait_event(ready[i % 2])
            cfg, st = self.config(num_streams=n), self.state(s0)
            logs = _lib.Logs(None, None, None, None)
            _lib.check(fn(ctypes.byref(cfg), ctypes.byref(st), _ptr(rb), rb.stride(0), _ptr(tb), tb.stride(0), T,
                          ctypes.byref(logs), ctypes.c_void_p(compute.cuda_stream)), "rgb_ingest")
            free[i % 2].record(compute)
            launches += 1
        return launches

    def project(self, rows):
        """coords [B, r_cap], rejection [B, m], rej_sq [B], dependent [B] for one row per stream."""
        rows = rows.contiguous()
        kw = dict(dtype=self.dtype, device=self.device)
        coords = torch.empty((self.B, self.r_cap), **kw)
        rej = torch.empty((self.B, self.m), **kw)
        rsq = torch.empty(self.B, **kw)
        dep = torch.empty(self.B, dtype=torch.uint8, device=self.device)
        cfg, st = self.config(), self.state()
        _lib.check(self.lib.rgb_project(ctypes.byref(cfg), ctypes.byref(st), _ptr(rows), _ptr(coords),
                                        _ptr(rej), _ptr(rsq), _ptr(dep), _stream_handle(self.device)),
                   "rgb_project")
        return coords, rej, rsq, dep

    def pinv(self, coords_log):
        """A+ [B, m, n] from the coordinate-factor log [B, n, r_cap]."""
        n = coords_log.shape[1]
        out = torch.empty((self.B, self.m, n), dtype=self.dtype, device=self.device)
        cfg, st = self.config(), self.state()
        _lib.check(self.lib.rgb_pinv(ctypes.byref(cfg), ctypes.byref(st), _ptr(coords_log.contiguous()), n,
                                     _ptr(out), _stream_handle(self.device)), "rgb_pinv")
        return out

    def covariance(self):
        """V = A+ A+^T [B, m, m]."""
        out = torch.empty((self.B, self.m, self.m), dtype=self.dtype, device=self.device)
        cfg, st = self.config(), self.state()
        _lib.check(self.lib.rgb_covariance(ctypes.byref(cfg), ctypes.byref(st), _ptr(out),
                                           _stream_handle(self.device)), "rgb_covariance")
        return out

    # -- read access ----------------------------------------------------------
    @property
    def solution(self):
        """X as [B, m, k] (a view of the device state)."""
        return self.x_t.transpose(1, 2)

    @property
    def rank(self):
        return self.rank_t

    @property
    def num_observations(self):
        return self.nobs_t

    @property
    def status(self):
        return self.status_t
