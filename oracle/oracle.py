"""CPU oracle for the rank-Greville update path -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline leg
(``cpu_baseline`` / ``--impl reference``) may import this module, and only as
the checker or the timed CPU reference -- never as the product path.  The
product (``paper_2106_11594_b200``) has no import of ``oracle`` and fails
loudly when its CUDA library is missing.

Two restatements of rankrls 0.1.0 (``/root/reference/pkg/src/rankrls``):

* ``ingest`` -- ctypes front end of ``rgb_oracle.c``, the C restatement of
  ``RecursiveSolver.ingest`` (solver.py:252-319) for B independent streams and
  k right-hand sides, with the per-row branch log, coords log (the rows of the
  coordinate factor B, tracking.py:59-74) and a-priori residuals.
* ``pinv_tracker`` -- numpy restatement of ``PseudoinverseTracker`` (the
  Theorem 2/3 column update, tracking.py:48-85) for small cases.

Pinning: ``tests/test_oracle.py`` checks both against golden vectors that
``tests/golden/make_golden.py`` produced by running the reference itself
(identical branch sequences and ranks; x and A+ within 1e-12 relative).
"""

from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = None

VARIANT_CODES = {"general": 0, "orthogonal": 1, "orthonormal": 2}
ST_RANK_CAP = 1


class _Cfg(ctypes.Structure):
    _fields_ = [
        ("m", ctypes.c_int32), ("k", ctypes.c_int32), ("r_cap", ctypes.c_int32),
        ("variant", ctypes.c_int32), ("eps_mode", ctypes.c_int32), ("pad", ctypes.c_int32),
        ("eps_value", ctypes.c_double), ("alpha", ctypes.c_double),
    ]


def build():
    """Compile liborc.so from rgb_oracle.c (gcc; no GPU needed)."""
    subprocess.run(["make", "-s", "-C", _HERE], check=True)


def lib():
    global _LIB
    if _LIB is None:
        path = os.path.join(_HERE, "liborc.so")
        src = os.path.join(_HERE, "rgb_oracle.c")
        if not os.path.exists(path) or os.path.getmtime(path) < os.path.getmtime(src):
            build()
        _LIB = ctypes.CDLL(path)
        _LIB.orc_ingest_batch.restype = ctypes.c_int
    return _LIB


def _ptr(a):
    return ctypes.c_void_p(0 if a is None else a.ctypes.data)


def new_state(B, m, k, r_cap, dtype=np.float64):
    return {
        "C": np.zeros((B, r_cap, m), dtype),
        "D": np.zeros((B, r_cap, m), dtype),
        "P": np.zeros((B, r_cap, r_cap), dtype),
        "X": np.zeros((B, k, m), dtype),
        "rank": np.zeros(B, np.int32),
        "nobs": np.zeros(B, np.int64),
        "status": np.zeros(B, np.int32),
    }


def ingest(rows, targets, *, variant="general", eps=None, alpha=1.0, r_cap=None,
           dtype=np.float64, state=None, logs=True, nthreads=1):
    """Fold rows[B, T, m] with targets[B, T, k] (or [B, T]) through B streams.

    ``eps`` None means the auto policy (solver.py:66-72), a float means the
    fixed policy.  ``r_cap`` bounds the stored rank (default min(T, m) plus the
    current rank); a stream whose rank would exceed it gets status bit 1 and
    stops, mirroring the CUDA library.  Returns the state dict plus logs.
    """
    rows = np.ascontiguousarray(rows, dtype=dtype)
    if rows.ndim == 2:
        rows = rows[None]
    B, T, m = rows.shape
    targets = np.asarray(targets, dtype=dtype)
    if targets.ndim == rows.ndim - 1:
        targets = targets[..., None]
    targets = np.ascontiguousarray(targets.reshape(B, T, -1))
    k = targets.shape[2]
    if state is None:
        if r_cap is None:
            r_cap = max(1, min(T, m))
        state = new_state(B, m, k, r_cap, dtype)
    r_cap = state["C"].shape[1]
    cfg = _Cfg(m, k, r_cap, VARIANT_CODES[variant], 0 if eps is None else 1, 0,
               0.0 if eps is None else float(eps), float(alpha))
    out = dict(state)
    out["branch"] = np.zeros((B, T), np.uint8) if logs else None
    out["coords"] = np.zeros((B, T, r_cap), dtype) if logs else None
    out["resid"] = np.zeros((B, T, k), dtype) if logs else None
    out["rho"] = np.zeros((B, T), np.float64) if logs else None
    lib().orc_ingest_batch(
        ctypes.byref(cfg), int(dtype == np.float32), ctypes.c_longlong(B),
        _ptr(state["C"]), _ptr(state["D"]), _ptr(state["P"]), _ptr(state["X"]),
        _ptr(state["rank"]), _ptr(state["nobs"]), _ptr(state["status"]),
        _ptr(rows), _ptr(targets), ctypes.c_longlong(T),
        _ptr(out["branch"]), _ptr(out["coords"]), _ptr(out["resid"]), _ptr(out["rho"]),
        int(nthreads))
    return out


def solution(out):
    """X as [B, m, k] (the state stores one column per RHS: [B, k, m])."""
    return np.swapaxes(out["X"], 1, 2)


def pinv_closed_form(out, b=0, variant="general"):
    """A+ = C~^T P^-1 B^T (test_tracking.py:87-98) from the
    final state and the coords log of stream b."""
    r = int(out["rank"][b])
    D = out["C"][b, :r] if variant == "orthonormal" else out["D"][b, :r]
    P = out["P"][b, :r, :r]
    Bf = out["coords"][b, :, :r]
    return D.T @ (P @ Bf.T)


def pinv_tracker(A, *, variant="general", eps=None, alpha=1.0):
    """numpy restatement of PseudoinverseTracker over a whole matrix
    (pinv_from_scratch, tracking.py:128-142).  Small cases only."""
    A = np.asarray(A, dtype=np.float64)
    n, m = A.shape
    eps_m = float(np.finfo(np.float64).eps)
    C = np.zeros((0, m)); D = np.zeros((0, m)); P = np.zeros((0, 0))
    pinv = np.zeros((m, 0)); Bf = np.zeros((0, 0))
    for row in A:
        r = C.shape[0]
        coords = D @ row if r else np.zeros(0)
        rej = row - coords @ C if r else row.copy()
        rej_sq = float(rej @ rej)
        e = float(eps) if eps is not None else (m * m * r + m * r + m) * eps_m
        dep = rej_sq < e * e or rej_sq < e * e * float(row @ row)
        if dep:
            if r:
                z = P @ coords
                denom = 1.0 + coords @ z
                gain = (z / denom) @ D
            else:
                z = np.zeros(0); denom = 1.0; gain = np.zeros(m)
            coords_row = coords
        else:
            gain = rej / rej_sq
            if r:
                z = P @ coords
                denom = 1.0 + coords @ z
            else:
                z = np.zeros(0); denom = 1.0
            coords_row = np.zeros(r + 1)
            if variant == "general":
                coords_row[r] = 1.0
            else:
                resc = 1.0 / np.sqrt(rej_sq) if variant == "orthonormal" else float(alpha)
                coords_row[:r] = coords
                coords_row[r] = 1.0 / resc
        # tracking.py:76-85 -- A+ <- [A+ - gain (B z)^T, gain]
        fitted = Bf @ z if Bf.shape[1] else np.zeros(pinv.shape[1])
        pinv = np.hstack([pinv - np.outer(gain, fitted), gain[:, None]])
        nb = Bf.shape[0]
        if dep:
            Bf = np.vstack([Bf, coords_row[None, :]]) if r else np.zeros((nb + 1, 0))
        else:
            Bn = np.zeros((nb + 1, r + 1)); Bn[:nb, :r] = Bf; Bn[nb] = coords_row; Bf = Bn
        # factor update (solver.py:242-246, 368-397)
        if dep:
            if r:
                P = P - np.outer(z, z / denom)
        else:
            G = np.zeros((r + 1, r + 1)); G[:r, :r] = P
            if variant == "general":
                C = np.vstack([C, row]); D = np.vstack([D - np.outer(coords, gain), gain])
                G[r, r] = 1.0
            else:
                a = 1.0 / coords_row[r]
                C = np.vstack([C, a * rej])
                D = C if variant == "orthonormal" else np.vstack([D, rej / (a * rej_sq)])
                if r:
                    G[:r, r] = -(a * z); G[r, :r] = -(a * z)
                G[r, r] = a * a * denom
            P = G
    return pinv
