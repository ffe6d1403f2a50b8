"""ctypes binding of librgb.so (include/rgb.h).

The library is built in-tree by ``__graft_entry__.build()`` /
``python -m paper_2106_11594_b200._build``.  There is no CPU fallback: when the
library or a CUDA device is missing, every entry point raises.
"""

from __future__ import annotations

import ctypes
import os

HERE = os.path.dirname(os.path.abspath(__file__))
# RGB_LIB_PATH selects an alternative build of the same library (tuning A/B runs)
LIB_PATH = os.environ.get("RGB_LIB_PATH") or os.path.join(HERE, "librgb.so")

RGB_ABI_VERSION = 4
F64, F32 = 0, 1
GENERAL, ORTHOGONAL, ORTHONORMAL = 0, 1, 2
EPS_AUTO, EPS_FIXED = 0, 1
OK, E_INVALID, E_UNSUPPORTED, E_CUDA = 0, -1, -2, -3
ST_RANK_CAP, ST_NONFINITE, ST_BAD_ALPHA = 1, 2, 4

EXPORTS = ("rgb_abi_version", "rgb_last_error", "rgb_state_reset", "rgb_ingest", "rgb_ingest_f32in",
           "rgb_memcpy_async",
           "rgb_project", "rgb_pinv", "rgb_covariance",
           "rgb_rowpipe_layout", "rgb_rowpipe_create", "rgb_rowpipe_run", "rgb_rowpipe_quiesce",
           "rgb_rowpipe_destroy", "rgb_rowpipe_project", "rgb_rowpipe_proj_offset")
# row pipe host-block header (include/rgb.h)
ROWPIPE_HEADER, ROWPIPE_OFF_SEQ, ROWPIPE_OFF_NOBS, ROWPIPE_OFF_RANK = 64, 0, 8, 16
ROWPIPE_OFF_STATUS, ROWPIPE_OFF_BRANCH, ROWPIPE_OFF_REQ, ROWPIPE_OFF_STOP = 20, 24, 32, 40
ROWPIPE_OFF_PREQ, ROWPIPE_OFF_PSEQ = 48, 56


class Config(ctypes.Structure):
    _fields_ = [
        ("num_streams", ctypes.c_int64),
        ("m", ctypes.c_int32),
        ("k", ctypes.c_int32),
        ("r_cap", ctypes.c_int32),
        ("dtype", ctypes.c_int32),
        ("variant", ctypes.c_int32),
        ("eps_mode", ctypes.c_int32),
        ("eps_value", ctypes.c_double),
        ("alpha", ctypes.c_double),
    ]


class State(ctypes.Structure):
    _fields_ = [
        ("basis", ctypes.c_void_p),
        ("dual", ctypes.c_void_p),
        ("gram_inv", ctypes.c_void_p),
        ("x", ctypes.c_void_p),
        ("rank", ctypes.c_void_p),
        ("nobs", ctypes.c_void_p),
        ("status", ctypes.c_void_p),
    ]


class Logs(ctypes.Structure):
    _fields_ = [
        ("branch", ctypes.c_void_p),
        ("coords", ctypes.c_void_p),
        ("resid", ctypes.c_void_p),
        ("gain", ctypes.c_void_p),
    ]


class RgbError(RuntimeError):
    """A librgb.so call failed (RGB_E_UNSUPPORTED / RGB_E_CUDA)."""


_LIB = None


def load():
    """Load librgb.so (raises if it was not built)."""
    global _LIB
    if _LIB is not None:
        return _LIB
    if not os.path.exists(LIB_PATH):
        raise RgbError(
            f"{LIB_PATH} is missing: build it with `python -m paper_2106_11594_b200._build` "
            "(there is no CPU fallback for the rank-Greville path)")
    lib = ctypes.CDLL(LIB_PATH)
    vp, i64 = ctypes.c_void_p, ctypes.c_int64
    cfgp, stp, lgp = ctypes.POINTER(Config), ctypes.POINTER(State), ctypes.POINTER(Logs)
    lib.rgb_abi_version.restype = ctypes.c_int
    lib.rgb_last_error.restype = ctypes.c_char_p
    lib.rgb_state_reset.argtypes = [cfgp, stp, vp]
    lib.rgb_ingest.argtypes = [cfgp, stp, vp, i64, vp, i64, i64, lgp, vp]
    lib.rgb_ingest_f32in.argtypes = [cfgp, stp, vp, i64, vp, i64, i64, lgp, vp]
    lib.rgb_project.argtypes = [cfgp, stp, vp, vp, vp, vp, vp, vp]
    lib.rgb_pinv.argtypes = [cfgp, stp, vp, i64, vp, vp]
    lib.rgb_covariance.argtypes = [cfgp, stp, vp, vp]
    lib.rgb_memcpy_async.argtypes = [vp, vp, i64, vp]
    i64p = ctypes.POINTER(ctypes.c_int64)
    lib.rgb_rowpipe_layout.argtypes = [cfgp, ctypes.c_int, i64p, i64p, i64p]
    lib.rgb_rowpipe_create.argtypes = [cfgp, stp, ctypes.c_int, ctypes.c_int, vp, ctypes.POINTER(vp),
                                       ctypes.POINTER(vp)]
    lib.rgb_rowpipe_run.argtypes = [vp, vp]
    lib.rgb_rowpipe_quiesce.argtypes = [vp]
    lib.rgb_rowpipe_project.argtypes = [vp, vp]
    lib.rgb_rowpipe_proj_offset.argtypes = [cfgp, ctypes.c_int]
    lib.rgb_rowpipe_destroy.argtypes = [vp]
    for name in EXPORTS[2:]:
        getattr(lib, name).restype = ctypes.c_int
    lib.rgb_rowpipe_layout.restype = ctypes.c_int64
    lib.rgb_rowpipe_proj_offset.restype = ctypes.c_int64
    lib.rgb_rowpipe_destroy.restype = None
    if lib.rgb_abi_version() != RGB_ABI_VERSION:
        raise RgbError(f"librgb.so ABI {lib.rgb_abi_version()} != {RGB_ABI_VERSION}")
    _LIB = lib
    return lib


def check(rc, what):
    """Map a return code to the reference's exception types (solver.py:142-158)."""
    if rc == OK:
        return
    msg = load().rgb_last_error().decode(errors="replace")
    if rc == E_INVALID:
        raise ValueError(f"{what}: {msg}")
    raise RgbError(f"{what} failed ({rc}): {msg}")
