"""The float32-state path of config 5 (csrc/rgb_f32.cu: one warp per stream on
the fp32 CUDA cores) -- a kind the reference does not have (scalars.py:141-157).

Parity policy (SURVEY.md section 7 hard part 1, option
(c)): pure fp32 arithmetic with the auto eps policy at eps_32 = 2^-23.  Ranks
and branch sequences are compared with the C oracle's fp32 mode on the same
float32 bytes (a first disagreement only on a noise-band row); x is compared
with the fp64 oracle within 1e-3 on every stream whose fp32 and fp64 ranks
agree, and with the fp32 oracle within 1e-3."""

import os

import numpy as np
import pytest

from oracle import oracle
from paper_2106_11594_b200 import workloads
from rgb_testutil import compare_branches, relerr

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

TOL32 = 1e-3


def run32(rows, tg, r_cap=16, splits=None, coords=False):
    from paper_2106_11594_b200.batched import BatchedSolver

    B, T, m = rows.shape
    bs = BatchedSolver(B, m, k=tg.shape[2], r_cap=r_cap, dtype=torch.float32)
    rd = torch.as_tensor(np.ascontiguousarray(rows), dtype=torch.float32, device="cuda")
    td = torch.as_tensor(np.ascontiguousarray(tg), dtype=torch.float32, device="cuda")
    brs, cls = [], []
    lo = 0
    for hi in (splits or []) + [T]:
        if hi > lo:  # per-call logs are [B, rows of the call] (contiguous)
            brs.append(torch.zeros((B, hi - lo), dtype=torch.uint8, device="cuda"))
            cls.append(torch.zeros((B, hi - lo, r_cap), dtype=torch.float32, device="cuda") if coords else None)
            bs.ingest(rd[:, lo:hi].contiguous(), td[:, lo:hi].contiguous(), branch_log=brs[-1], coords_log=cls[-1])
        lo = hi
    torch.cuda.synchronize()
    br = torch.cat(brs, dim=1)
    cl = torch.cat(cls, dim=1) if coords else None
    out = {"branch": br.cpu().numpy(), "rank": bs.rank.cpu().numpy(), "nobs": bs.nobs_t.cpu().numpy(),
           "status": bs.status.cpu().numpy(), "x": bs.solution.cpu().numpy().astype(np.float64), "solver": bs}
    if coords:
        out["coords"] = cl
    return out


def check_fp32(rows64, tg64, res, r_cap=16):
    r32, t32 = rows64.astype(np.float32), tg64.astype(np.float32)
    o32 = oracle.ingest(r32, t32, r_cap=r_cap, dtype=np.float32, nthreads=16)
    o64 = oracle.ingest(rows64, tg64, r_cap=r_cap, nthreads=16)
    cmp = compare_branches(res["branch"], res["nobs"], o32["branch"], o32["rho"])
    assert cmp["outside_disagree"] == 0, cmp["disagreements"]
    X32, X64 = oracle.solution(o32).astype(np.float64), oracle.solution(o64)
    B = rows64.shape[0]
    same = [b for b in range(B) if res["status"][b] == 0 and o32["status"][b] == 0
            and np.array_equal(res["branch"][b], o32["branch"][b])]
    for b in same:
        assert res["rank"][b] == o32["rank"][b]
        assert relerr(res["x"][b], X32[b]) <= TOL32, b
    agree64 = [b for b in same if o64["status"][b] == 0 and o64["rank"][b] == res["rank"][b]]
    for b in agree64:
        assert relerr(res["x"][b], X64[b]) <= TOL32, b
    return cmp, same, agree64


def test_c5_fp32_gaussian_and_integer_streams():
    rows, tg = workloads.host_batch("c5", list(range(128)))
    res = run32(rows, tg)
    cmp, same, agree64 = check_fp32(rows, tg, res)
    assert len(same) >= 124 and len(agree64) >= 120
    # the integer half (exact rank detection) matches the fp64 rank everywhere
    assert all(res["rank"][b] == 16 for b in range(1, 128, 2) if res["status"][b] == 0)


@pytest.mark.parametrize("k", [1, 3, 8])
def test_c5_fp32_continuation_calls_and_fewer_rhs(k):
    rows, tg = workloads.host_batch("c5", list(range(24)), n=301)
    tg = np.ascontiguousarray(tg[..., :k])
    one = run32(rows, tg)
    split = run32(rows, tg, splits=[5, 40, 133, 300])
    assert np.array_equal(one["rank"], split["rank"])
    ok = [b for b in range(24) if np.array_equal(one["branch"][b], split["branch"][b])]
    assert len(ok) >= 22
    for b in ok:
        assert relerr(split["x"][b], one["x"][b]) <= TOL32  # fp32: x0 is re-rounded at each call boundary
    check_fp32(rows, tg, split)


def test_c5_fp32_kernel_agrees_with_generic_fp32_kernel(monkeypatch):
    rows, tg = workloads.host_batch("c5", list(range(32)), n=400)
    a = run32(rows, tg)
    monkeypatch.setenv("RGB_NO_F32K", "1")
    b = run32(rows, tg)
    assert np.array_equal(a["rank"], b["rank"])
    same = [s for s in range(32) if np.array_equal(a["branch"][s], b["branch"][s])]
    assert len(same) >= 30
    for s in same:
        assert relerr(a["x"][s], b["x"][s]) <= TOL32


def test_c5_fp32_nonfinite_rank_cap_and_partial_tiles():
    rows, tg = workloads.host_batch("c5", list(range(6)), n=37)
    rows = rows.copy()
    rows[1, 20, 3] = np.nan                      # frozen at row 20
    rows[2, 10:30] = np.random.default_rng(3).standard_normal((20, 64))  # rank past the capacity
    res = run32(rows, tg)
    assert res["status"][1] == 2 and res["nobs"][1] == 20
    assert res["status"][2] == 1 and res["rank"][2] == 16
    ok = [0, 3, 4, 5]
    for b in ok:
        assert res["status"][b] == 0 and res["nobs"][b] == 37
    o32 = oracle.ingest(rows[ok].astype(np.float32), tg[ok].astype(np.float32), r_cap=16, dtype=np.float32)
    assert np.array_equal(res["rank"][ok], o32["rank"])


def test_c5_fp32_coords_log_and_pinv():
    rows, tg = workloads.host_batch("c5", [0, 1, 2, 3], n=96)
    res = run32(rows, tg, coords=True)
    pinv = res["solver"].pinv(res["coords"]).cpu().numpy().astype(np.float64)
    for b in range(4):
        ref = np.linalg.pinv(rows[b], rcond=1e-10)
        assert relerr(pinv[b], ref) <= 1e-3


def test_fp32_state_dispatches_to_the_fp32_kernel():
    """The tuned kernel is the one that runs (not the generic fallback): its
    results differ in the last bits from the generic kernel's."""
    rows, tg = workloads.host_batch("c5", [0, 2], n=64)
    a = run32(rows, tg)
    os.environ["RGB_NO_F32K"] = "1"
    try:
        b = run32(rows, tg)
    finally:
        del os.environ["RGB_NO_F32K"]
    assert not np.array_equal(a["x"], b["x"])
