"""The row server of the per-row drop-in API (include/rgb.h rgb_rowpipe_run /
rgb_rowpipe_quiesce, csrc/rgb_rowpipe.cu row1_serve_kernel).

RecursiveSolver.update (solver.py:231-250) goes to a persistent one-CTA kernel
that keeps the state in shared memory between calls.  It must give exactly the
bits of the one-launch-per-row path (RGB_ROWSERVE_IDLE_US=0, the graph replay
of row1_kernel, same arithmetic) through every transition: idle exits and
relaunches, one-row ingests through the same pipe, multi-row ingests (the
server is stopped first and restaged after), capacity growth (the pipe is
recreated), and reports / counters / the live solution view.
"""
import time

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _drive(m, idle_us, monkeypatch, seed=0, n=260):
    import paper_2106_11594_b200 as p

    monkeypatch.setenv("RGB_ROWSERVE_IDLE_US", str(idle_us))
    rng = np.random.default_rng(seed)
    A = rng.standard_normal((48, m))
    rows = rng.standard_normal((n, 20)) @ A[:20]
    rows[::13] = rng.standard_normal((len(rows[::13]), m))  # independent rows (m 128: past r_cap 32)
    ys = rng.standard_normal(n)
    s = p.RecursiveSolver(m)
    view = s.solution
    out = []
    for i in range(n):
        if i % 50 == 25:
            time.sleep(0.003)  # past the idle time: the server exits and is relaunched
        if i % 60 == 30:
            s.ingest(rows[i:i + 1], ys[i:i + 1])  # one row through the same pipe
            out.append(("ingest1", s.rank, s.num_observations))
            continue
        if i % 70 == 35:
            s.ingest(rows[i:i + 5], ys[i:i + 5])  # several rows: the server stops first
        r = s.update(rows[i], ys[i])
        out.append((r.branch, r.predicted_residual, r.new_rank, r.gain.copy(), s.num_observations))
    return s, view.copy(), out


@pytest.mark.parametrize("m", [16, 128, 1024])  # 1 024: the state stays in global memory
def test_row_server_bit_identical_to_graph_path(m, monkeypatch):
    s1, v1, o1 = _drive(m, 400, monkeypatch)
    s0, v0, o0 = _drive(m, 0, monkeypatch)
    assert s1.rank == s0.rank and s1.num_observations == s0.num_observations
    if m > 32:
        assert s1.rank > 32  # the capacity doubled on the way (pipe recreated)
    assert np.array_equal(v1, v0)  # the live view followed every call
    assert np.array_equal(v1, s1.solution)
    assert len(o1) == len(o0)
    for a, b in zip(o1, o0):
        assert a[0] == b[0]
        for x, y in zip(a[1:], b[1:]):
            assert np.array_equal(np.asarray(x), np.asarray(y))
    C1, D1, P1 = s1.basis()
    C0, D0, P0 = s0.basis()
    assert np.array_equal(C1, C0) and np.array_equal(D1, D0) and np.array_equal(P1, P0)


def test_row_server_state_visible_to_other_kernels(monkeypatch):
    """After update() calls the server keeps running; project() and a multi-row
    ingest on the caller's stream see the state it wrote."""
    import paper_2106_11594_b200 as p
    from oracle import oracle

    monkeypatch.setenv("RGB_ROWSERVE_IDLE_US", "100000")  # stays alive for the whole test
    rng = np.random.default_rng(3)
    m = 64
    A = rng.standard_normal((12, m)) @ rng.standard_normal((m, m))
    rows = rng.standard_normal((80, 12)) @ A
    ys = rng.standard_normal(80)
    s = p.RecursiveSolver(m)
    for i in range(40):
        s.update(rows[i], ys[i])
    pr = s.project(rows[41])  # read while the server is alive
    s.ingest(rows[40:80], ys[40:80])
    o = oracle.ingest(rows[None], ys[None, :, None], r_cap=s._bs.r_cap, nthreads=1)
    assert s.rank == int(o["rank"][0]) == 12
    x = oracle.solution(o)[0, :, 0]
    assert np.abs(s.solution - x).max() <= 1e-9 * max(1.0, np.abs(x).max())
    assert pr.coords.shape == (12,)


@pytest.mark.parametrize("m", [16, 128, 1024])
def test_project_through_row_server(m, monkeypatch):
    """project() (solver.py:210-219) goes to the row server when the solver has one:
    the same coords / rejection as the projection kernel (RGB_ROWSERVE_IDLE_US=0)
    to rounding, nothing written to the state, and is_dependent(project(a), a)
    (solver.py:221-229) predicts update(a)'s branch."""
    import paper_2106_11594_b200 as p

    rng = np.random.default_rng(11)
    A = rng.standard_normal((12, m))
    probe = np.vstack([rng.standard_normal((6, 12)) @ A, rng.standard_normal((6, m))])  # dependent, independent

    def run(idle):
        monkeypatch.setenv("RGB_ROWSERVE_IDLE_US", str(idle))
        s = p.RecursiveSolver(m)
        for i in range(12):
            s.update(A[i], float(i))
        x0 = s.solution.copy()
        projs = [s.project(a) for a in probe]
        assert np.array_equal(s.solution, x0) and s.num_observations == 12  # state untouched
        return s, projs

    s1, p1 = run(400)
    s0, p0 = run(0)
    for a, x, y in zip(probe, p1, p0):
        scale = max(1.0, float(np.abs(a).max()))
        assert x.coords.shape == y.coords.shape == (min(12, m),)
        assert np.abs(x.coords - y.coords).max() <= 1e-11 * max(1.0, np.abs(y.coords).max())
        assert np.abs(x.rejection - y.rejection).max() <= 1e-11 * scale
        assert abs(x.rejection_sq_norm - y.rejection_sq_norm) <= 1e-10 * scale * scale
    for a in probe:  # project, test, then fold: the test predicts the fold's branch
        dep = s1.is_dependent(s1.project(a), a)
        rep = s1.update(a, 0.0)
        assert (rep.branch == "dependent") == dep
