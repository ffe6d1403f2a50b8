"""The CLI `solve` front end and the matrix text format (the reference's
cli.py:93-134 and matrices.py:225-274), with the reference's own CLI cases
(test_cli.py:17-62).  Parsing, formatting and the exit-2 paths that fail
before the solve run on CPU; the solves are `-m gpu`."""

import numpy as np
import pytest

from paper_2106_11594_b200 import FLOAT64, RATIONAL, matrices
from paper_2106_11594_b200.cli import main


def write(path, text):
    path.write_text(text)
    return str(path)


def test_text_format_round_trip(tmp_path):
    A = np.array([[1.0, -0.6, 1e-300], [0.1, 2.0 / 3.0, -7.25]])
    p = tmp_path / "a.txt"
    matrices.write_matrix(p, A)
    assert p.read_text().splitlines()[0] == "2 3"
    assert np.array_equal(matrices.read_matrix(p), A)  # shortest round-trip decimals
    assert matrices.parse_matrix("1 2\n1/2 -3/4\n").tolist() == [[0.5, -0.75]]
    R = matrices.parse_matrix("1 2\n1/3 2\n", RATIONAL)
    assert matrices.format_matrix(R, RATIONAL) == "1 2\n1/3 2\n"
    assert matrices.format_matrix(np.eye(2)) == "2 2\n1.0 0.0\n0.0 1.0\n"


@pytest.mark.parametrize("text", ["", "2", "2 x\n1 2\n", "-1 2\n", "2 2\n1 0\n0\n", "1 1\nnan\n"])
def test_text_format_errors(text):
    with pytest.raises(ValueError):
        matrices.parse_matrix(text, FLOAT64)


def test_read_vector_shapes(tmp_path):
    assert matrices.read_vector(write(tmp_path / "c.txt", "2 1\n3\n4\n")).tolist() == [3.0, 4.0]
    assert matrices.read_vector(write(tmp_path / "r.txt", "1 2\n3 4\n")).tolist() == [3.0, 4.0]
    with pytest.raises(ValueError):
        matrices.read_vector(write(tmp_path / "m.txt", "2 2\n1 2\n3 4\n"))


def test_solve_dimension_mismatch_exits_2(tmp_path, capsys):
    mat = write(tmp_path / "a.txt", "2 2\n1 0\n0 1\n")
    rhs = write(tmp_path / "y.txt", "3 1\n1\n2\n3\n")
    assert main(["solve", mat, rhs]) == 2
    assert "rows" in capsys.readouterr().err


def test_solve_parse_failure_exits_2(tmp_path, capsys):
    mat = write(tmp_path / "a.txt", "2 2\n1 0\n0\n")
    rhs = write(tmp_path / "y.txt", "2 1\n1\n2\n")
    assert main(["solve", mat, rhs]) == 2
    assert "rankrls solve" in capsys.readouterr().err


def test_solve_missing_file_exits_2(tmp_path):
    assert main(["solve", str(tmp_path / "none.txt"), str(tmp_path / "y.txt")]) == 2


def test_bad_eps_is_a_usage_error(tmp_path):
    with pytest.raises(SystemExit) as e:
        main(["solve", "a", "b", "--eps", "loose"])
    assert e.value.code == 2


# -- solves on the device ---------------------------------------------------------------

@pytest.mark.gpu
def test_solve_identity(tmp_path, capsys):
    """test_cli.py:17-23"""
    mat = write(tmp_path / "a.txt", "2 2\n1 0\n0 1\n")
    rhs = write(tmp_path / "y.txt", "2 1\n3\n4\n")
    assert main(["solve", mat, rhs]) == 0
    out = capsys.readouterr().out.splitlines()
    assert out[0] == "3.0 4.0"
    assert out[1] == "rank 2"


@pytest.mark.gpu
def test_solve_writes_pinv_and_cov(tmp_path):
    """test_cli.py:51-60"""
    mat = write(tmp_path / "a.txt", "2 2\n1 0\n0 1\n")
    rhs = write(tmp_path / "y.txt", "2 1\n3\n4\n")
    pinv_path, cov_path = tmp_path / "pinv.txt", tmp_path / "cov.txt"
    assert main(["solve", mat, rhs, "--pinv", str(pinv_path), "--cov", str(cov_path)]) == 0
    assert np.allclose(matrices.read_matrix(pinv_path), np.eye(2))
    assert np.allclose(matrices.read_matrix(cov_path), np.eye(2))


@pytest.mark.gpu
@pytest.mark.parametrize("variant", ["general", "orthogonal", "orthonormal"])
def test_solve_file_round_trip_against_oracle(tmp_path, capsys, variant):
    """A rank-deficient system written in the text format, solved by the CLI:
    x (printed and --out) equals the oracle's, the rank is the construction
    rank, and --pinv matches the closed form."""
    from oracle import oracle
    from rgb_testutil import conditioned_stream, relerr

    rng = np.random.default_rng(9)
    A = conditioned_stream(rng, 40, 12, 5)
    y = rng.standard_normal(40)
    mat, rhs = tmp_path / "a.txt", tmp_path / "y.txt"
    matrices.write_matrix(mat, A)
    matrices.write_matrix(rhs, y[:, None])
    out, pinv = tmp_path / "x.txt", tmp_path / "p.txt"
    assert main(["solve", str(mat), str(rhs), "--variant", variant, "--out", str(out), "--pinv", str(pinv)]) == 0
    lines = capsys.readouterr().out.splitlines()
    assert lines[1] == "rank 5"
    x_printed = np.array([float(v) for v in lines[0].split()])
    x_file = matrices.read_vector(out)
    assert np.array_equal(x_printed, x_file)
    o = oracle.ingest(A[None], y[None], r_cap=12, variant=variant)
    assert relerr(x_file, oracle.solution(o)[0, :, 0]) <= 1e-9
    assert relerr(matrices.read_matrix(pinv), oracle.pinv_closed_form(o, variant=variant)) <= 1e-9


@pytest.mark.gpu
def test_solve_rational_is_cpu_only(tmp_path, capsys):
    """The exact-rational kind parses but does not solve on the device
    (CapabilityError, exit 2) -- DESIGN.md section 7."""
    mat = write(tmp_path / "a.txt", "2 2\n1 0\n0 1/2\n")
    rhs = write(tmp_path / "y.txt", "2 1\n1\n1\n")
    assert main(["solve", mat, rhs, "--scalar", "rational"]) == 2
    assert "rational" in capsys.readouterr().err.lower()
