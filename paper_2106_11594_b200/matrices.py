"""The reference's matrix text format (rankrls.matrices, matrices.py:225-274),
shared by the CLI and file interfaces: line 1 "n m", then n lines of m
whitespace-separated scalars, each a decimal float or an exact "p/q".  Host
text handling only; the numbers go to the device through the solver."""

from __future__ import annotations

import io

from .scalars import FLOAT64


def format_matrix(matrix, kind=FLOAT64):
    arr = kind.matrix(matrix)
    lines = [f"{arr.shape[0]} {arr.shape[1]}"]
    lines.extend(" ".join(kind.render(v) for v in row) for row in arr)
    return "\n".join(lines) + "\n"


def parse_matrix(text, kind=FLOAT64):
    tokens = text.split()
    if len(tokens) < 2:
        raise ValueError("matrix text must start with 'n m'")
    try:
        n, m = int(tokens[0]), int(tokens[1])
    except ValueError as err:
        raise ValueError(f"bad matrix header {tokens[:2]!r}") from err
    if n < 0 or m < 0:
        raise ValueError(f"bad matrix dimensions {n} x {m}")
    values = tokens[2:]
    if len(values) != n * m:
        raise ValueError(f"expected {n * m} entries for a {n} x {m} matrix, got {len(values)}")
    out = kind.zeros((n, m))
    for idx, tok in enumerate(values):
        out[idx // m, idx % m] = kind.parse(tok)
    return out


def write_matrix(path, matrix, kind=FLOAT64):
    data = format_matrix(matrix, kind)
    if isinstance(path, io.TextIOBase):
        path.write(data)
    else:
        with open(path, "w", encoding="ascii") as handle:
            handle.write(data)


def read_matrix(path, kind=FLOAT64):
    if isinstance(path, io.TextIOBase):
        return parse_matrix(path.read(), kind)
    with open(path, "r", encoding="ascii") as handle:
        return parse_matrix(handle.read(), kind)


def read_vector(path, kind=FLOAT64):
    """An n x 1 or 1 x n matrix file as a flat vector."""
    out = read_matrix(path, kind)
    if 1 in out.shape or 0 in out.shape:
        return out.reshape(-1)
    raise ValueError(f"expected a vector-shaped file, got {out.shape}")
