"""Command-line front end: ``solve`` a least-squares system from matrix / rhs
files in the reference's text format (rankrls.cli, cli.py:93-134), with the
solve on the GPU through the drop-in API.

    python -m paper_2106_11594_b200.cli solve MATRIX RHS [--variant V] [--eps E]
        [--scalar f64|f32] [--out X] [--pinv FILE] [--cov FILE]

Prints x (shortest round-trip decimals, space separated) and "rank r"; exit
code 0 on success, 2 for usage, parse or dimension errors -- as the
reference.  The reference's other subcommands (gen / bench / stability) and
the exact-rational kind are not part of this drop-in:
``--scalar rational`` parses but the solve raises CapabilityError (exit 2).
"""

from __future__ import annotations

import argparse
import sys

import numpy as np

from . import matrices
from .scalars import KINDS
from .solver import VARIANTS, EpsPolicy, RecursiveSolver, solve_batch
from .tracking import CovarianceTracker, PseudoinverseTracker


def _parse_eps(text):
    """--eps: a float, 'auto' or 'exact' (cli.py:28-38)."""
    if text == "auto":
        return EpsPolicy.auto()
    if text == "exact":
        return EpsPolicy.exact_zero()
    try:
        return EpsPolicy.fixed(float(text))
    except ValueError as err:
        raise argparse.ArgumentTypeError(f"--eps expects a float, 'auto' or 'exact', got {text!r}") from err


def build_parser():
    parser = argparse.ArgumentParser(prog="rankrls", description=__doc__.split("\n\n")[0])
    sub = parser.add_subparsers(dest="command", required=True)
    solve = sub.add_parser("solve", help="solve a least-squares system from matrix/rhs files")
    solve.add_argument("matrix")
    solve.add_argument("rhs")
    solve.add_argument("--scalar", choices=sorted(KINDS), default="f64")
    solve.add_argument("--variant", choices=VARIANTS, default="general")
    solve.add_argument("--eps", type=_parse_eps, default=None,
                       help="dependency threshold: float, 'auto' or 'exact'")
    solve.add_argument("--out", default=None, help="write x here (an m x 1 matrix file)")
    solve.add_argument("--pinv", default=None, help="also write the pseudoinverse here")
    solve.add_argument("--cov", default=None, help="also write the solution covariance here")
    return parser


def main(argv=None):
    args = build_parser().parse_args(argv)
    try:
        return _cmd_solve(args)
    except (ValueError, OSError, ZeroDivisionError) as err:
        print(f"rankrls {args.command}: {err}", file=sys.stderr)
        return 2


def _cmd_solve(args):
    """cli.py:109-134: read, check shapes, solve (with trackers when A+ / the
    covariance are requested), print x and the rank, optionally write files."""
    kind = KINDS[args.scalar]
    A = matrices.read_matrix(args.matrix, kind)
    y = matrices.read_vector(args.rhs, kind)
    if A.shape[0] != y.shape[0]:
        raise ValueError(f"matrix has {A.shape[0]} rows but rhs has {y.shape[0]} entries")
    if args.pinv or args.cov:
        solver = RecursiveSolver(A.shape[1], variant=args.variant, eps=args.eps, scalar=kind)
        pinv_tracker = PseudoinverseTracker(solver) if args.pinv else None
        cov_tracker = CovarianceTracker(solver) if args.cov else None
        solver.ingest(A, y)
        x, rank = np.asarray(solver.solution), solver.rank
        if pinv_tracker is not None:
            matrices.write_matrix(args.pinv, pinv_tracker.pinv, kind)
        if cov_tracker is not None:
            matrices.write_matrix(args.cov, cov_tracker.covariance, kind)
    else:
        x, rank = solve_batch(A, y, variant=args.variant, eps=args.eps, scalar=kind)
    print(" ".join(kind.render(v) for v in x))
    print(f"rank {rank}")
    if args.out:
        matrices.write_matrix(args.out, np.reshape(x, (-1, 1)), kind)
    return 0


if __name__ == "__main__":
    sys.exit(main())
