"""Report driver for the hot path (the in-scope subcommands of the reference CLI, src/cli.py).

``python -m paper_2407_09621_b200 {solve,convergence,error-profile,residuals} ...`` writes the same
CSV (``# version`` / ``# config`` provenance comments, then one header row) or JSON report as the
reference (src/cli.py:50-78) with the same columns, flags and exit codes (0 ok, 2 usage error,
3 non-convergence with the report still written; src/cli.py:32-34).  Every solve and operator
apply runs on the B200.  The A100 analytical subcommands (bank-sim, roofline, flops) are out of
scope.
"""
from __future__ import annotations

import argparse
import csv
import io
import json
import sys

from . import __version__

EXIT_OK, EXIT_USAGE, EXIT_NO_CONVERGENCE = 0, 2, 3


def _cell(v):
    if isinstance(v, float):
        return format(v, ".17g")
    return "" if v is None else str(v)


def _report(args, columns, rows):
    config = {k: v for k, v in sorted(vars(args).items()) if k not in ("func", "out")}
    if args.format == "json":
        text = json.dumps({"version": __version__, "config": config, "columns": list(columns), "rows": rows},
                          indent=2, sort_keys=True) + "\n"
    else:
        buf = io.StringIO()
        buf.write(f"# version: {__version__}\n# config: {json.dumps(config, sort_keys=True)}\n")
        w = csv.writer(buf, lineterminator="\n")
        w.writerow(columns)
        for row in rows:
            w.writerow([_cell(row.get(c)) for c in columns])
        text = buf.getvalue()
    if args.out:
        with open(args.out, "w") as fh:
            fh.write(text)
    else:
        sys.stdout.write(text)


def _modes(spec):
    from .precision import PrecisionMode

    return [PrecisionMode.parse(s) for s in spec.split(",") if s.strip()]


def cmd_solve(args) -> int:
    """src/cli.py:88-135: one row per precision, speed-up relative to the fp64 row."""
    from . import build_hierarchy, run_solve
    from .precision import PrecisionMode

    hier = build_hierarchy(args.levels, args.k)
    outs = [run_solve(args.k, args.levels, mode=m, solver=args.solver, tol=args.tol, maxit=args.maxit,
                      coarse_level=args.coarse_level, pre_smooth=args.pre_smooth, post_smooth=args.post_smooth,
                      hier=hier) for m in _modes(args.precision)]
    base = next((o.report.wall_time for o in outs if o.mode is PrecisionMode.FP64), None)
    rows = []
    for o in outs:
        fast = None
        if base and o.mode is not PrecisionMode.FP64 and not args.no_timing:
            fast = base / o.report.wall_time
        rows.append({"precision": o.mode.value, "time_s": 0.0 if args.no_timing else o.report.wall_time,
                     "iterations": o.report.iterations, "l2_error": o.l2, "h1_error": o.h1,
                     "speedup_vs_fp64": fast, "converged": o.report.converged, "dofs": o.dofs})
    _report(args, ["precision", "time_s", "iterations", "l2_error", "h1_error", "speedup_vs_fp64", "converged",
                   "dofs"], rows)
    return EXIT_OK if all(o.report.converged for o in outs) else EXIT_NO_CONVERGENCE


def cmd_convergence(args) -> int:
    from .experiments import convergence_study

    rows = convergence_study(args.k, args.levels, solver=args.solver, tol=args.tol, maxit=args.maxit)
    _report(args, ["level", "h", "dofs", "l2_error", "h1_error", "rate", "iterations"], rows)
    return EXIT_OK


def cmd_error_profile(args) -> int:
    from .experiments import error_profile

    rows = error_profile(args.k, args.levels, _modes(args.precision), seed=args.seed)
    _report(args, ["dofs", "level", "mode", "relative_error"], rows)
    return EXIT_OK


def cmd_residuals(args) -> int:
    from . import run_solve

    rows = []
    for m in _modes(args.precision):
        hist = run_solve(args.k, args.levels, mode=m, solver=args.solver, tol=args.tol,
                         maxit=args.maxit).report.residual_history
        rows += [{"precision": m.value, "iteration": i, "residual": r, "relative_residual": r / hist[0]}
                 for i, r in enumerate(hist)]
    _report(args, ["precision", "iteration", "residual", "relative_residual"], rows)
    return EXIT_OK


def build_parser() -> argparse.ArgumentParser:
    ap = argparse.ArgumentParser(prog="paper_2407_09621_b200", description="B200 SIPG sum-factorisation hot path")
    ap.add_argument("--version", action="version", version=__version__)
    sub = ap.add_subparsers(dest="command", required=True)

    def common(p):
        p.add_argument("--out", default=None)
        p.add_argument("--format", choices=("csv", "json"), default="csv")
        p.add_argument("--seed", type=int, default=0)

    def solver_opts(p, precision):
        p.add_argument("--k", type=int, default=3)
        p.add_argument("--levels", type=int, default=3)
        p.add_argument("--precision", default=precision)
        p.add_argument("--solver", choices=("fgmres", "gmres"), default="fgmres")
        p.add_argument("--tol", type=float, default=1e-8)
        p.add_argument("--maxit", type=int, default=100)
        p.add_argument("--coarse-level", type=int, default=1)
        p.add_argument("--pre-smooth", type=int, default=1)
        p.add_argument("--post-smooth", type=int, default=1)

    p = sub.add_parser("solve")
    solver_opts(p, "fp64")
    p.add_argument("--no-timing", action="store_true")
    common(p)
    p.set_defaults(func=cmd_solve)
    p = sub.add_parser("convergence")
    p.add_argument("--k", type=int, default=3)
    p.add_argument("--levels", type=int, default=3)
    p.add_argument("--solver", choices=("fgmres", "gmres"), default="fgmres")
    p.add_argument("--tol", type=float, default=1e-8)
    p.add_argument("--maxit", type=int, default=100)
    common(p)
    p.set_defaults(func=cmd_convergence)
    p = sub.add_parser("error-profile")
    p.add_argument("--k", type=int, default=7)
    p.add_argument("--levels", type=int, default=4)
    p.add_argument("--precision", default="fp32,fp16,fp16_ec")
    common(p)
    p.set_defaults(func=cmd_error_profile)
    p = sub.add_parser("residuals")
    solver_opts(p, "fp64,fp32,fp16_ec")
    common(p)
    p.set_defaults(func=cmd_residuals)
    return ap


def main(argv=None) -> int:
    args = build_parser().parse_args(argv)
    return args.func(args)


if __name__ == "__main__":
    sys.exit(main())
