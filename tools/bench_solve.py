"""Time-to-solution of the manufactured Poisson problem (BASELINE configs[3]):
FGMRES (fp64) preconditioned by the V-cycle in fp64 / fp16 / fp16_ec.

Setup (hierarchy, eigh, coarse LU, rhs) is excluded from the timed region and
reported separately, as SURVEY.md §8d prescribes.  One JSON line per solve.
python tools/bench_solve.py --degree 7 --level 6 --modes fp64,fp16_ec,fp16
"""
import argparse
import json
import math
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2407_09621_b200 as sf  # noqa: E402
from paper_2407_09621_b200.discretization import assemble_rhs_separable, l2_error_separable  # noqa: E402
from paper_2407_09621_b200.experiments import make_operator  # noqa: E402


def solve_once(hier, level, mode, tol=1e-8, reps=5, graph=False):
    """Median (and min / max) wall time of `reps` FGMRES solves after one warm-up V-cycle; setup excluded."""
    t0 = time.perf_counter()
    sine = lambda x: np.sin(np.pi * x)
    b = assemble_rhs_separable(hier, level, sine, 3.0 * math.pi**2)
    mg = sf.MultigridPreconditioner(hier, sf.VCycleConfig(mode=mode)).setup().enable_graph(graph)
    A = make_operator(hier, level)
    M = lambda v: mg.apply(v, level)
    M(b)  # warm-up: workspaces, table uploads
    torch.cuda.synchronize()
    setup = time.perf_counter() - t0
    times, rep, x = [], None, None
    for _ in range(reps):
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        x, rep = sf.fgmres(A, M, b, tol=tol, maxit=100)
        torch.cuda.synchronize()
        times.append(time.perf_counter() - t1)
    l2 = l2_error_separable(hier, level, x, sine)
    med = float(np.median(times))
    return {"degree": hier.degree, "level": level, "dofs": hier.n_dofs(level), "mode": mode.value,
            "iterations": rep.iterations, "solve_s": med, "solve_s_min": min(times), "solve_s_max": max(times),
            "solves_timed": reps, "setup_s": setup, "l2_error": l2,
            "final_rel_res": rep.final_relative_residual, "converged": rep.converged, "cuda_graph": graph}


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--degree", type=int, default=7)
    ap.add_argument("--level", type=int, default=6)
    ap.add_argument("--modes", default="fp64,fp16_ec,fp16")
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--graph", action="store_true", help="replay V-cycles from captured CUDA graphs")
    a = ap.parse_args()
    hier = sf.build_hierarchy(a.level, a.degree, max_dofs=2**34)
    for m in a.modes.split(","):
        print(json.dumps(solve_once(hier, a.level, sf.PrecisionMode.parse(m), reps=a.reps, graph=a.graph)), flush=True)
