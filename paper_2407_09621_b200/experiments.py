"""Solve driver and measurement harnesses (mirror of src/experiments.py: run_solve :57-103,
convergence_study :106-127, error_profile :130-148)."""
from __future__ import annotations

from dataclasses import dataclass

import torch

from .discretization import MeshHierarchy, build_hierarchy, sine_product_problem, vmult_device
from .krylov import fgmres, gmres
from .multigrid import MultigridPreconditioner, VCycleConfig
from .precision import PrecisionMode


@dataclass
class SolveOutcome:
    degree: int
    level: int
    mode: PrecisionMode
    solver: str
    dofs: int
    report: object
    l2: float
    h1: float
    x: object = None


def make_operator(hier: MeshHierarchy, level: int):
    """fp64 vmult on device tensors: the apply_A the solve hands to (F)GMRES."""
    def apply_A(v: torch.Tensor) -> torch.Tensor:
        out = torch.empty_like(v)
        vmult_device(hier, level, v, out, PrecisionMode.FP64)
        return out
    return apply_A


def run_solve(degree: int, level: int, mode: PrecisionMode = PrecisionMode.FP64, solver: str = "fgmres",
              tol: float = 1e-8, maxit: int = 100, coarse_level: int = 1, pre_smooth: int = 1,
              post_smooth: int = 1, hier: MeshHierarchy | None = None, keep_solution: bool = False) -> SolveOutcome:
    """Solve the manufactured Poisson problem with a V-cycle preconditioner (experiments.py:57-103).

    The Krylov vectors never leave the device; the rhs is uploaded once and
    the solution downloaded once for the error norms.
    """
    if solver not in ("fgmres", "gmres"):
        raise ValueError(f"unknown solver {solver!r}")
    import math

    import numpy as np

    from .discretization import assemble_rhs_separable, h1_seminorm_error_separable, l2_error_separable

    hier = hier or build_hierarchy(level, degree)
    sine_product_problem(hier.dim)  # the manufactured problem of the reference (discretization.py:504-531)
    # its data are separable products of sin(pi x): load vector and error norms stay on the device
    sine = lambda x: np.sin(np.pi * x)
    dsine = lambda x: np.pi * np.cos(np.pi * x)
    b = assemble_rhs_separable(hier, level, sine, 3.0 * math.pi**2)
    mg = MultigridPreconditioner(hier, VCycleConfig(pre_smooth_steps=pre_smooth, post_smooth_steps=post_smooth,
                                                    coarse_level=coarse_level, mode=mode))
    run = fgmres if solver == "fgmres" else gmres
    x, report = run(make_operator(hier, level), lambda v: mg.apply(v, level), b, tol=tol, maxit=maxit)
    report.l2_error = l2_error_separable(hier, level, x, sine)
    report.h1_error = h1_seminorm_error_separable(hier, level, x, sine, dsine)
    return SolveOutcome(degree=degree, level=level, mode=mode, solver=solver, dofs=hier.n_dofs(level),
                        report=report, l2=report.l2_error, h1=report.h1_error, x=x if keep_solution else None)


def convergence_study(degree: int, max_level: int, solver: str = "fgmres", tol: float = 1e-8,
                      maxit: int = 100) -> list[dict]:
    """Per-level errors and observed orders for the manufactured problem (experiments.py:106-127)."""
    import numpy as np

    hier = build_hierarchy(max_level, degree)
    rows = []
    prev_l2 = None
    for level in hier.levels():
        out = run_solve(degree, level, solver=solver, tol=tol, maxit=maxit, hier=hier)
        rate = float(np.log2(prev_l2 / out.l2)) if prev_l2 else None
        rows.append({"level": level, "h": hier.h(level), "dofs": out.dofs, "l2_error": out.l2,
                     "h1_error": out.h1, "rate": rate, "iterations": out.report.iterations})
        prev_l2 = out.l2
    return rows


def error_profile(degree: int, max_level: int, modes, seed: int = 0) -> list[dict]:
    """Relative error of one operator apply against fp64, per size and mode (experiments.py:130-148).

    Same seeded inputs as the reference (one standard-normal draw per level, in level order);
    every apply runs on the device.
    """
    import numpy as np

    from .discretization import apply_operator
    from .precision import relative_error

    hier = build_hierarchy(max_level, degree)
    rng = np.random.default_rng(seed)
    rows = []
    for level in hier.levels():
        u = rng.standard_normal(hier.n_dofs(level))
        ref = apply_operator(hier, level, u, PrecisionMode.FP64)
        for mode in modes:
            out = apply_operator(hier, level, u, mode)
            rows.append({"dofs": hier.n_dofs(level), "level": level, "mode": mode.value,
                         "relative_error": relative_error(out, ref)})
    return rows
