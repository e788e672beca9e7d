"""The reference's end-to-end acceptance criteria for the hot path (tests/test_acceptance.py of the
reference, criteria 3-7 and 9), run through the B200 path.  Solves are cached across criteria the
same way (test_acceptance.py:41-57)."""
import itertools
import json
import os

import numpy as np
import pytest

import paper_2407_09621_b200 as sf

pytestmark = pytest.mark.gpu
P = sf.PrecisionMode
_H, _S = {}, {}
GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def hierarchy(k, max_level):
    if (k, max_level) not in _H:
        _H[(k, max_level)] = sf.build_hierarchy(max_level, k)
    return _H[(k, max_level)]


def solve(k, level, mode=P.FP64, solver="fgmres", max_level=None):
    key = (k, level, mode, solver)
    if key not in _S:
        _S[key] = sf.run_solve(k, level, mode=mode, solver=solver, hier=hierarchy(k, max_level or level))
    return _S[key]


def test_criterion_03_discretization_convergence():
    """test_acceptance.py:113-128: L2 slope >= k + 0.8 over levels 2..4."""
    for k in (1, 2, 3):
        levels = (2, 3, 4)
        errs = [solve(k, lvl, max_level=4).l2 for lvl in levels]
        hs = [hierarchy(k, 4).h(lvl) for lvl in levels]
        slope = np.polyfit(np.log(hs), np.log(errs), 1)[0]
        assert slope >= k + 0.8, (k, slope, errs)


def test_criterion_04_multigrid_efficiency_band():
    """test_acceptance.py:131-136: <= 6 iterations, spread <= 2."""
    for k in (1, 3):
        its = [solve(k, lvl, max_level=4).report.iterations for lvl in (2, 3, 4)]
        assert max(its) <= 6 and max(its) - min(its) <= 2, (k, its)


def test_criterion_05_precision_ladder():
    """test_acceptance.py:139-158."""
    levels = (2, 3, 4)
    fp32 = [solve(3, lvl, P.FP32, max_level=4).report.iterations for lvl in levels]
    ec = [solve(3, lvl, P.FP16_EC, max_level=4).report.iterations for lvl in levels]
    fp16_finest = solve(3, 4, P.FP16, max_level=4).report.iterations
    assert all(abs(a - b) <= 1 for a, b in zip(fp32, ec)), (fp32, ec)
    assert solve(3, 4, P.FP16_EC, max_level=4).l2 <= 2.0 * solve(3, 4, P.FP64, max_level=4).l2
    assert fp16_finest > ec[-1], (fp16_finest, ec)


def test_criterion_06_residual_overlap():
    """test_acceptance.py:161-170: residual histories within 10 %."""
    hists = {m: np.asarray(solve(3, 3, m, max_level=4).report.residual_history)
             for m in (P.FP64, P.FP32, P.FP16_EC)}
    worst = 0.0
    for a, b in itertools.combinations(hists.values(), 2):
        m = min(len(a), len(b))
        worst = max(worst, float(np.max(np.abs(a[:m] - b[:m]) / np.maximum(a[:m], b[:m]))))
    assert worst <= 0.10, worst


def test_criterion_07_fgmres_vs_gmres():
    """test_acceptance.py:173-183: flexible beats standard GMRES with half-precision cycles."""
    f = solve(3, 4, P.FP16, "fgmres", max_level=4).l2
    g = solve(3, 4, P.FP16, "gmres", max_level=4).l2
    assert f <= g, (f, g)


def test_criterion_09_error_profile_ordering_and_reference_values():
    """test_acceptance.py:213-233 (ordering clause) + the reference's own error_profile(7, 4) values."""
    modes = (P.FP32, P.FP16, P.FP16_EC)
    rows = sf.error_profile(7, 4, modes, seed=0)
    by = {m.value: np.array([r["relative_error"] for r in rows if r["mode"] == m.value]) for m in modes}
    assert np.all(by["fp16"] >= 10 * by["fp32"]) and np.all(by["fp16_ec"] <= 4 * by["fp32"]), by
    ref = json.load(open(os.path.join(GOLDEN, "error_profile_k7_l4.json")))
    for r, g in zip(rows, ref):
        assert (r["level"], r["mode"]) == (g["level"], g["mode"])
        # same inputs, same per-contraction demotion: errors agree to within a factor 2
        assert 0.5 * g["relative_error"] <= r["relative_error"] <= 2.0 * g["relative_error"], (r, g)


def test_fused_gram_schmidt_is_bitwise_the_separate_one():
    """sf_axpy_dot / sf_dot2 (one pass over w per MGS step) reproduce the separate sf_dot + sf_axpy_dev sweep
    bit for bit: same iterates, residual history and solution."""
    from paper_2407_09621_b200 import krylov

    hier = sf.build_hierarchy(4, 3)
    b = np.random.default_rng(7).standard_normal(hier.n_dofs(4))
    mg = sf.MultigridPreconditioner(hier)
    A = lambda v: sf.apply_operator(hier, 4, v)
    M = lambda v: mg.apply(v, 4)
    outs = []
    for fused in (True, False):
        krylov.FUSED_MGS = fused
        try:
            outs.append(sf.fgmres(A, M, b, tol=1e-10, maxit=40))
        finally:
            krylov.FUSED_MGS = True
    (x1, r1), (x2, r2) = outs
    assert r1.iterations == r2.iterations and r1.residual_history == r2.residual_history
    assert np.array_equal(x1, x2)
