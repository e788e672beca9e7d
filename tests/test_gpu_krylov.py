"""GPU FGMRES/GMRES: reference behaviour on dense SPD systems and the
manufactured-solution solves against the reference's golden iteration counts
and L2 errors."""
import numpy as np
import pytest

import paper_2407_09621_b200 as sf

pytestmark = pytest.mark.gpu
P = sf.PrecisionMode


def make_spd(n, seed, cond=100.0):
    rng = np.random.default_rng(seed)
    Q, _ = np.linalg.qr(rng.standard_normal((n, n)))
    return Q @ np.diag(np.geomspace(1.0, cond, n)) @ Q.T


def test_identity_and_exact_preconditioner_one_iteration():
    b = np.arange(1.0, 6.0)
    for solver in (sf.fgmres, sf.gmres):
        x, rep = solver(lambda v: v, None, b)
        assert rep.iterations == 1 and rep.converged and np.allclose(x, b)
    d = np.array([1.0, 10.0, 100.0, 1000.0])
    x, rep = sf.fgmres(lambda v: d * v, lambda v: v / d, np.ones(4))
    assert rep.iterations == 1 and np.allclose(x, 1 / d, rtol=1e-12)


def test_dense_solve_history_and_maxit():
    A = make_spd(40, 0)
    x, rep = sf.fgmres(lambda v: A @ v, None, np.ones(40), tol=1e-10, maxit=60)
    assert rep.converged and np.linalg.norm(A @ x - 1.0) <= 1e-9 * np.sqrt(40)
    h = np.asarray(rep.residual_history)
    assert len(h) == rep.iterations + 1 and np.all(h[1:] <= h[:-1] + 10 * np.finfo(float).eps * h[0])
    A2 = make_spd(50, 2, cond=1e6)
    _, rep2 = sf.fgmres(lambda v: A2 @ v, None, np.ones(50), tol=1e-12, maxit=5)
    assert not rep2.converged and rep2.iterations == 5 and len(rep2.residual_history) == 6


def test_flexible_arnoldi_relation():
    """tests/test_krylov.py:78-100: A Z = V (V^T A Z) with a different M every call."""
    A = make_spd(20, 5)
    rng = np.random.default_rng(6)
    precs = [np.linalg.inv(make_spd(20, 10 + i, cond=5.0)) for i in range(30)]
    calls = {"n": 0}

    def M(v):
        out = precs[calls["n"] % len(precs)] @ v
        calls["n"] += 1
        return out

    b = rng.standard_normal(20)
    _, rep = sf.fgmres(lambda v: A @ v, M, b, tol=1e-12, maxit=15, collect_bases=True)
    V, H, Z = rep.bases
    AZ = A @ Z
    assert np.linalg.norm(AZ - V @ (V.T @ AZ)) <= 1e-12 * np.linalg.norm(AZ)
    assert V.shape[1] in (rep.iterations, rep.iterations + 1)


def test_gmres_equals_fgmres_for_fixed_linear_preconditioner():
    A = make_spd(25, 3)
    M = np.linalg.inv(make_spd(25, 4, cond=10.0))
    b = np.sin(np.arange(25.0))
    xf, rf = sf.fgmres(lambda v: A @ v, lambda v: M @ v, b, tol=1e-10, maxit=40)
    xg, rg = sf.gmres(lambda v: A @ v, lambda v: M @ v, b, tol=1e-10, maxit=40)
    assert rf.iterations == rg.iterations
    assert np.allclose(rf.residual_history, rg.residual_history, rtol=1e-10)
    assert np.allclose(xf, xg, rtol=1e-9, atol=1e-12)


def test_fgmres_beats_gmres_with_nonlinear_preconditioner():
    A = make_spd(30, 7)
    count = {"n": 0}

    def rough(v):
        count["n"] += 1
        return (v / np.diag(A)) * (1.0 + 0.2 * np.sin(count["n"] * np.arange(30.0)))

    b = np.ones(30)
    xf, _ = sf.fgmres(lambda v: A @ v, rough, b, tol=1e-10, maxit=30)
    count["n"] = 0
    xg, _ = sf.gmres(lambda v: A @ v, rough, b, tol=1e-10, maxit=30)
    assert np.linalg.norm(A @ xf - b) < np.linalg.norm(A @ xg - b)


def test_zero_rhs():
    x, rep = sf.fgmres(lambda v: v, None, np.zeros(7))
    assert rep.iterations == 0 and rep.converged and np.all(x == 0)


SOLVE_CASES = [(1, 2), (1, 3), (2, 3), (3, 2), (3, 3), (7, 2)]


@pytest.mark.parametrize("k,lvl", SOLVE_CASES)
@pytest.mark.parametrize("mode", [P.FP64, P.FP32, P.FP16, P.FP16_EC])
def test_solve_matches_reference(gold, k, lvl, mode):
    g = gold("solves")
    sel = (g["k"] == k) & (g["level"] == lvl) & (g["mode"] == mode.value) & (g["solver"] == "fgmres")
    i = int(np.flatnonzero(sel)[0])
    out = sf.run_solve(k, lvl, mode=mode)
    rep = out.report
    assert rep.converged
    ref_its, ref_l2 = int(g["iterations"][i]), float(g["l2"][i])
    j = int(np.flatnonzero((g["k"] == k) & (g["level"] == lvl) & (g["mode"] == "fp64"))[0])
    ref64_l2 = float(g["l2"][j])
    # comparable iteration count ...
    assert abs(rep.iterations - ref_its) <= (1 if mode in (P.FP64, P.FP32) else 2), (rep.iterations, ref_its)
    # ... and the reference's FP64 discretisation error.  Where the algebraic error
    # (tol 1e-8) dominates (Q7 L2, L2 ~ 1e-10), require the same error level instead.
    if ref64_l2 > 1e-9:
        assert abs(out.l2 - ref_l2) <= 0.02 * ref_l2, (out.l2, ref_l2)
    else:
        assert out.l2 <= 1.5 * max(ref_l2, ref64_l2), (out.l2, ref_l2, ref64_l2)


def test_device_rhs_and_l2_error_match_host():
    import math

    import torch

    from paper_2407_09621_b200.discretization import assemble_rhs_separable, l2_error_separable

    hier = sf.build_hierarchy(3, 3)
    prob = sf.sine_product_problem(3)
    sine = lambda x: np.sin(np.pi * x)
    b_dev = assemble_rhs_separable(hier, 3, sine, 3.0 * math.pi**2)
    b_host = sf.assemble_rhs(hier, 3, prob.rhs)
    assert np.linalg.norm(b_dev.cpu().numpy() - b_host) <= 1e-13 * np.linalg.norm(b_host)
    u = torch.randn(hier.n_dofs(3), dtype=torch.float64, device="cuda")
    e_dev = l2_error_separable(hier, 3, u, sine)
    e_host = sf.l2_error(hier, 3, u.cpu().numpy(), prob.exact)
    assert abs(e_dev - e_host) <= 1e-12 * e_host
    from paper_2407_09621_b200.discretization import h1_seminorm_error_separable

    h_dev = h1_seminorm_error_separable(hier, 3, u, sine, lambda x: np.pi * np.cos(np.pi * x))
    h_host = sf.h1_seminorm_error(hier, 3, u.cpu().numpy(), prob.gradient)
    assert abs(h_dev - h_host) <= 1e-12 * h_host
