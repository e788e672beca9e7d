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
    A = make_spd(30, 3)
    rng = np.random.default_rng(4)
    Ms = [np.diag(rng.uniform(0.5, 2.0, 30)) for _ in range(40)]
    calls = {"i": 0}

    def M(v):
        m = Ms[calls["i"]]
        calls["i"] += 1
        return m @ v

    _, rep = sf.fgmres(lambda v: A @ v, M, np.ones(30), tol=1e-10, maxit=20, collect_bases=True)
    V, H, Z = rep.bases
    m = rep.iterations
    assert np.linalg.norm(A @ Z[:, :m] - V[:, :m + 1] @ H) <= 1e-10 * np.linalg.norm(A @ Z[:, :m]) or rep.breakdown


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
    # comparable iteration count, same discretisation error
    assert abs(rep.iterations - ref_its) <= (0 if mode in (P.FP64, P.FP32) else 2), (rep.iterations, ref_its)
    assert abs(out.l2 - ref_l2) <= 0.02 * ref_l2, (out.l2, ref_l2)
