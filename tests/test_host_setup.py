"""Host-side setup of the product (1-D matrices, packed kernel blocks, API guards)
against the reference's golden matrices -- CPU only."""
import numpy as np
import pytest

import paper_2407_09621_b200 as sf
from paper_2407_09621_b200.basis import gauss_lobatto_points, penalty


@pytest.mark.parametrize("k", [1, 2, 3, 7])
@pytest.mark.parametrize("lvl", [1, 2, 3])
def test_level_matrices_bitwise_match_reference(gold, k, lvl):
    g = gold("matrices")
    lm = sf.build_hierarchy(lvl, k).matrices(lvl)
    for name in ("M_cell", "L_cell", "M_patch", "L_tile", "B_left", "B_right", "F_cross"):
        assert np.array_equal(getattr(lm, name), g[f"k{k}_l{lvl}_{name}"]), name
    for (lb, rb), L in lm.L_smooth.items():
        assert np.array_equal(L, g[f"k{k}_l{lvl}_Ls{int(lb)}{int(rb)}"])


def test_cellwise_blocks_reassemble_the_global_operator():
    """The packed (M, D, U, Bl, Br) blocks rebuild the reference's dense operator."""
    from oracle import port

    for k, L in [(1, 1), (2, 2), (3, 1)]:
        lm = sf.build_hierarchy(L, k).matrices(L)
        K, n = k + 1, 2**L
        op = lm.cell_op
        M = op[:K * K].reshape(K, K)
        D = op[K * K:2 * K * K].reshape(K, K)
        ucol, urow, bl, br = (op[2 * K * K + i * K:2 * K * K + (i + 1) * K] for i in range(4))
        U = np.zeros((K, K)); U[:, 0] = ucol; U[K - 1, :] = urow
        Bl = np.zeros((K, K)); Bl[:, 0] = bl; Bl[0, :] = bl
        Br = np.zeros((K, K)); Br[:, K - 1] = br; Br[K - 1, :] = br
        A1 = np.zeros((n * K, n * K))
        M1 = np.kron(np.eye(n), M)
        for c in range(n):
            s = slice(c * K, (c + 1) * K)
            A1[s, s] = D + (Bl if c == 0 else 0) + (Br if c == n - 1 else 0)
            if c + 1 < n:
                s2 = slice((c + 1) * K, (c + 2) * K)
                A1[s, s2] = U
                A1[s2, s] = U.T
        A3 = np.kron(np.kron(A1, M1), M1) + np.kron(np.kron(M1, A1), M1) + np.kron(np.kron(M1, M1), A1)
        Aref = port.materialize(port.Hierarchy(L, k), L)
        assert np.linalg.norm(A3 - Aref) / np.linalg.norm(Aref) < 1e-14


def test_hierarchy_guards():
    with pytest.raises(ValueError):
        sf.build_hierarchy(0, 1)
    with pytest.raises(ValueError):
        sf.build_hierarchy(3, 3, max_dofs=1000)
    with pytest.raises(ValueError):
        sf.build_hierarchy(2, 1, dim=4)
    with pytest.raises(NotImplementedError):
        sf.build_hierarchy(2, 8)
    h = sf.build_hierarchy(2, 3)
    assert h.n_dofs(2) == 4096 and h.matrices(2).M_patch.shape == (8, 8)


def test_precision_parse_and_storage():
    P = sf.PrecisionMode
    assert P.parse("half") is P.FP16 and P.parse("FP16-EC") is P.FP16_EC and P.parse("double") is P.FP64
    with pytest.raises(ValueError):
        P.parse("fp8")
    assert P.FP64.storage_dtype == np.float64 and P.FP16.storage_dtype == np.float32


def test_basis_basics():
    assert np.allclose(gauss_lobatto_points(2), [0.0, 0.5, 1.0])
    assert penalty(3, 0.25, 0.25) == pytest.approx(96.0)


def test_vcycle_config_guards():
    with pytest.raises(ValueError):
        sf.VCycleConfig(pre_smooth_steps=0)
    with pytest.raises(ValueError):
        sf.VCycleConfig(coarse_level=0)
    h = sf.build_hierarchy(2, 1)
    with pytest.raises(ValueError, match="ordering"):
        sf.MultigridPreconditioner(h, sf.VCycleConfig(smoother_ordering=((0, 0, 0), (1, 1, 1))))
    sf.MultigridPreconditioner(h, sf.VCycleConfig(smoother_ordering=tuple(reversed(sf.default_ordering(3)))))


def test_krylov_argument_guards():
    with pytest.raises(ValueError):
        sf.fgmres(lambda v: v, None, None)
    with pytest.raises(ValueError):
        sf.gmres(lambda v: v, None, np.ones(3), tol=1.5)
