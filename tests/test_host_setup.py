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


def _global_1d(k, L):
    """The level's 1-D SIPG operator over all cells, rebuilt from the packed cell-wise blocks."""
    lm = sf.build_hierarchy(L, k).matrices(L)
    K, n = k + 1, 2**L
    op = lm.cell_op
    D = op[K * K:2 * K * K].reshape(K, K)
    ucol, urow, bl, br = (op[2 * K * K + i * K:2 * K * K + (i + 1) * K] for i in range(4))
    U = np.zeros((K, K)); U[:, 0] = ucol; U[K - 1, :] = urow
    Bl = np.zeros((K, K)); Bl[:, 0] = bl; Bl[0, :] = bl
    Br = np.zeros((K, K)); Br[:, K - 1] = br; Br[K - 1, :] = br
    A1 = np.zeros((n * K, n * K))
    for c in range(n):
        s = slice(c * K, (c + 1) * K)
        A1[s, s] = D + (Bl if c == 0 else 0) + (Br if c == n - 1 else 0)
        if c + 1 < n:
            s2 = slice((c + 1) * K, (c + 2) * K)
            A1[s, s2], A1[s2, s] = U, U.T
    return A1, lm


@pytest.mark.parametrize("k", [1, 3, 7])
def test_tile_line_operators_are_principal_submatrices(k):
    """The tensor-core kernels contract 16-point tile lines (16/K cells) with the block-tridiagonal line
    operator and couple to the cells outside the line through rank-2 (alpha, beta) halos.  For that to be
    exact, the line operator must be the principal 16 x 16 submatrix of the global 1-D operator and the
    coupling to the outside must touch only the face nodes -- checked for every line position."""
    K = k + 1
    A1, lm = _global_1d(k, 4)
    n = 2**4
    cpl = 16 // K
    for c0 in range(0, n - cpl + 1, 2 if k == 7 else cpl):
        s = slice(c0 * K, c0 * K + 16)
        block = A1[s, s]
        assert np.allclose(block, block.T)
        outside = np.delete(A1[s, :], np.r_[s], axis=1)
        rows, cols = np.nonzero(outside)
        # only the line's first and last cell couple outside, each through a rank-2 face block
        assert set(rows) <= set(range(K)) | set(range(16 - K, 16))
        if outside.any():
            assert np.linalg.matrix_rank(outside) <= 4
    # the 2-cell (Q7 patch) line with Nitsche at both ends is L_smooth[(True, True)] at level 1
    A1b, lmb = _global_1d(k, 1)
    if k == 7:
        assert np.allclose(A1b, lmb.L_smooth[(True, True)], atol=1e-12 * np.abs(A1b).max())


def test_slab_levels_property_sweep():
    """Every (max level, world) combination: slabs partition z, are even and >= 2 cells, agree across ranks."""
    from paper_2407_09621_b200 import slab

    for L in range(1, 7):
        hier = sf.build_hierarchy(L, 1)
        for G in (1, 2, 3, 4, 6, 8, 16):
            per_rank = [slab.slab_levels(hier, r, G) for r in range(G)]
            lv = sorted(per_rank[0])
            assert all(sorted(p) == lv for p in per_rank)
            for lvl in lv:
                n = hier.n_cells(lvl)
                nz = [p[lvl].nz for p in per_rank]
                assert sum(nz) == n and all(z == nz[0] and z % 2 == 0 and z >= 2 for z in nz)
                assert [p[lvl].z0 for p in per_rank] == list(range(0, n, nz[0]))
                for p in per_rank:
                    sl = p[lvl]
                    assert sl.ext_dofs == sl.local_dofs + (sl.h_lo + sl.h_hi) * sl.cell_layer


@pytest.mark.parametrize("fmt", ["csv", "bin"])
def test_vector_serialization_roundtrip(tmp_path, fmt):
    """tests/test_discretization.py:364-374 of the reference: exact round trip, unknown format -> ValueError."""
    from paper_2407_09621_b200.discretization import load_vector, save_vector

    u = np.random.default_rng(21).standard_normal(64)
    path = tmp_path / f"vec.{fmt}"
    save_vector(path, u, fmt=fmt)
    assert np.array_equal(load_vector(path, fmt=fmt), u)
    with pytest.raises(ValueError):
        save_vector(path, u, fmt="hdf5")
    with pytest.raises(ValueError):
        load_vector(path, fmt="hdf5")


def test_vector_csv_format_matches_reference_writer(tmp_path):
    """Byte-identical to the reference's per-row f"{i},{v:.17g}" writer (discretization.py:470-472), and rows are
    re-sorted by index on load."""
    from paper_2407_09621_b200.discretization import load_vector, save_vector

    u = np.concatenate([np.random.default_rng(3).standard_normal(40) * 10.0 ** np.arange(-20, 20),
                        [0.0, -0.0, 1e308, -5e-324, 1.0 / 3.0, np.inf, -np.inf]])
    path = tmp_path / "v.csv"
    save_vector(path, u)
    expect = "index,value\n" + "".join(f"{i},{v:.17g}\n" for i, v in enumerate(u))
    assert path.read_text() == expect
    lines = path.read_text().splitlines()
    shuffled = tmp_path / "s.csv"
    shuffled.write_text("\n".join([lines[0]] + lines[1:][::-1]) + "\n")
    got = load_vector(shuffled)
    assert np.array_equal(got, u)
    one = tmp_path / "one.csv"
    save_vector(one, u[:1])
    assert np.array_equal(load_vector(one), u[:1])
