"""Pins the cell-local vmult evaluator (tests/local_stencil.py) to the oracle
on whole meshes, so the GPU spot checks at bench size inherit the oracle's
parity (CPU only)."""
import numpy as np
import pytest

from conftest import rel_l2
from local_stencil import LocalVmult, global_1d, sample_cells
from oracle import port


@pytest.mark.parametrize("k,lvl", [(1, 1), (1, 3), (3, 2), (3, 3), (7, 1), (7, 2)])
def test_local_evaluator_equals_oracle(k, lvl):
    H = port.Hierarchy(lvl, k)
    u = np.random.default_rng(3).standard_normal(H.n_dofs(lvl))
    ref = port.apply_operator(H, lvl, u)
    v = LocalVmult(k, lvl).apply_full(u)
    assert rel_l2(v, ref) <= 1e-13


def test_global_1d_is_symmetric_and_block_tridiagonal():
    L1, M1 = global_1d(7, 3)
    assert np.allclose(L1, L1.T, atol=1e-12 * np.abs(L1).max())
    K = 8
    for i in range(8):
        for j in range(8):
            if abs(i - j) > 1:
                assert not L1[i * K:(i + 1) * K, j * K:(j + 1) * K].any()


def test_sample_cells_cover_corners_and_band_edges():
    cells = sample_cells(128, 100)
    assert (0, 0, 0) in cells and (127, 127, 127) in cells
    assert any(c[1] == 16 for c in cells) and any(c[1] == 15 for c in cells)
    assert all(0 <= x < 128 for c in cells for x in c)
