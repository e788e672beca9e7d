"""Pin the CPU oracle (oracle/port.py) against golden vectors from the reference.

The fixtures in tests/golden/ were produced by tools/make_golden.py, which
imports the reference package itself.  If the port drifts from the reference,
these fail before any GPU comparison is trusted.
"""
import numpy as np
import pytest

from conftest import rel_l2
from oracle import port

MODES = port.MODES


@pytest.mark.parametrize("k", [1, 2, 3, 7])
@pytest.mark.parametrize("lvl", [1, 2, 3])
def test_level_matrices_match_reference(gold, k, lvl):
    g = gold("matrices")
    lm = port.level_matrices(k, lvl)
    for name in ("M_cell", "L_cell", "M_patch", "L_tile", "B_left", "B_right", "F_cross"):
        ref = g[f"k{k}_l{lvl}_{name}"]
        assert np.allclose(getattr(lm, name), ref, rtol=1e-13, atol=1e-13 * np.abs(ref).max())
    for (lb, rb), L in lm.L_smooth.items():
        ref = g[f"k{k}_l{lvl}_Ls{int(lb)}{int(rb)}"]
        assert np.allclose(L, ref, rtol=1e-13, atol=1e-13 * np.abs(ref).max())
    assert np.array_equal(port.embedding(k), g[f"k{k}_P"])


@pytest.mark.parametrize("k,lvl", [(1, 1), (1, 2), (2, 2), (3, 2), (3, 3), (7, 1), (7, 2)])
@pytest.mark.parametrize("mode", MODES)
def test_port_vmult_matches_reference(gold, k, lvl, mode):
    H = port.Hierarchy(lvl, k)
    u = np.random.default_rng(0).standard_normal(H.n_dofs(lvl))
    v = port.apply_operator(H, lvl, u, mode)
    ref = gold("vmult")[f"k{k}_l{lvl}_{mode}"]
    assert v.dtype == ref.dtype
    tol = 1e-14 if mode == "fp64" else 1e-6
    assert rel_l2(v, ref) <= tol


def test_port_vmult_matches_dense_assembly(gold):
    """The reference's independent dense SIPG assembly (tests/sipg_oracle.py)."""
    g = gold("sipg_dense")
    for k, lvl, key in [(1, 1, "k1_l1"), (1, 2, "k1_l2"), (2, 1, "k2_l1")]:
        A = port.materialize(port.Hierarchy(lvl, k), lvl)
        assert rel_l2(A, g[key]) <= 1e-12


@pytest.mark.parametrize("k,lvl", [(1, 2), (2, 2), (3, 2), (7, 2), (1, 3)])
@pytest.mark.parametrize("mode", MODES)
def test_port_smoother_and_transfers_match_reference(gold, k, lvl, mode):
    g = gold("smoother")
    H = port.Hierarchy(lvl, k)
    D = H.n_dofs(lvl)
    x = np.random.default_rng(1).standard_normal(D)
    x /= np.linalg.norm(x)
    b = np.random.default_rng(2).standard_normal(D)
    b /= np.linalg.norm(b)
    tol = 1e-12 if mode == "fp64" else 1e-5
    mg = port.VCycle(H, mode=mode)
    assert rel_l2(mg.smooth(lvl, x, b, mode), g[f"smooth_k{k}_l{lvl}_{mode}"]) <= tol
    assert rel_l2(port.restrict(H, lvl, x, mode), g[f"restrict_k{k}_l{lvl}_{mode}"]) <= tol
    e = np.random.default_rng(3).standard_normal(H.n_dofs(lvl - 1))
    assert rel_l2(port.prolongate(H, lvl - 1, e, mode), g[f"prolong_k{k}_l{lvl}_{mode}"]) <= tol


@pytest.mark.parametrize("k,lvl", [(1, 3), (3, 3), (2, 2), (7, 2)])
@pytest.mark.parametrize("mode", MODES)
def test_port_vcycle_matches_reference(gold, k, lvl, mode):
    H = port.Hierarchy(lvl, k)
    b = np.random.default_rng(4).standard_normal(H.n_dofs(lvl))
    b /= np.linalg.norm(b)
    out = port.VCycle(H, mode=mode).apply(b, lvl)
    ref = gold("vcycle")[f"vcycle_k{k}_l{lvl}_{mode}"]
    tol = 1e-11 if mode == "fp64" else 2e-3
    assert rel_l2(out, ref) <= tol


def test_port_demote16_matches_reference(gold):
    g = gold("half")
    assert np.array_equal(port.demote16(g["x"]).view(np.uint32), g["demoted"].view(np.uint32))
