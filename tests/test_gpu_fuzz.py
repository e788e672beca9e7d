"""Randomised parity sweep (seeded): vmult, smoother sweep and V-cycle against the oracle port for random
degree / level / mode combinations, and slab-ghost vmults for random slab splits."""
import numpy as np
import pytest
import torch

import paper_2407_09621_b200 as sf
from conftest import rel_l2
from oracle import port

pytestmark = pytest.mark.gpu
P = sf.PrecisionMode
RNG = np.random.default_rng(20261017)
CASES = [(int(k), int(l)) for k, l in zip(RNG.integers(1, 8, 12), RNG.integers(1, 4, 12)) if (k + 1) ** 3 * 8**l <= 2**19]


@pytest.mark.parametrize("k,lvl", CASES)
def test_random_fp64_vmult_smoother_vcycle(k, lvl):
    rng = np.random.default_rng(k * 100 + lvl)
    hier = sf.build_hierarchy(lvl, k)
    H = port.Hierarchy(lvl, k)
    D = hier.n_dofs(lvl)
    u = rng.standard_normal(D)
    assert rel_l2(sf.apply_operator(hier, lvl, u), port.apply_operator(H, lvl, u)) <= 1e-12
    if lvl >= 2:
        x, b = rng.standard_normal(D), rng.standard_normal(D)
        got = sf.MultigridPreconditioner(hier).smooth(lvl, x, b)
        ref = port.VCycle(H).smooth(lvl, x, b)
        assert rel_l2(got, ref) <= 1e-11
        b /= np.linalg.norm(b)
        got = sf.MultigridPreconditioner(hier).apply(b, lvl)
        ref = port.VCycle(H).apply(b, lvl)
        assert rel_l2(got, ref) <= 1e-10


@pytest.mark.parametrize("seed", range(6))
def test_random_slab_ghost_vmult(seed):
    """A z-slab [z0, z1) with ghost planes reproduces the rows of the full vmult (any degree, any mode)."""
    rng = np.random.default_rng(seed)
    k = int(rng.integers(1, 8))
    lvl = 3 if k < 5 else 2
    mode = [P.FP64, P.FP32, P.FP16, P.FP16_EC][int(rng.integers(0, 4))]
    hier = sf.build_hierarchy(lvl, k)
    n, K = hier.n_cells(lvl), k + 1
    plane = (n * K) ** 2
    u = torch.randn(hier.n_dofs(lvl), dtype=mode.torch_dtype, device="cuda")
    full = sf.apply_operator(hier, lvl, u, mode)
    z0 = 2 * int(rng.integers(0, n // 2))
    z1 = 2 * int(rng.integers(z0 // 2 + 1, n // 2 + 1))
    from paper_2407_09621_b200 import _native
    from paper_2407_09621_b200.discretization import vmult_device

    us = u[z0 * K * plane:z1 * K * plane].contiguous()
    glo = u[(z0 - 1) * K * plane:z0 * K * plane].contiguous() if z0 > 0 else None
    ghi = u[z1 * K * plane:(z1 + 1) * K * plane].contiguous() if z1 < n else None
    grid = _native.SfGrid(n, n, z1 - z0, glo.data_ptr() if glo is not None else None,
                          ghi.data_ptr() if ghi is not None else None)
    v = torch.empty_like(us)
    vmult_device(hier, lvl, us, v, mode, grid=grid)
    ref = full[z0 * K * plane:z1 * K * plane]
    tol = 1e-14 if mode is P.FP64 else (1e-6 if mode in (P.FP32, P.FP16_EC) else 2e-3)
    assert float((v.double() - ref.double()).norm() / ref.double().norm()) <= tol
