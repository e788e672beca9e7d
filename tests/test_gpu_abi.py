"""C-ABI error paths and edge cases with device memory (the reference's validation behaviour: bad
arguments raise ValueError / NotImplementedError through the Python mirror; empty work is a no-op)."""
import ctypes

import numpy as np
import pytest
import torch

import paper_2407_09621_b200 as sf
from paper_2407_09621_b200 import _native, device

pytestmark = pytest.mark.gpu
L = _native.lib()


def _ptr(t):
    return ctypes.c_void_p(t.data_ptr())


def test_vmult_zrange_validation_and_equivalence():
    hier = sf.build_hierarchy(3, 7)
    n, D = hier.n_cells(3), hier.n_dofs(3)
    u = torch.randn(D, dtype=torch.float64, device="cuda")
    full = sf.apply_operator(hier, 3, u)
    v = torch.zeros_like(u)
    grid = hier.grid(3)
    op = _native.host_ptr(hier.matrices(3).cell_op)
    for z0, z1 in ((0, 2), (2, n - 2), (n - 2, n)):  # the three layers cover the array
        assert L.sf_vmult_zrange(0, 7, grid, z0, z1, op, _ptr(u), _ptr(v), device.stream_ptr()) == 0
    assert torch.equal(v, full)
    for z0, z1 in ((1, 4), (0, n + 2), (4, 4), (-2, 2)):
        rc = L.sf_vmult_zrange(0, 7, grid, z0, z1, op, _ptr(u), _ptr(v), device.stream_ptr())
        assert rc == _native.SF_EINVAL


def test_bad_arguments_raise_like_the_reference():
    hier = sf.build_hierarchy(2, 3)
    with pytest.raises(ValueError):
        sf.apply_operator(hier, 2, np.zeros(hier.n_dofs(2) + 1))
    with pytest.raises(ValueError):  # odd cell counts are rejected by the library
        _native.check(L.sf_vmult(0, 3, _native.SfGrid(3, 4, 4, None, None), _native.host_ptr(hier.matrices(2).cell_op),
                                 ctypes.c_void_p(1), ctypes.c_void_p(1), 1, device.stream_ptr()), "sf_vmult")
    with pytest.raises(NotImplementedError):
        _native.check(L.sf_vmult(0, 9, hier.grid(2), _native.host_ptr(hier.matrices(2).cell_op),
                                 ctypes.c_void_p(1), ctypes.c_void_p(1), 1, device.stream_ptr()), "sf_vmult")
    with pytest.raises(ValueError):
        _native.check(L.sf_vmult(7, 3, hier.grid(2), _native.host_ptr(hier.matrices(2).cell_op),
                                 ctypes.c_void_p(1), ctypes.c_void_p(1), 1, device.stream_ptr()), "sf_vmult")


def test_empty_work_is_a_no_op():
    z = torch.zeros(4, dtype=torch.float64, device="cuda")
    assert L.sf_contract(0, 0, 4, 3, 2, _ptr(z), _ptr(z), _ptr(z), device.stream_ptr()) == 0
    assert L.sf_axpby(0, 1.0, None, 0.0, None, device.stream_ptr()) == 0
    out = torch.empty(1, dtype=torch.float64, device="cuda")
    device.dot(z[:0], z[:0], out)
    assert float(out) == 0.0


def test_batched_vmult_equals_single_vmults():
    hier = sf.build_hierarchy(2, 7)
    D = hier.n_dofs(2)
    U = torch.randn(5, D, dtype=torch.float64, device="cuda")
    V = torch.empty_like(U)
    from paper_2407_09621_b200.discretization import vmult_device

    vmult_device(hier, 2, U, V, sf.PrecisionMode.FP64, batch=5)
    for i in range(5):
        assert torch.equal(V[i], sf.apply_operator(hier, 2, U[i].contiguous()))


def _chain(vecs, coefs, n):
    out = torch.zeros(n, dtype=torch.float64, device="cuda")
    for v, c in zip(vecs, coefs):
        device.axpby(float(c), v, 1.0, out)
    return out


@pytest.mark.parametrize("m", [0, 1, 7, _native.SF_LINCOMB_MAX_TERMS])
def test_lincomb_is_bitwise_the_axpby_chain(m):
    n = 100_003
    g = torch.Generator(device="cuda")
    g.manual_seed(m)
    vecs = [torch.randn(n, dtype=torch.float64, device="cuda", generator=g) for _ in range(m)]
    coefs = np.random.default_rng(m).standard_normal(m)
    out = torch.full((n,), 7.0, dtype=torch.float64, device="cuda")
    device.lincomb(vecs, coefs, out)
    assert torch.equal(out, _chain(vecs, coefs, n))  # m = 0 writes zeros


def test_lincomb_rejects_more_terms_than_the_limit():
    n = 64
    vecs = [torch.ones(n, dtype=torch.float64, device="cuda")] * (_native.SF_LINCOMB_MAX_TERMS + 1)
    with pytest.raises(ValueError, match="term count"):
        device.lincomb(vecs, np.ones(len(vecs)), torch.empty(n, dtype=torch.float64, device="cuda"))


def test_axpy_dot_norm_form_and_dot2_are_bitwise_the_separate_ops():
    n = 300_001
    x, w, y = (torch.randn(n, dtype=torch.float64, device="cuda") for _ in range(3))
    coef = torch.tensor([0.37], dtype=torch.float64, device="cuda")
    for yy in (y, None):
        w1, w2 = w.clone(), w.clone()
        o1 = torch.empty(1, dtype=torch.float64, device="cuda")
        o2 = torch.empty(1, dtype=torch.float64, device="cuda")
        device.axpy_dot(-1.0, coef, x, w1, yy, o1)
        device.axpy_dev(-1.0, coef, x, w2)
        device.dot(yy if yy is not None else w2, w2, o2)
        assert torch.equal(w1, w2) and torch.equal(o1, o2)
    a1, a2, b1, b2 = (torch.empty(1, dtype=torch.float64, device="cuda") for _ in range(4))
    device.dot2(x, w, y, a1, a2)
    device.dot(x, y, b1)
    device.dot(w, y, b2)
    assert torch.equal(a1, b1) and torch.equal(a2, b2)


def test_div_rounds_like_the_reference_division():
    x = torch.randn(10_007, dtype=torch.float64, device="cuda")
    y = torch.empty_like(x)
    d = 3.000000000000001
    device.div(x, d, y)
    assert np.array_equal(y.cpu().numpy(), x.cpu().numpy() / d)  # numpy's IEEE division, bitwise


def test_krylov_solution_update_fallback_beyond_the_lincomb_limit(monkeypatch):
    """m > SF_LINCOMB_MAX_TERMS takes the axpby chain; with a lowered limit the two paths agree bitwise."""
    from paper_2407_09621_b200 import krylov

    rng = np.random.default_rng(5)
    Q, _ = np.linalg.qr(rng.standard_normal((60, 60)))
    A = Q @ np.diag(np.geomspace(1, 1e3, 60)) @ Q.T
    b = rng.standard_normal(60)
    At = torch.from_numpy(A).cuda()
    apply = lambda v: At @ v
    bt = torch.from_numpy(b).cuda()
    x1, r1 = sf.fgmres(apply, None, bt, tol=1e-12, maxit=60)
    monkeypatch.setattr(_native, "SF_LINCOMB_MAX_TERMS", 3)
    x2, r2 = sf.fgmres(apply, None, bt, tol=1e-12, maxit=60)
    assert r1.iterations == r2.iterations > 3
    assert torch.equal(x1, x2)


@pytest.mark.parametrize("solver", ["fgmres", "gmres"])
def test_fused_mgs_toggle_is_bitwise_for_both_solvers(monkeypatch, solver):
    from paper_2407_09621_b200 import krylov

    hier = sf.build_hierarchy(3, 3)
    mg = sf.MultigridPreconditioner(hier)
    b = torch.randn(hier.n_dofs(3), dtype=torch.float64, device="cuda")
    A = lambda v: sf.apply_operator(hier, 3, v)
    M = lambda v: mg.apply(v, 3)
    run = getattr(sf, solver)
    xa, ra = run(A, M, b, tol=1e-9, maxit=30)
    monkeypatch.setattr(krylov, "FUSED_MGS", False)
    xb, rb = run(A, M, b, tol=1e-9, maxit=30)
    assert ra.iterations == rb.iterations
    assert ra.residual_history == rb.residual_history
    assert torch.equal(xa, xb)


@pytest.mark.parametrize("xd,yd,dem", [(torch.float64, torch.float64, False), (torch.float32, torch.float32, False),
                                       (torch.float32, torch.float32, True), (torch.float64, torch.float32, False),
                                       (torch.float32, torch.float64, False)])
def test_dense_apply_matches_matmul(xd, yd, dem):
    """The coarse solve's product with the explicit inverse (sf_dense_apply) against an fp64 matmul."""
    from paper_2407_09621_b200 import device

    g = torch.Generator(device="cuda").manual_seed(3)
    for n in (1, 37, 512, 4096):
        A = torch.randn(n, n, dtype=torch.float64, device="cuda", generator=g)
        x = torch.randn(n, dtype=torch.float64, device="cuda", generator=g).to(xd)
        y = torch.empty(n, dtype=yd, device="cuda")
        device.dense_apply(A, x, y, demote16=dem)
        xr = x.float().half().double() if dem else x.double()
        ref = A @ xr
        tol = 1e-13 if yd == torch.float64 else 2e-7
        assert ((y.double() - ref).abs().max() / ref.abs().max()).item() <= tol, (n, xd, yd, dem)
        y2 = torch.empty_like(y)
        device.dense_apply(A, x, y2, demote16=dem)
        assert torch.equal(y, y2)  # deterministic


def test_coarse_solve_uses_the_inverse_kernel():
    import paper_2407_09621_b200 as sf

    hier = sf.build_hierarchy(2, 3)
    mg = sf.MultigridPreconditioner(hier).setup()
    assert mg._coarse_factor(sf.PrecisionMode.FP64)[0] == "inverse"
    A = mg._coarse_matrix()
    b = torch.randn(A.shape[0], dtype=torch.float64, device="cuda")
    x = mg.coarse_solve(b)
    assert (torch.linalg.norm(A @ x - b) / torch.linalg.norm(b)).item() <= 1e-12
