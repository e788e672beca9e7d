"""Bitwise reproducibility of every kernel in every precision mode (the reference's promise of
bit-identical repeated runs, SPEC.md:116 / pkg/tests/test_multigrid.py:120-125): repeated vmults, colour
passes, V-cycles and solves on the same input must agree bit for bit.  The sizes are those at which a
block-exponent race of the binary16 kernels once showed (a few entries 1 ulp apart, ~1 run in 2)."""
import pytest
import torch

import paper_2407_09621_b200 as sf
from paper_2407_09621_b200.discretization import vmult_device

pytestmark = pytest.mark.gpu
P = sf.PrecisionMode
MODES = [P.FP64, P.FP32, P.FP16, P.FP16_EC]


@pytest.mark.parametrize("k,lvl", [(7, 5), (3, 6), (1, 7), (2, 4)])
def test_vmult_bitwise_reproducible(k, lvl):
    hier = sf.build_hierarchy(lvl, k, max_dofs=2**34, min_level=lvl)
    n = hier.n_dofs(lvl)
    u = torch.randn(n, dtype=torch.float64, device="cuda", generator=torch.Generator(device="cuda").manual_seed(5))
    for m in MODES:
        ui = u.to(m.torch_dtype)
        outs = []
        for _ in range(4):
            v = torch.empty(n, dtype=m.torch_dtype, device="cuda")
            vmult_device(hier, lvl, ui, v, m)
            outs.append(v)
        for o in outs[1:]:
            assert torch.equal(o, outs[0]), (k, lvl, m, int((o != outs[0]).sum()))


@pytest.mark.parametrize("k,lvl", [(7, 4), (3, 5), (1, 6)])
def test_smoother_and_vcycle_bitwise_reproducible(k, lvl):
    hier = sf.build_hierarchy(lvl, k)
    n = hier.n_dofs(lvl)
    g = torch.Generator(device="cuda").manual_seed(6)
    b = torch.randn(n, dtype=torch.float64, device="cuda", generator=g)
    x = torch.randn(n, dtype=torch.float64, device="cuda", generator=g)
    for m in MODES:
        mg = sf.MultigridPreconditioner(hier, sf.VCycleConfig(mode=m))
        s = [mg.smooth(lvl, x.to(m.torch_dtype), b.to(m.torch_dtype)) for _ in range(3)]
        z = [mg.apply(b, lvl) for _ in range(3)]
        for t in s[1:]:
            assert torch.equal(t, s[0]), (k, lvl, m, "smooth")
        for t in z[1:]:
            assert torch.equal(t, z[0]), (k, lvl, m, "vcycle")


@pytest.mark.parametrize("mode", [P.FP64, P.FP16_EC])
def test_solve_bitwise_reproducible(mode):
    a = sf.run_solve(3, 5, mode, keep_solution=True)
    b = sf.run_solve(3, 5, mode, keep_solution=True)
    assert a.report.residual_history == b.report.residual_history
    assert torch.equal(torch.as_tensor(a.x), torch.as_tensor(b.x))


@pytest.mark.parametrize("k,lvl", [(7, 4), (3, 5), (1, 6), (2, 3)])
def test_zero_iterate_colour_pass_is_bitwise_the_full_pass(k, lvl):
    """sf_smooth_colour with x_old = NULL (the V-cycle's first unshifted colour on a zero iterate) against the
    full pass on an explicit zero vector; degree 2 has no tensor-core colour kernel and reports
    SF_EUNSUPPORTED, shifted colours are SF_EINVAL."""
    import ctypes

    from paper_2407_09621_b200 import _native, device

    hier = sf.build_hierarchy(lvl, k)
    n = hier.n_dofs(lvl)
    L = _native.lib()
    lm = hier.matrices(lvl)
    b = torch.randn(n, dtype=torch.float64, device="cuda", generator=torch.Generator(device="cuda").manual_seed(8))
    for m in MODES:
        mg = sf.MultigridPreconditioner(hier, sf.VCycleConfig(mode=m))
        table = mg.solvers[lvl].table
        bs = b.to(m.torch_dtype)
        zero = torch.zeros(n, dtype=m.torch_dtype, device="cuda")
        full = torch.empty_like(zero)
        fast = torch.full_like(zero, float("nan"))
        s0 = (ctypes.c_int * 3)(0, 0, 0)
        args = (m.code, k, hier.grid(lvl), s0, _native.host_ptr(lm.cell_op), _native.host_ptr(table))
        _native.check(L.sf_smooth_colour(*args, device.ptr(zero), device.ptr(bs), device.ptr(full), device.stream_ptr()),
                      "sf_smooth_colour")
        rc = L.sf_smooth_colour(*args, None, device.ptr(bs), device.ptr(fast), device.stream_ptr())
        if k == 2:
            assert rc == _native.SF_EUNSUPPORTED
            continue
        assert rc == 0
        torch.cuda.synchronize()
        assert torch.equal(fast, full), (k, lvl, m)
        s1 = (ctypes.c_int * 3)(1, 0, 0)
        assert L.sf_smooth_colour(m.code, k, hier.grid(lvl), s1, _native.host_ptr(lm.cell_op),
                                  _native.host_ptr(table), None, device.ptr(bs), device.ptr(fast),
                                  device.stream_ptr()) == _native.SF_EINVAL
