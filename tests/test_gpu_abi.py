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
