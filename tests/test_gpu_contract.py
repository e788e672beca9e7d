"""contract_batch / contract_mode on the GPU vs the reference's compiled kernel semantics
(tests/test_kernels.py:15-95 of the reference: literal ascending-k loop, backend agreement on
(4,8,64)/(27,16,256)/(1,3,2), validation exceptions, arbitrary axis)."""
import numpy as np
import pytest
import torch

import paper_2407_09621_b200 as sf
from oracle import build_ref

pytestmark = pytest.mark.gpu
P = sf.PrecisionMode


def literal(m, u3):
    """contract_f8/f4 exactly: out = 0; out += m[i,k] * u[o,k,r] for ascending k (mul, then add)."""
    out = np.zeros((u3.shape[0], m.shape[0], u3.shape[2]), dtype=u3.dtype)
    for k in range(m.shape[1]):
        out = out + m[None, :, k, None] * u3[:, None, k, :]
    return out


@pytest.mark.parametrize("shape", [(4, 8, 64), (27, 16, 256), (1, 3, 2), (7, 5, 1)])
@pytest.mark.parametrize("dtype", [np.float64, np.float32])
def test_bitwise_literal_loop(shape, dtype):
    rng = np.random.default_rng(3)
    u = rng.standard_normal(shape).astype(dtype)
    m = rng.standard_normal((6, shape[1])).astype(dtype)
    got = sf.contract_batch(m, u, 1)
    assert got.dtype == dtype and got.shape == (shape[0], 6, shape[2])
    assert np.array_equal(got, literal(m, u))


def test_matches_reference_compiled_kernel():
    ref = build_ref.load()
    if ref is None:
        pytest.skip("oracle/_ref not built")
    rng = np.random.default_rng(9)
    for dtype, fn in ((np.float64, ref.contract_f8), (np.float32, ref.contract_f4)):
        u = rng.standard_normal((27, 16, 256)).astype(dtype)
        m = rng.standard_normal((16, 16)).astype(dtype)
        out = np.empty((27, 16, 256), dtype=dtype)
        fn(u, m, out)
        assert np.array_equal(sf.contract_batch(m, u, 1), out)


@pytest.mark.parametrize("axis", [0, 1, 2, 3])
def test_arbitrary_axis_and_tensor_io(axis):
    rng = np.random.default_rng(axis)
    u = rng.standard_normal((3, 4, 5, 6))
    m = rng.standard_normal((2, u.shape[axis]))
    ref = np.moveaxis(np.tensordot(m, u, axes=([1], [axis])), 0, axis)
    got = sf.contract_batch(m, u, axis)
    assert np.allclose(got, ref, rtol=1e-14, atol=1e-14)
    gt = sf.contract_batch(torch.from_numpy(m).cuda(), torch.from_numpy(u).cuda(), axis)
    assert gt.is_cuda and np.array_equal(gt.cpu().numpy(), got)


def test_validation_exceptions():
    u = np.zeros((2, 3, 4))
    with pytest.raises(TypeError):
        sf.contract_batch(np.zeros((3, 3), np.float32), u, 1)
    with pytest.raises(ValueError):
        sf.contract_batch(np.zeros(3), u, 1)
    with pytest.raises(IndexError):
        sf.contract_batch(np.zeros((3, 3)), u, 3)
    with pytest.raises(ValueError):
        sf.contract_batch(np.zeros((3, 4)), u, 1)
    with pytest.raises(TypeError):
        sf.contract_batch(np.zeros((3, 3), np.int64), u.astype(np.int64), 1)


def _demote(x):
    return x.astype(np.float16).astype(np.float32)


@pytest.mark.parametrize("mode", [P.FP16, P.FP16_EC, P.FP32])
def test_contract_mode_semantics_bitwise(mode):
    """precision.py:206-230 restated with the literal loop: bitwise equal."""
    rng = np.random.default_rng(1)
    u = rng.standard_normal((5, 16, 33)).astype(np.float32) * 3
    m = rng.standard_normal((16, 16)).astype(np.float32)
    got = sf.contract_mode(m, u, 1, mode)
    if mode is P.FP32:
        ref = literal(m, u)
    elif mode is P.FP16:
        ref = literal(_demote(m), _demote(u))
    else:
        mh, uh = _demote(m), _demote(u)
        dm = ((m - mh) * np.float32(2048)).astype(np.float16).astype(np.float32)
        du = ((u - uh) * np.float32(2048)).astype(np.float16).astype(np.float32)
        ref = literal(mh, uh) + (literal(dm, uh) + literal(mh, du)) / np.float32(2048)
    assert got.dtype == np.float32
    assert np.array_equal(got, ref)
    # error ordering of the reference's precision bands
    exact = np.moveaxis(np.tensordot(m.astype(np.float64), u.astype(np.float64), axes=([1], [1])), 0, 1)
    err = np.linalg.norm(got - exact) / np.linalg.norm(exact)
    assert err < {P.FP32: 1e-6, P.FP16: 5e-3, P.FP16_EC: 1e-6}[mode]
