"""The reference's native plugin point served by the B200 (paper_2407_09621_b200._impl): the
reference's own kernel tests (pkg/tests/test_kernels.py:15-72) against it, and bitwise agreement
with the reference's compiled kernel built from its sources (oracle/_ref)."""
import numpy as np
import pytest

from oracle import build_ref
from paper_2407_09621_b200 import _impl

pytestmark = pytest.mark.gpu
ref = build_ref.load()


def reference_loop(m, u3):
    """test_kernels.py:15-27: literal ascending-k accumulation."""
    outer, n, inner = u3.shape
    out = np.zeros((outer, m.shape[0], inner), dtype=u3.dtype)
    for o in range(outer):
        for i in range(m.shape[0]):
            acc = np.zeros(inner, dtype=u3.dtype)
            for k in range(n):
                acc = acc + m[i, k] * u3[o, k]
            out[o, i] = acc
    return out


@pytest.mark.parametrize("dtype", [np.float64, np.float32])
def test_matches_reference_loop_bitwise(dtype):
    rng = np.random.default_rng(0)
    u = rng.standard_normal((3, 5, 7)).astype(dtype)
    m = rng.standard_normal((4, 5)).astype(dtype)
    out = np.empty((3, 4, 7), dtype=dtype)
    kern = _impl.contract_f8 if dtype == np.float64 else _impl.contract_f4
    assert kern(u, m, out) is None
    assert np.array_equal(out, reference_loop(m, u))


@pytest.mark.skipif(ref is None, reason="oracle/_ref not built")
@pytest.mark.parametrize("dtype", [np.float64, np.float32])
@pytest.mark.parametrize("shape,rows", [((4, 8, 64), 8), ((27, 16, 256), 16), ((1, 3, 2), 5)])
def test_bitwise_the_reference_compiled_kernel(dtype, shape, rows):
    rng = np.random.default_rng(2)
    u = rng.standard_normal(shape).astype(dtype)
    m = rng.standard_normal((rows, shape[1])).astype(dtype)
    a = np.empty((shape[0], rows, shape[2]), dtype=dtype)
    b = np.full_like(a, np.nan)
    (ref.contract_f8 if dtype == np.float64 else ref.contract_f4)(u, m, a)
    (_impl.contract_f8 if dtype == np.float64 else _impl.contract_f4)(u, m, b)
    assert np.array_equal(a, b)


def test_validation_like_the_memoryview_signatures():
    u = np.zeros((2, 3, 4))
    out = np.empty((2, 3, 4))
    with pytest.raises(ValueError, match="dtype"):
        _impl.contract_f8(u.astype(np.float32), np.zeros((3, 3)), out)
    with pytest.raises(ValueError, match="dimensions"):
        _impl.contract_f8(u, np.zeros(3), out)
    with pytest.raises(ValueError, match="C-contiguous"):
        _impl.contract_f8(np.zeros((2, 4, 3)).transpose(0, 2, 1), np.zeros((3, 3)), out)
    with pytest.raises(ValueError, match="extent"):
        _impl.contract_f8(u, np.zeros((3, 5)), out)
    empty = np.empty((0, 3, 4))
    assert _impl.contract_f8(np.zeros((0, 3, 4)), np.zeros((3, 3)), empty) is None
