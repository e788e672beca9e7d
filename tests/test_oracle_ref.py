"""Pin the oracle's contraction to the reference's own compiled kernel (oracle/_ref).

The reference's native plugin is ``contract_f8/contract_f4`` (src/sumfact/_core/_contract.pyx:14-45):
out[o,i,r] = sum_k m[i,k] u[o,k,r], ascending k.  oracle/build_ref.py compiles it from the
reference's sources; these tests check oracle.port.contract against it on the operator shapes
(tests/test_kernels.py:57-72 of the reference uses the same shapes).
"""
import numpy as np
import pytest

from oracle import build_ref, port

ref = build_ref.load() or (build_ref.build() and build_ref.load())
pytestmark = pytest.mark.skipif(ref is None, reason="oracle/_ref not built and /root/reference absent")


def _ref_contract(m, w, axis):
    """contract_batch's reshape (src/sumfact/_core/__init__.py:46-58) around the compiled kernel."""
    w = np.ascontiguousarray(w)
    outer = int(np.prod(w.shape[:axis], dtype=np.int64))
    inner = int(np.prod(w.shape[axis + 1:], dtype=np.int64))
    u3 = w.reshape(outer, w.shape[axis], inner)
    out = np.empty((outer, m.shape[0], inner), dtype=w.dtype)
    (ref.contract_f8 if w.dtype == np.float64 else ref.contract_f4)(u3, np.ascontiguousarray(m), out)
    shape = list(w.shape)
    shape[axis] = m.shape[0]
    return out.reshape(shape)


@pytest.mark.parametrize("shape,axis", [((4, 8, 64), 1), ((27, 16, 256), 1), ((1, 3, 2), 1),
                                        ((2, 2, 2, 16, 16, 16), 5), ((2, 2, 2, 16, 16, 16), 4),
                                        ((2, 2, 2, 16, 16, 16), 3), ((3, 3, 3, 8, 8, 8), 3)])
@pytest.mark.parametrize("dtype,tol", [(np.float64, 1e-14), (np.float32, 1e-5)])
def test_port_contract_matches_reference_kernel(shape, axis, dtype, tol):
    rng = np.random.default_rng(7)
    w = rng.standard_normal(shape).astype(dtype)
    m = rng.standard_normal((shape[axis], shape[axis])).astype(dtype)
    a = port.contract(m, w, axis)
    b = _ref_contract(m, w, axis)
    assert a.dtype == b.dtype
    assert np.max(np.abs(a - b)) <= tol * max(1.0, float(np.max(np.abs(b))))


def test_reference_kernel_is_the_ascending_k_loop():
    rng = np.random.default_rng(3)
    u = rng.standard_normal((3, 5, 4))
    m = rng.standard_normal((6, 5))
    out = np.empty((3, 6, 4))
    ref.contract_f8(u, m, out)
    lit = np.zeros_like(out)
    for o in range(3):
        for i in range(6):
            for k in range(5):
                lit[o, i] += m[i, k] * u[o, k]
    assert np.array_equal(out, lit)
