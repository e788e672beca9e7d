"""Drop-in backend for the reference's native plugin point (src/sumfact/_core/__init__.py:12-24).

The reference selects a module ``_impl`` exporting ``contract_f8(u3, m, out)`` and
``contract_f4(u3, m, out)`` (Cython defs over typed memoryviews ``double[:, :, ::1]`` /
``double[:, ::1]``, src/_core/_contract.pyx:14-45): out[o, i, r] = sum_k m[i, k] u3[o, k, r],
ascending k, every element of ``out`` written, ``None`` returned.  This module is that backend on
the B200: the arrays go through device memory and ``sf_contract`` (csrc/sf_contract.cu), whose
ascending-k rounded multiply-then-add is bitwise the reference's compiled kernel.  Validation
mirrors the memoryview coercion the Cython signatures perform (ValueError on a dtype, rank or
contiguity mismatch) plus the extent checks the unchecked C loop relies on its caller for.
INTEGRATION.md shows the one-line switch in the reference's ``_core/__init__.py``.
"""
from __future__ import annotations

import numpy as np
import torch

from . import _native, device


def _check(u3, m, out, dtype):
    for name, a, nd in (("u3", u3, 3), ("m", m, 2), ("out", out, 3)):
        if not isinstance(a, np.ndarray):
            raise TypeError(f"{name}: expected a numpy array")
        if a.dtype != dtype:
            raise ValueError(f"Buffer dtype mismatch, expected '{np.dtype(dtype).name}' but got "
                             f"'{a.dtype.name}' ({name})")
        if a.ndim != nd:
            raise ValueError(f"Buffer has wrong number of dimensions (expected {nd}, got {a.ndim}) ({name})")
        if not a.flags.c_contiguous:
            raise ValueError(f"ndarray is not C-contiguous ({name})")
    if not out.flags.writeable:
        raise ValueError("buffer source array is read-only (out)")
    outer, n, inner = u3.shape
    if m.shape[1] != n or out.shape != (outer, m.shape[0], inner):
        raise ValueError(f"extent mismatch: u3 {u3.shape}, m {m.shape}, out {out.shape}")


def _run(u3, m, out, dtype, mode_code):
    _check(u3, m, out, dtype)
    outer, n, inner = u3.shape
    rows = m.shape[0]
    if out.size == 0:
        return None
    device.require_cuda()
    td = torch.float64 if dtype == np.float64 else torch.float32
    ut = torch.from_numpy(u3).to("cuda", non_blocking=False).reshape(-1)
    mt = torch.from_numpy(m).to("cuda", non_blocking=False).reshape(-1)
    ot = torch.empty(out.size, dtype=td, device="cuda")
    rc = _native.lib().sf_contract(mode_code, outer, n, inner, rows, device.ptr(mt), device.ptr(ut),
                                   device.ptr(ot), device.stream_ptr())
    _native.check(rc, "sf_contract")
    out[...] = ot.cpu().numpy().reshape(out.shape)
    return None


def contract_f8(u3, m, out):
    """_contract.pyx:14-28: float64 batched contraction into ``out``."""
    return _run(u3, m, out, np.float64, 0)


def contract_f4(u3, m, out):
    """_contract.pyx:31-45: float32 batched contraction into ``out``."""
    return _run(u3, m, out, np.float32, 1)
