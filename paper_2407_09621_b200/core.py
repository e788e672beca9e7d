"""Batched 1-D contraction on the GPU: the reference's native plugin point.

Mirror of src/_core/__init__.py:27-59 (``contract_batch``) and src/precision.py:206-230
(``contract_mode``) with the arithmetic in ``sf_contract`` (csrc/sf_contract.cu): ascending-k,
rounded multiply then add -- bitwise the reference's compiled ``contract_f8`` / ``contract_f4``
-- and the per-operand demotion of the low-precision modes.  numpy in -> numpy out (through the
device); CUDA tensor in -> CUDA tensor out.  The operator/solver hot path does not go through
this call (it is fused into the tile kernels); it is the drop-in for code that uses the
reference's contraction API directly.
"""
from __future__ import annotations

import numpy as np
import torch

from . import _native, device
from .precision import PrecisionMode

_TORCH_OF = {np.dtype(np.float64): torch.float64, np.dtype(np.float32): torch.float32}


def _dtype_of(x):
    return np.dtype(str(x.dtype).replace("torch.", "")) if isinstance(x, torch.Tensor) else np.asarray(x).dtype


def _contract(mode_code: int, m, u, axis: int, out_dtype):
    host = not (isinstance(u, torch.Tensor) and u.is_cuda)
    shape = tuple(u.shape)
    outer = int(np.prod(shape[:axis], dtype=np.int64))
    inner = int(np.prod(shape[axis + 1:], dtype=np.int64))
    n, rows = shape[axis], int(m.shape[0])
    td = _TORCH_OF[np.dtype(out_dtype)]
    device.require_cuda()
    ut, _ = device.as_device(u, td)
    mt, _ = device.as_device(m, td)
    out = torch.empty(outer * rows * inner, dtype=td, device="cuda")
    rc = _native.lib().sf_contract(mode_code, outer, n, inner, rows, device.ptr(mt), device.ptr(ut), device.ptr(out),
                                   device.stream_ptr())
    _native.check(rc, "sf_contract")
    out_shape = shape[:axis] + (rows,) + shape[axis + 1:]
    out = out.reshape(out_shape)
    return device.to_host(out, out_dtype) if host else out


def contract_batch(m, u, axis: int):
    """out[..., i, ...] = sum_k m[i, k] * u[..., k, ...] along numpy ``axis`` (_core/__init__.py:27-59).

    Same validation and exceptions as the reference: dtype mismatch -> TypeError, m not 2-D ->
    ValueError, axis out of range -> IndexError, extent mismatch -> ValueError, dtype other than
    float32/float64 -> TypeError.
    """
    md, ud = _dtype_of(m), _dtype_of(u)
    if md != ud:
        raise TypeError(f"dtype mismatch: {md} vs {ud}")
    if len(m.shape) != 2:
        raise ValueError("matrix operand must be 2-dimensional")
    axis = int(axis)
    if not 0 <= axis < len(u.shape):
        raise IndexError(f"axis {axis} out of range for {len(u.shape)}-d operand")
    if m.shape[1] != u.shape[axis]:
        raise ValueError(f"cannot contract axis of extent {u.shape[axis]} with {m.shape[0]}x{m.shape[1]} matrix")
    if ud == np.float64:
        return _contract(0, m, u, axis, np.float64)
    if ud == np.float32:
        return _contract(1, m, u, axis, np.float32)
    raise TypeError(f"unsupported dtype {ud}")


def contract_mode(m, u, axis: int, mode: PrecisionMode):
    """Contract ``axis`` of ``u`` with ``m`` under a precision mode (precision.py:206-230)."""
    if mode is PrecisionMode.FP64:
        return contract_batch(np.asarray(m, dtype=np.float64) if not isinstance(m, torch.Tensor) else m.double(),
                              np.asarray(u, dtype=np.float64) if not isinstance(u, torch.Tensor) else u.double(), axis)
    m32 = np.asarray(m, dtype=np.float32) if not isinstance(m, torch.Tensor) else m.float()
    u32 = np.asarray(u, dtype=np.float32) if not isinstance(u, torch.Tensor) else u.float()
    if mode is PrecisionMode.FP32:
        return contract_batch(m32, u32, axis)
    if mode in (PrecisionMode.FP16, PrecisionMode.FP16_EC):
        axis = int(axis)
        if not 0 <= axis < len(u32.shape):
            raise IndexError(f"axis {axis} out of range for {len(u32.shape)}-d operand")
        if len(m32.shape) != 2 or m32.shape[1] != u32.shape[axis]:
            raise ValueError("matrix/operand extents do not match")
        return _contract(mode.code, m32, u32, axis, np.float32)
    raise ValueError(f"unsupported mode {mode}")
