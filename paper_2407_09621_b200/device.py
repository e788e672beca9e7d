"""Device plumbing: torch owns memory and streams; the kernels come from libsumfact_b200.so.

Public functions accept numpy arrays (copied to the current CUDA device and
back -- the reference-facing path) or CUDA tensors (zero copy).
"""
from __future__ import annotations

import numpy as np
import torch

from . import _native


def require_cuda():
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2407_09621_b200 needs a CUDA (sm_100a) device; there is no CPU fallback")
    _native.lib()


def stream_ptr() -> int:
    return torch.cuda.current_stream().cuda_stream


def as_device(x, dtype: torch.dtype, n: int | None = None) -> tuple[torch.Tensor, bool]:
    """Return (contiguous CUDA tensor of dtype, was_host)."""
    if isinstance(x, torch.Tensor):
        if not x.is_cuda:
            t = x.detach().to(device="cuda", dtype=dtype).contiguous()
            host = True
        else:
            t = x.detach().reshape(-1)
            if t.dtype != dtype:
                t = t.to(dtype)
            t = t.contiguous()
            host = False
    else:
        arr = np.asarray(x)
        t = torch.from_numpy(np.ascontiguousarray(arr.reshape(-1))).to(device="cuda", dtype=dtype)
        host = True
    t = t.reshape(-1)
    if n is not None and t.numel() != n:
        raise ValueError(f"expected {n} entries, got {t.numel()}")
    return t, host


def to_host(t: torch.Tensor, np_dtype) -> np.ndarray:
    return t.detach().cpu().numpy().astype(np_dtype, copy=False)


def ptr(t: torch.Tensor) -> int:
    assert t.is_cuda and t.is_contiguous()
    return t.data_ptr()


class Scratch:
    """Scratch of the deterministic two-pass reductions, one per (device, stream): dots enqueued on
    different streams never share partial-sum storage."""

    _buf: dict = {}

    @classmethod
    def dot(cls) -> torch.Tensor:
        key = (torch.cuda.current_device(), torch.cuda.current_stream().cuda_stream)
        buf = cls._buf.get(key)
        if buf is None:
            buf = torch.empty(2 * _native.SF_DOT_SCRATCH, dtype=torch.float64, device="cuda")
            cls._buf[key] = buf
        return buf


def dot(x: torch.Tensor, y: torch.Tensor, out: torch.Tensor | None = None) -> torch.Tensor:
    """Deterministic fp64 dot into a 1-element device tensor (no host sync)."""
    if out is None:
        out = torch.empty(1, dtype=torch.float64, device="cuda")
    _native.check(_native.lib().sf_dot(x.numel(), ptr(x), ptr(y), out.data_ptr(), ptr(Scratch.dot()), stream_ptr()),
                  "sf_dot")
    return out


def axpy_dot(sign: float, coef: torch.Tensor, x: torch.Tensor, w: torch.Tensor, y: torch.Tensor | None,
             out: torch.Tensor) -> torch.Tensor:
    """w += sign * coef[0] * x, then out[0] = y . w (w . w when y is None) -- one pass, bitwise the separate ops."""
    _native.check(_native.lib().sf_axpy_dot(x.numel(), sign, coef.data_ptr(), ptr(x), ptr(w),
                                            ptr(y) if y is not None else None, out.data_ptr(), ptr(Scratch.dot()),
                                            stream_ptr()), "sf_axpy_dot")
    return out


def dot2(x1: torch.Tensor, x2: torch.Tensor, y: torch.Tensor, out1: torch.Tensor, out2: torch.Tensor):
    """out1[0] = x1 . y, out2[0] = x2 . y in one pass over y (each bitwise sf_dot)."""
    _native.check(_native.lib().sf_dot2(y.numel(), ptr(x1), ptr(x2), ptr(y), out1.data_ptr(), out2.data_ptr(),
                                        ptr(Scratch.dot()), stream_ptr()), "sf_dot2")


def lincomb(vecs, coefs, out: torch.Tensor) -> torch.Tensor:
    """out = sum_t coefs[t] vecs[t] in one pass (bitwise the axpby chain from zero)."""
    import ctypes

    m = len(vecs)
    P = (ctypes.c_void_p * max(m, 1))(*[ptr(v) for v in vecs])
    C = (ctypes.c_double * max(m, 1))(*[float(c) for c in coefs])
    _native.check(_native.lib().sf_lincomb(out.numel(), m, ctypes.cast(P, ctypes.c_void_p),
                                           ctypes.cast(C, ctypes.c_void_p), ptr(out), stream_ptr()), "sf_lincomb")
    return out


def axpy_dev(sign: float, coef: torch.Tensor, x: torch.Tensor, y: torch.Tensor):
    """y += sign * coef[0] * x, coef on the device."""
    _native.check(_native.lib().sf_axpy_dev(x.numel(), sign, coef.data_ptr(), ptr(x), ptr(y), stream_ptr()),
                  "sf_axpy_dev")


def axpby(alpha: float, x: torch.Tensor, beta: float, y: torch.Tensor):
    """y = alpha x + beta y (dtype of y: fp64 or fp32)."""
    L = _native.lib()
    if y.dtype == torch.float64:
        rc = L.sf_axpby(x.numel(), float(alpha), ptr(x), float(beta), ptr(y), stream_ptr())
    else:
        rc = L.sf_axpby_f32(x.numel(), float(alpha), ptr(x), float(beta), ptr(y), stream_ptr())
    _native.check(rc, "sf_axpby")


def div(x: torch.Tensor, d: float, y: torch.Tensor):
    """y = x / d (fp64, IEEE division: the reference's normalisation rounding)."""
    _native.check(_native.lib().sf_div(x.numel(), ptr(x), float(d), ptr(y), stream_ptr()), "sf_div")


def convert(src: torch.Tensor, dst: torch.Tensor):
    code = {torch.float64: 0, torch.float32: 1}
    _native.check(_native.lib().sf_convert(src.numel(), ptr(src), code[src.dtype], ptr(dst), code[dst.dtype],
                                           stream_ptr()), "sf_convert")


def dense_apply(A: torch.Tensor, x: torch.Tensor, y: torch.Tensor, demote16: bool = False):
    """y = A x (A dense fp64 n x n on the device; x, y f64 or f32; demote16 rounds x to binary16 first)."""
    code = {torch.float64: 0, torch.float32: 1}
    if A.dtype != torch.float64 or A.dim() != 2 or A.shape[0] != A.shape[1] or not A.is_contiguous():
        raise ValueError("A must be a contiguous square fp64 matrix")
    n = A.shape[0]
    if x.numel() != n or y.numel() != n:
        raise ValueError("vector lengths must match the matrix")
    _native.check(_native.lib().sf_dense_apply(n, ptr(A), ptr(x), code[x.dtype], int(demote16), ptr(y),
                                               code[y.dtype], stream_ptr()), "sf_dense_apply")
