"""Precision modes of the hot path (mirror of src/precision.py:29-54).

The arithmetic itself lives in the CUDA kernels (csrc/sf_common.cuh): fp64
runs double throughout; fp32 single; fp16 demotes both operands of every
contraction to binary16 (round-to-nearest-even, subnormals kept) and
accumulates in fp32; fp16_ec adds the 2^11-scaled residual correction
(precision.py:206-230).  Vectors are stored in fp64 for fp64 and fp32 otherwise.
"""
from __future__ import annotations

from dataclasses import dataclass
from enum import Enum

import numpy as np

HALF_MAX = 65504.0
EC_SCALE = 2048


class HalfRangeError(ValueError):
    """precision.py:25-26 -- value cannot be represented by the main + residual half pair."""


class PrecisionMode(Enum):
    FP64 = "fp64"
    FP32 = "fp32"
    FP16 = "fp16"
    FP16_EC = "fp16_ec"

    @property
    def storage_dtype(self):
        """precision.py:36-39."""
        return np.float64 if self is PrecisionMode.FP64 else np.float32

    @property
    def accumulate_dtype(self):
        """precision.py:41-44."""
        return np.float64 if self is PrecisionMode.FP64 else np.float32

    @property
    def code(self) -> int:
        """Mode id of the C ABI (include/sumfact_b200.h)."""
        return _CODES[self]

    @property
    def torch_dtype(self):
        import torch

        return torch.float64 if self is PrecisionMode.FP64 else torch.float32

    @classmethod
    def parse(cls, name: str) -> "PrecisionMode":
        """precision.py:46-54 -- same aliases and error."""
        key = name.strip().lower().replace("-", "_")
        key = {"fp16ec": "fp16_ec", "half": "fp16", "double": "fp64", "single": "fp32"}.get(key, key)
        try:
            return cls(key)
        except ValueError:
            raise ValueError(f"unknown precision mode {name!r}") from None


_CODES = {PrecisionMode.FP64: 0, PrecisionMode.FP32: 1, PrecisionMode.FP16: 2, PrecisionMode.FP16_EC: 3}


def relative_error(v_low, v_ref) -> float:
    """precision.py:257-266 -- relative l2 distance (host arrays or tensors)."""
    v_low = np.asarray(_host(v_low), dtype=np.float64).ravel()
    v_ref = np.asarray(_host(v_ref), dtype=np.float64).ravel()
    if v_low.shape != v_ref.shape:
        raise ValueError("vectors must have equal length")
    ref_norm = float(np.linalg.norm(v_ref))
    if ref_norm == 0.0:
        raise ValueError("reference vector has zero norm")
    return float(np.linalg.norm(v_low - v_ref) / ref_norm)


def _host(x):
    if hasattr(x, "detach"):
        return x.detach().cpu().numpy()
    return x


# ------------------------------------------------- binary16 primitives on the GPU (precision.py:60-197)
# Same conversion instruction as the FP16 / FP16-EC kernels (csrc/sf_half.cu, sf_common.cuh demote16).
# numpy in -> numpy out (scalar in -> scalar out); CUDA tensors stay on the device (bit patterns as int16).


def _run(fn_name, *args):
    from . import _native, device

    _native.check(getattr(_native.lib(), fn_name)(*args, device.stream_ptr()), fn_name)


def _in(x, np_dtype, torch_dtype):
    import torch

    from . import device

    device.require_cuda()
    if isinstance(x, torch.Tensor) and x.is_cuda:
        return x.detach().reshape(-1).to(torch_dtype).contiguous(), True, x.shape
    a = np.asarray(x, dtype=np_dtype)
    scalar = a.ndim == 0
    flat = np.ascontiguousarray(a.reshape(-1))
    if np_dtype == np.uint16:
        flat = flat.view(np.int16)
    return torch.from_numpy(flat).to("cuda"), False, (None if scalar else a.shape)


def _out(t, on_device, shape, np_view=None):
    if on_device:
        return t.reshape(shape)
    a = t.cpu().numpy()
    if np_view is not None:
        a = a.view(np_view)
    return a[0] if shape is None else a.reshape(shape)


def to_half(x):
    """precision.py:60-113 -- fp32 -> binary16 bit patterns (RNE, subnormals exact, overflow -> inf, NaN -> 0x7E00|s)."""
    import torch

    t, dev, shape = _in(x, np.float32, torch.float32)
    out = torch.empty(t.numel(), dtype=torch.int16, device="cuda")
    _run("sf_to_half", t.numel(), t.data_ptr(), out.data_ptr())
    return _out(out, dev, shape, np.uint16)


def from_half(h):
    """precision.py:116-127 -- exact fp32 values of binary16 bit patterns."""
    import torch

    t, dev, shape = _in(h, np.uint16, torch.int16)
    out = torch.empty(t.numel(), dtype=torch.float32, device="cuda")
    _run("sf_from_half", t.numel(), t.data_ptr(), out.data_ptr())
    return _out(out, dev, shape)


def demote16(x):
    """precision.py:130-137 -- round fp32 through binary16, back as fp32 (out-of-range -> inf)."""
    import torch

    t, dev, shape = _in(x, np.float32, torch.float32)
    out = torch.empty_like(t)
    _run("sf_demote16", t.numel(), t.data_ptr(), out.data_ptr())
    return _out(out, dev, shape if shape is not None else ())


@dataclass
class EcPair:
    """precision.py:143-154 -- main half plus 2^11-scaled residual half (uint16 bit patterns)."""

    main: np.ndarray
    residual: np.ndarray
    scale: int = EC_SCALE

    def reconstruct(self):
        m = from_half(self.main)
        r = from_half(self.residual)
        return m + r / np.float32(self.scale)


def ec_split(x) -> EcPair:
    """precision.py:157-167 -- HalfRangeError for non-finite or |x| > 65504."""
    import torch

    t, dev, shape = _in(x, np.float32, torch.float32)
    n = t.numel()
    hm = torch.empty(n, dtype=torch.int16, device="cuda")
    hr = torch.empty(n, dtype=torch.int16, device="cuda")
    flag = torch.zeros(1, dtype=torch.int32, device="cuda")
    _run("sf_ec_split", n, t.data_ptr(), hm.data_ptr(), hr.data_ptr(), flag.data_ptr())
    if int(flag.item()):
        raise HalfRangeError("values outside the correctable half range")
    if dev:
        return EcPair(main=hm.reshape(shape), residual=hr.reshape(shape))
    shp = (1,) if shape is None else shape  # np.atleast_1d, as the reference
    return EcPair(main=hm.cpu().numpy().view(np.uint16).reshape(shp), residual=hr.cpu().numpy().view(np.uint16).reshape(shp))


def ec_matmul(A: EcPair, B: EcPair, refine: str = "both"):
    """precision.py:170-197 -- residual-corrected product with fp32 accumulation."""
    import torch

    codes = {"both": 0, "left": 1, "right": 2}
    if refine not in codes:
        raise ValueError(f"unknown refinement choice {refine!r}")
    parts = []
    for arr in (A.main, A.residual, B.main, B.residual):
        t, dev, shape = _in(arr, np.uint16, torch.int16)
        parts.append((t, shape if shape is not None else ()))
    (am, sa), (ar, _), (bm, sb), (br, _) = parts
    if len(sa) != 2 or len(sb) != 2 or sa[-1] != sb[0]:
        raise ValueError(f"shape mismatch: {tuple(sa)} @ {tuple(sb)}")
    m, k, n = sa[0], sa[1], sb[1]
    out = torch.empty(m * n, dtype=torch.float32, device="cuda")
    _run("sf_ec_matmul", m, k, n, am.data_ptr(), ar.data_ptr(), bm.data_ptr(), br.data_ptr(), codes[refine],
         out.data_ptr())
    on_dev = isinstance(A.main, torch.Tensor) and A.main.is_cuda
    return out.reshape(m, n) if on_dev else out.cpu().numpy().reshape(m, n)
