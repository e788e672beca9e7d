"""Precision modes of the hot path (mirror of src/precision.py:29-54).

The arithmetic itself lives in the CUDA kernels (csrc/sf_common.cuh): fp64
runs double throughout; fp32 single; fp16 demotes both operands of every
contraction to binary16 (round-to-nearest-even, subnormals kept) and
accumulates in fp32; fp16_ec adds the 2^11-scaled residual correction
(precision.py:206-230).  Vectors are stored in fp64 for fp64 and fp32 otherwise.
"""
from __future__ import annotations

from enum import Enum

import numpy as np

HALF_MAX = 65504.0
EC_SCALE = 2048


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
