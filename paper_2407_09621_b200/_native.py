"""ctypes binding of libsumfact_b200.so (the C ABI in include/sumfact_b200.h).

There is no fallback: importing the product package on a machine without the
built library, or calling a kernel without a CUDA device, raises.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libsumfact_b200.so")

SF_OK = 0
SF_EINVAL = -1
SF_EUNSUPPORTED = -2
SF_ECUDA = -3
SF_DOT_SCRATCH = 1024
SF_LINCOMB_MAX_TERMS = 128  # include/sumfact_b200.h
ABI_VERSION = 5
MAX_DEGREE = 7


class NativeError(RuntimeError):
    """A CUDA-side failure reported by the library (SF_ECUDA)."""


class SfGrid(ctypes.Structure):
    _fields_ = [("nx", ctypes.c_int), ("ny", ctypes.c_int), ("nz", ctypes.c_int),
                ("ghost_lo", ctypes.c_void_p), ("ghost_hi", ctypes.c_void_p)]


_lib = None


def lib():
    """Load the library once; raise ImportError with the build hint when missing."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: run `python -m paper_2407_09621_b200.build` "
                              "(there is no CPU fallback)")
        L = ctypes.CDLL(LIB_PATH)
        c_i, c_ll, c_p, c_d, c_f = ctypes.c_int, ctypes.c_longlong, ctypes.c_void_p, ctypes.c_double, ctypes.c_float
        P_grid = ctypes.POINTER(SfGrid)
        sigs = {
            "sf_abi_version": ([], c_i),
            "sf_last_error": ([], ctypes.c_char_p),
            "sf_vec_last_error": ([], ctypes.c_char_p),
            "sf_vmult": ([c_i, c_i, P_grid, c_p, c_p, c_p, c_i, c_p], c_i),
            "sf_vmult_zrange": ([c_i, c_i, P_grid, c_i, c_i, c_p, c_p, c_p, c_p], c_i),
            "sf_smooth_colour": ([c_i, c_i, P_grid, c_p, c_p, c_p, c_p, c_p, c_p, c_p], c_i),
            "sf_smooth_colour_zrange": ([c_i, c_i, P_grid, c_p, c_i, c_i, c_p, c_p, c_p, c_p, c_p, c_p], c_i),
            "sf_copy_uncovered": ([c_i, c_i, P_grid, c_p, c_p, c_p, c_p], c_i),
            "sf_residual_restrict": ([c_i, c_i, P_grid, c_p, c_p, c_p, c_p, c_p, c_p], c_i),
            "sf_prolongate_add": ([c_i, c_i, P_grid, c_p, c_p, c_p, c_p], c_i),
            "sf_patch_apply": ([c_i, c_i, c_ll, c_p, c_p, c_p, c_p, c_p], c_i),
            "sf_convert": ([c_ll, c_p, c_i, c_p, c_i, c_p], c_i),
            "sf_dot": ([c_ll, c_p, c_p, c_p, c_p, c_p], c_i),
            "sf_axpy_dev": ([c_ll, c_d, c_p, c_p, c_p, c_p], c_i),
            "sf_axpy_dot": ([c_ll, c_d, c_p, c_p, c_p, c_p, c_p, c_p, c_p], c_i),
            "sf_dot2": ([c_ll, c_p, c_p, c_p, c_p, c_p, c_p, c_p], c_i),
            "sf_lincomb": ([c_ll, c_i, c_p, c_p, c_p, c_p], c_i),
            "sf_axpby": ([c_ll, c_d, c_p, c_d, c_p, c_p], c_i),
            "sf_div": ([c_ll, c_p, c_d, c_p, c_p], c_i),
            "sf_axpby_f32": ([c_ll, c_f, c_p, c_f, c_p, c_p], c_i),
            "sf_dense_apply": ([c_ll, c_p, c_p, c_i, c_i, c_p, c_i, c_p], c_i),
            "sf_contract": ([c_i, c_ll, c_i, c_ll, c_i, c_p, c_p, c_p, c_p], c_i),
            "sf_contract_last_error": ([], ctypes.c_char_p),
            "sf_half_last_error": ([], ctypes.c_char_p),
            "sf_to_half": ([c_ll, c_p, c_p, c_p], c_i),
            "sf_from_half": ([c_ll, c_p, c_p, c_p], c_i),
            "sf_demote16": ([c_ll, c_p, c_p, c_p], c_i),
            "sf_ec_split": ([c_ll, c_p, c_p, c_p, c_p, c_p], c_i),
            "sf_ec_matmul": ([c_i, c_i, c_i, c_p, c_p, c_p, c_p, c_i, c_p, c_p], c_i),
            "sf_quad_error": ([c_i, c_i, c_i, c_i, c_i, c_p, c_p, c_p, c_p, c_p, c_p, c_p], c_i),
            "sf_quad_load": ([c_i, c_i, c_i, c_i, c_i, c_p, c_p, c_p, c_p, c_p], c_i),
            "sf_face_load": ([c_i, c_i, c_i, c_i, c_i, c_i, c_i, c_p, c_p, c_p, c_p, c_p, c_p], c_i),
            "sf_quad_last_error": ([], ctypes.c_char_p),
        }
        try:
            version = L.sf_abi_version()
            for name, (args, res) in sigs.items():
                fn = getattr(L, name)
                fn.argtypes = args
                fn.restype = res
        except AttributeError as e:  # a library built before an entry point was added
            raise ImportError(f"libsumfact_b200.so ABI mismatch ({e}); rebuild") from e
        if version != ABI_VERSION:
            raise ImportError(f"libsumfact_b200.so ABI {version} != {ABI_VERSION}; rebuild")
        _lib = L
    return _lib


EXPORTED = ("sf_abi_version", "sf_last_error", "sf_vmult", "sf_vmult_zrange", "sf_smooth_colour", "sf_residual_restrict",
            "sf_prolongate_add", "sf_patch_apply", "sf_convert", "sf_dot", "sf_axpy_dev", "sf_axpby", "sf_axpby_f32",
            "sf_contract", "sf_to_half", "sf_from_half", "sf_demote16", "sf_ec_split", "sf_ec_matmul", "sf_axpy_dot", "sf_dot2", "sf_lincomb", "sf_div", "sf_quad_error",
            "sf_quad_load", "sf_face_load",
            "sf_smooth_colour_zrange", "sf_copy_uncovered", "sf_dense_apply")

# which thread-local error buffer each entry point writes (each module clears its own on entry)
_VEC = {"sf_convert", "sf_dot", "sf_axpy_dev", "sf_axpy_dot", "sf_dot2", "sf_lincomb", "sf_axpby", "sf_axpby_f32",
        "sf_div", "sf_dense_apply"}
_HALF = {"sf_to_half", "sf_from_half", "sf_demote16", "sf_ec_split", "sf_ec_matmul"}


def _error_message(what: str) -> str:
    L = lib()
    name = what.split()[0]
    if name in _VEC:
        getter = L.sf_vec_last_error
    elif name in _HALF:
        getter = L.sf_half_last_error
    elif name in ("sf_quad_error", "sf_quad_load", "sf_face_load",
            "sf_smooth_colour_zrange", "sf_copy_uncovered", "sf_dense_apply"):
        getter = L.sf_quad_last_error
    elif name == "sf_contract":
        getter = L.sf_contract_last_error
    else:
        getter = L.sf_last_error
    return (getter() or b"").decode()


def check(rc: int, what: str):
    if rc == SF_OK:
        return
    msg = _error_message(what)
    if rc == SF_EINVAL:
        raise ValueError(f"{what}: {msg}")
    if rc == SF_EUNSUPPORTED:
        raise NotImplementedError(f"{what}: {msg}")
    raise NativeError(f"{what}: {msg}")


def host_ptr(a: np.ndarray) -> int:
    assert a.dtype == np.float64 and a.flags.c_contiguous
    return a.ctypes.data
