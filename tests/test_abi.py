"""CPU-side checks of the drop-in boundary: the C-ABI library exists, loads and
exports every entry point include/sumfact_b200.h declares (no compute)."""
import ctypes
import os
import re

import pytest

from conftest import ROOT

HEADER = os.path.join(ROOT, "include", "sumfact_b200.h")
LIB = os.path.join(ROOT, "paper_2407_09621_b200", "libsumfact_b200.so")


def declared():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:int|const char\*)\s+(sf_\w+)\s*\(", text, re.M)))


def test_header_declares_the_path():
    names = declared()
    for must in ("sf_vmult", "sf_smooth_colour", "sf_residual_restrict", "sf_prolongate_add", "sf_patch_apply",
                 "sf_dot", "sf_axpy_dev", "sf_axpby", "sf_convert"):
        assert must in names


def test_library_exports_every_declared_symbol():
    assert os.path.exists(LIB), "run __graft_entry__.build() first"
    lib = ctypes.CDLL(LIB)
    missing = [n for n in declared() if not hasattr(lib, n)]
    assert not missing, missing
    lib.sf_abi_version.restype = ctypes.c_int
    assert lib.sf_abi_version() == 1


def test_library_is_sm100a_only():
    import subprocess

    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", LIB], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    for other in ("sm_80", "sm_90", "sm_103"):
        assert other not in out


def test_argument_validation_without_gpu():
    """Validation happens before any CUDA call, so it is testable on CPU."""
    from paper_2407_09621_b200 import _native

    L = _native.lib()
    g = _native.SfGrid(3, 2, 2, None, None)
    rc = L.sf_vmult(0, 7, g, None, None, None, 1, None)
    assert rc == _native.SF_EINVAL
    rc = L.sf_vmult(0, 9, g, None, None, None, 1, None)
    assert rc == _native.SF_EUNSUPPORTED
    rc = L.sf_vmult(7, 3, g, None, None, None, 1, None)
    assert rc == _native.SF_EINVAL
    with pytest.raises(ValueError):
        _native.check(_native.SF_EINVAL, "x")
    with pytest.raises(NotImplementedError):
        _native.check(_native.SF_EUNSUPPORTED, "x")


def test_product_refuses_cpu():
    """No CPU fallback: the public API raises without a CUDA device."""
    import numpy as np
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    import paper_2407_09621_b200 as sf

    hier = sf.build_hierarchy(1, 1)
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        sf.apply_operator(hier, 1, np.zeros(hier.n_dofs(1)))
