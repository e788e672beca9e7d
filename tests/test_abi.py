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
    from paper_2407_09621_b200 import _native

    assert lib.sf_abi_version() == _native.ABI_VERSION == 5


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


def test_vector_entry_points_validate_with_messages():
    """Every SF_EINVAL of the vector module carries its own message (no stale text from another module)."""
    import ctypes

    from paper_2407_09621_b200 import _native

    L = _native.lib()
    # leave a message in the ops module's buffer first
    assert L.sf_vmult(0, 7, _native.SfGrid(3, 2, 2, None, None), None, None, None, 1, None) == _native.SF_EINVAL
    M = _native.SF_LINCOMB_MAX_TERMS
    P = (ctypes.c_void_p * (M + 1))(*([1] * (M + 1)))
    C = (ctypes.c_double * (M + 1))()
    out = ctypes.c_void_p(16)
    cases = [
        ("sf_lincomb", lambda: L.sf_lincomb(8, M + 1, ctypes.cast(P, ctypes.c_void_p), ctypes.cast(C, ctypes.c_void_p),
                                            out, None), "term count"),
        ("sf_lincomb", lambda: L.sf_lincomb(8, -1, None, None, out, None), "term count"),
        ("sf_lincomb", lambda: L.sf_lincomb(8, 2, None, None, out, None), "null term arrays"),
        ("sf_axpy_dot", lambda: L.sf_axpy_dot(8, 1.0, None, None, None, None, None, None, None), "null"),
        ("sf_dot2", lambda: L.sf_dot2(-1, None, None, None, None, None, None, None), "negative"),
        ("sf_div", lambda: L.sf_div(8, None, 2.0, None, None), "null"),
        ("sf_dense_apply", lambda: L.sf_dense_apply(8, None, out, 0, 0, out, 0, None), "null"),
        ("sf_dense_apply", lambda: L.sf_dense_apply(8, out, out, 2, 0, out, 0, None), "dtype"),
        ("sf_convert", lambda: L.sf_convert(4, out, 3, out, 0, None), "dtype"),
        ("sf_smooth_colour", lambda: L.sf_smooth_colour(3, 7, _native.SfGrid(4, 4, 4, None, None),
                                                        (ctypes.c_int * 3)(1, 0, 0), out, out, None, out,
                                                        ctypes.c_void_p(32), None), "unshifted colour"),
    ]
    for name, call, frag in cases:
        assert call() == _native.SF_EINVAL, name
        with pytest.raises(ValueError, match=frag):
            _native.check(_native.SF_EINVAL, name)
    # a null entry inside the term array
    P2 = (ctypes.c_void_p * 2)(16, None)
    assert L.sf_lincomb(8, 2, ctypes.cast(P2, ctypes.c_void_p), ctypes.cast(C, ctypes.c_void_p), out,
                        None) == _native.SF_EINVAL
    with pytest.raises(ValueError, match="null term vector"):
        _native.check(_native.SF_EINVAL, "sf_lincomb")
    # the ops buffer is cleared by its next entry point, so its old message cannot leak either
    assert L.sf_vmult(0, 9, _native.SfGrid(2, 2, 2, None, None), None, None, None, 1, None) == _native.SF_EUNSUPPORTED
    with pytest.raises(NotImplementedError, match="degree"):
        _native.check(_native.SF_EUNSUPPORTED, "sf_vmult")


def test_abi_mismatch_is_an_import_error(tmp_path, monkeypatch):
    """A library missing a declared entry point raises ImportError with the rebuild hint, not AttributeError."""
    import shutil
    import subprocess

    from paper_2407_09621_b200 import _native

    src = tmp_path / "old.c"
    src.write_text("int sf_abi_version(void) { return 4; }\n")
    so = tmp_path / "libold.so"
    subprocess.run(["gcc", "-shared", "-fPIC", "-o", str(so), str(src)], check=True)
    monkeypatch.setattr(_native, "LIB_PATH", str(so))
    monkeypatch.setattr(_native, "_lib", None)
    with pytest.raises(ImportError, match="rebuild"):
        _native.lib()
