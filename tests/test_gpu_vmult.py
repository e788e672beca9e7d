"""GPU parity of the vmult (sf_vmult) against the reference's golden vectors,
the CPU oracle, and size-independent properties at large sizes."""
import numpy as np
import pytest
import torch

import paper_2407_09621_b200 as sf
from conftest import rel_l2
from oracle import port

pytestmark = pytest.mark.gpu
P = sf.PrecisionMode
CASES = [(1, 1), (1, 2), (2, 2), (3, 2), (3, 3), (7, 1), (7, 2)]

# error band of the reference's own low-precision vmults (golden), per mode:
# ours must land within a factor of it (cell-wise schedule, same operand semantics)
BAND = {P.FP32: 4.0, P.FP16: 4.0, P.FP16_EC: 4.0}


@pytest.mark.parametrize("k,lvl", CASES)
def test_fp64_vmult_matches_reference_1e12(gold, k, lvl):
    hier = sf.build_hierarchy(lvl, k)
    u = np.random.default_rng(0).standard_normal(hier.n_dofs(lvl))
    v = sf.apply_operator(hier, lvl, u)
    assert v.dtype == np.float64
    assert rel_l2(v, gold("vmult")[f"k{k}_l{lvl}_fp64"]) <= 1e-12


@pytest.mark.parametrize("k,lvl", CASES)
@pytest.mark.parametrize("mode", [P.FP32, P.FP16, P.FP16_EC])
def test_low_precision_vmult_error_band(gold, k, lvl, mode):
    hier = sf.build_hierarchy(lvl, k)
    u = np.random.default_rng(0).standard_normal(hier.n_dofs(lvl))
    ref64 = gold("vmult")[f"k{k}_l{lvl}_fp64"]
    ref_low = gold("vmult")[f"k{k}_l{lvl}_{mode.value}"]
    v = sf.apply_operator(hier, lvl, u, mode)
    assert v.dtype == np.float32
    err, ref_err = rel_l2(v, ref64), rel_l2(ref_low, ref64)
    assert err <= BAND[mode] * ref_err + 1e-7, (err, ref_err)


def test_precision_ordering_like_reference():
    """tests/test_discretization.py:261-276: fp32 < 1e-5, fp32 < fp16 < 0.1, ec < fp16."""
    hier = sf.build_hierarchy(2, 2)
    u = np.random.default_rng(2).standard_normal(hier.n_dofs(2))
    ref = sf.apply_operator(hier, 2, u, P.FP64)
    r32 = rel_l2(sf.apply_operator(hier, 2, u, P.FP32), ref)
    r16 = rel_l2(sf.apply_operator(hier, 2, u, P.FP16), ref)
    rec = rel_l2(sf.apply_operator(hier, 2, u, P.FP16_EC), ref)
    assert r32 < 1e-5 and r32 < r16 < 0.1 and rec < r16


@pytest.mark.parametrize("k,lvl", [(7, 3), (3, 4), (2, 3), (4, 2), (5, 2), (6, 2)])
def test_fp64_vmult_matches_oracle(k, lvl):
    H = port.Hierarchy(lvl, k)
    u = np.random.default_rng(7).standard_normal(H.n_dofs(lvl))
    ref = port.apply_operator(H, lvl, u)
    v = sf.apply_operator(sf.build_hierarchy(lvl, k), lvl, u)
    assert rel_l2(v, ref) <= 1e-12


def test_dense_assembly_oracle(gold):
    """Independent dense SIPG assembly of the reference (tests/sipg_oracle.py)."""
    g = gold("sipg_dense")
    for k, lvl, key in [(1, 1, "k1_l1"), (1, 2, "k1_l2"), (2, 1, "k2_l1")]:
        A = sf.materialize_operator(sf.build_hierarchy(lvl, k), lvl)
        assert rel_l2(A, g[key]) <= 1e-12
        assert np.allclose(A, A.T, atol=1e-12 * np.abs(A).max())


def test_zero_and_length_guard():
    hier = sf.build_hierarchy(1, 2)
    assert np.all(sf.apply_operator(hier, 1, np.zeros(hier.n_dofs(1))) == 0)
    with pytest.raises(ValueError):
        sf.apply_operator(hier, 1, np.zeros(10))


def test_constants_annihilated_in_interior():
    hier = sf.build_hierarchy(2, 1)
    r = sf.apply_operator(hier, 2, np.ones(hier.n_dofs(2))).reshape(hier.shape(2))
    K = 2
    assert np.abs(r[K:-K, K:-K, K:-K]).max() <= 1e-10
    assert np.abs(r).max() > 0.1


def test_tensor_in_tensor_out_and_determinism():
    hier = sf.build_hierarchy(3, 7)
    u = torch.randn(hier.n_dofs(3), dtype=torch.float64, device="cuda")
    v1 = sf.apply_operator(hier, 3, u)
    v2 = sf.apply_operator(hier, 3, u)
    assert v1.is_cuda and torch.equal(v1, v2)


@pytest.mark.parametrize("k,lvl", [(7, 6), (3, 7), (7, 7), (3, 8)])
def test_large_vmult_symmetry_and_linearity(k, lvl):
    """At the bench sizes (1.3e8 and 1.07e9 DoF) parity is checked through properties."""
    hier = sf.build_hierarchy(lvl, k, max_dofs=2**31)
    n = hier.n_dofs(lvl)
    g = torch.Generator(device="cuda").manual_seed(3)
    u = torch.randn(n, dtype=torch.float64, device="cuda", generator=g)
    w = torch.randn(n, dtype=torch.float64, device="cuda", generator=g)
    Au, Aw = sf.apply_operator(hier, lvl, u), sf.apply_operator(hier, lvl, w)
    a, b = float(torch.dot(Au, w)), float(torch.dot(u, Aw))
    assert abs(a - b) <= 1e-11 * abs(a)
    Auw = sf.apply_operator(hier, lvl, 2.0 * u - 3.0 * w)
    assert float(torch.linalg.norm(Auw - (2.0 * Au - 3.0 * Aw)) / torch.linalg.norm(Auw)) <= 1e-13
    assert float(torch.dot(u, Au)) > 0


def test_slab_ghosts_reproduce_the_full_operator():
    """Two z-slabs with K-plane ghost layers (the multi-GPU layout) == one domain."""
    from paper_2407_09621_b200 import _native
    from paper_2407_09621_b200.discretization import vmult_device

    k, lvl = 3, 3
    hier = sf.build_hierarchy(lvl, k)
    K, n, A = k + 1, 2**lvl, hier.axis_dofs(lvl)
    u = torch.randn(hier.n_dofs(lvl), dtype=torch.float64, device="cuda")
    full = sf.apply_operator(hier, lvl, u).reshape(A, A, A)
    U = u.reshape(A, A, A)
    half = A // 2
    lo, hi = U[:half].contiguous(), U[half:].contiguous()
    g_lo = U[half:half + K].contiguous()   # planes above the lower slab
    g_hi = U[half - K:half].contiguous()   # planes below the upper slab
    out_lo, out_hi = torch.empty_like(lo), torch.empty_like(hi)
    vmult_device(hier, lvl, lo, out_lo, P.FP64, grid=_native.SfGrid(n, n, n // 2, None, g_lo.data_ptr()))
    vmult_device(hier, lvl, hi, out_hi, P.FP64, grid=_native.SfGrid(n, n, n // 2, g_hi.data_ptr(), None))
    got = torch.cat([out_lo, out_hi])
    assert float(torch.linalg.norm(got - full) / torch.linalg.norm(full)) <= 1e-14


@pytest.mark.parametrize("k,lvl", [(7, 3), (3, 4), (1, 5), (3, 2)])
def test_tensor_core_path_matches_cuda_core_path(tmp_path, k, lvl):
    """The DMMA kernels (Q7 tiles; Q3/Q1 16-point line tiles) and the generic CUDA-core tile engine
    agree (SUMFACT_B200_GENERIC=1)."""
    import os
    import subprocess
    import sys

    code = ("import numpy as np, sys; sys.path.insert(0, %r); import paper_2407_09621_b200 as sf; "
            f"h = sf.build_hierarchy({lvl}, {k}); u = np.random.default_rng(11).standard_normal(h.n_dofs({lvl})); "
            f"np.save(%r, sf.apply_operator(h, {lvl}, u))")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    outs = []
    for flag in ("0", "1"):
        path = str(tmp_path / f"v{flag}.npy")
        env = dict(os.environ, SUMFACT_B200_GENERIC=flag)
        subprocess.run([sys.executable, "-c", code % (root, path)], check=True, env=env)
        outs.append(np.load(path))
    assert rel_l2(outs[0], outs[1]) <= 1e-14


@pytest.mark.parametrize("lvl", [3, 4])
@pytest.mark.parametrize("mode", [P.FP16, P.FP16_EC])
def test_q7_half_precision_tensor_core_vmult_band(lvl, mode):
    """HMMA fp16 / fp16-EC Q7 vmult: error vs fp64 within the reference's own error band."""
    H = port.Hierarchy(lvl, 7)
    u = np.random.default_rng(0).standard_normal(H.n_dofs(lvl))
    ref64 = port.apply_operator(H, lvl, u, "fp64")
    ref_err = rel_l2(port.apply_operator(H, lvl, u, mode.value), ref64)
    err = rel_l2(sf.apply_operator(sf.build_hierarchy(lvl, 7), lvl, u, mode), ref64)
    assert 0.25 * ref_err <= err <= 4.0 * ref_err, (err, ref_err)


@pytest.mark.parametrize("mode", [P.FP64, P.FP16_EC])
@pytest.mark.parametrize("slab_cells", [2, 4, 6])
def test_streamed_host_vmult_matches_device(mode, slab_cells):
    """apply_operator on host buffers streams z-slabs with ghost planes through the GPU."""
    from paper_2407_09621_b200 import discretization as dz

    k, lvl = 3, 4
    hier = sf.build_hierarchy(lvl, k)
    n = hier.n_dofs(lvl)
    u = torch.randn(n, dtype=mode.torch_dtype).pin_memory()
    v = torch.empty_like(u).pin_memory()
    dz._stream_vmult(hier, lvl, u, v, mode, slab_cells=slab_cells)
    ref = torch.empty(n, dtype=mode.torch_dtype, device="cuda")
    dz.vmult_device(hier, lvl, u.cuda(), ref, mode)
    # (slabs thinner than a 16-point tile line use the CUDA-core tile engine: same value to rounding)
    assert float((v - ref.cpu()).norm() / ref.norm().cpu()) <= (1e-15 if mode is P.FP64 else 1e-6)
    # the public API takes this path for large host inputs
    old = dz.STREAM_MIN_DOFS
    dz.STREAM_MIN_DOFS = 1
    try:
        w = sf.apply_operator(hier, lvl, u.numpy(), mode)
    finally:
        dz.STREAM_MIN_DOFS = old
    assert isinstance(w, np.ndarray) and w.dtype == mode.storage_dtype
    assert np.abs(w - ref.cpu().numpy()).max() <= 1e-12 * float(ref.abs().max()) or mode is not P.FP64


def test_full_size_constants_annihilated_in_interior():
    """Q7 level 7 (1.07e9 DoF, the bench workload): A 1 = 0 away from the Nitsche boundary cells."""
    k, lvl = 7, 7
    hier = sf.build_hierarchy(lvl, k, max_dofs=2**31)
    n, K = hier.n_cells(lvl), k + 1
    u = torch.ones(hier.n_dofs(lvl), dtype=torch.float64, device="cuda")
    v = sf.apply_operator(hier, lvl, u).reshape(n * K, n * K, n * K)
    inner = v[K:-K, K:-K, K:-K]
    scale = float(sf.apply_operator(hier, lvl, torch.randn_like(u)).abs().max())
    assert float(inner.abs().max()) <= 1e-12 * scale
    assert float(v.abs().max()) > 1e-6 * scale  # the boundary layer is not zero


@pytest.mark.parametrize("k", [1, 2, 3, 4, 5, 6, 7])
@pytest.mark.parametrize("mode", [P.FP32, P.FP16, P.FP16_EC])
def test_every_degree_and_mode_against_oracle(k, mode):
    """Every compiled degree in every low-precision mode (tensor-core line/patch tiles for k = 1, 3, 7,
    the CUDA-core tile engine otherwise) against the oracle port's own low-precision apply: same
    per-contraction demotion semantics, so the two error levels agree within a small factor."""
    lvl = 3 if k <= 3 else 2
    hier = sf.build_hierarchy(lvl, k)
    u = np.random.default_rng(k).standard_normal(hier.n_dofs(lvl))
    H = port.Hierarchy(lvl, k)
    ref64 = port.apply_operator(H, lvl, u)
    ref_low = port.apply_operator(H, lvl, u.astype(np.float32), mode.value)
    v = sf.apply_operator(hier, lvl, u, mode)
    err, ref_err = rel_l2(v, ref64), rel_l2(ref_low, ref64)
    assert err <= 3.0 * ref_err + 1e-7, (err, ref_err)
    assert err >= ref_err / 30.0  # same precision class (not silently fp64)


@pytest.mark.parametrize("k,lvl", [(7, 7), (3, 8)])
def test_full_size_low_precision_error_levels(k, lvl):
    """1.07e9 DoF: the tensor-core FP16 / FP16-EC / FP32 vmults keep their precision class at the bench
    size (the power-of-two range management keeps binary16 operands normal), measured against FP64."""
    hier = sf.build_hierarchy(lvl, k, max_dofs=2**31)
    g = torch.Generator(device="cuda").manual_seed(21)
    u64 = torch.randn(hier.n_dofs(lvl), dtype=torch.float64, device="cuda", generator=g)
    ref = sf.apply_operator(hier, lvl, u64)
    u32 = u64.float()
    del u64
    errs = {}
    for mode in (P.FP32, P.FP16, P.FP16_EC):
        v = sf.apply_operator(hier, lvl, u32, mode)
        errs[mode] = float((v.double() - ref).norm() / ref.norm())
        del v
    assert errs[P.FP32] < 1e-5 and errs[P.FP16_EC] < 1e-5 and 1e-5 < errs[P.FP16] < 1e-2, errs


@pytest.mark.parametrize("k,lvl", [(7, 3), (3, 4), (1, 5)])
def test_fp32_dmma_path_matches_cuda_core_fp32(tmp_path, k, lvl):
    """FP32 storage on the DMMA kernels (stage outputs rounded to fp32) vs the CUDA-core engine's float
    arithmetic: both within fp32 rounding of each other and of the fp64 operator."""
    import os
    import subprocess
    import sys

    code = ("import numpy as np, sys; sys.path.insert(0, %r); import paper_2407_09621_b200 as sf; "
            f"h = sf.build_hierarchy({lvl}, {k}); u = np.random.default_rng(11).standard_normal(h.n_dofs({lvl})); "
            f"np.save(%r, sf.apply_operator(h, {lvl}, u, sf.PrecisionMode.FP32))")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    outs = []
    for flag in ("0", "1"):
        path = str(tmp_path / f"v{flag}.npy")
        subprocess.run([sys.executable, "-c", code % (root, path)], check=True,
                       env=dict(os.environ, SUMFACT_B200_GENERIC=flag))
        outs.append(np.load(path).astype(np.float64))
    hier = sf.build_hierarchy(lvl, k)
    ref64 = sf.apply_operator(hier, lvl, np.random.default_rng(11).standard_normal(hier.n_dofs(lvl)))
    assert rel_l2(outs[0], outs[1]) <= 2e-6
    assert rel_l2(outs[0], ref64) <= rel_l2(outs[1], ref64) * 2.0 + 1e-7


def test_misaligned_vectors_are_rejected():
    """Vectors feed 16-byte vector loads / cp.async chunks: a pointer that is not 16-byte aligned is an
    SF_EINVAL (ValueError), not a device fault."""
    from paper_2407_09621_b200.discretization import vmult_device

    hier = sf.build_hierarchy(3, 7)
    D = hier.n_dofs(3)
    for mode in (P.FP32, P.FP64):
        base = torch.randn(D + 1, dtype=mode.torch_dtype, device="cuda")
        v = torch.empty(D, dtype=mode.torch_dtype, device="cuda")
        with pytest.raises(ValueError, match="16-byte aligned"):
            vmult_device(hier, 3, base[1:], v, mode)
    torch.cuda.synchronize()  # no sticky device error
    u = torch.randn(D, dtype=torch.float32, device="cuda")
    assert torch.isfinite(sf.apply_operator(hier, 3, u, P.FP32)).all()
