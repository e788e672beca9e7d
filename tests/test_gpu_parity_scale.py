"""Parity where it matters: the FP64 vmult against the oracle at C1 (Q7 L4, the
BASELINE config the CPU reference runs) and beyond, and VALUE checks at the
1e9-DoF bench meshes (Q7 L7, Q3 L8) on sampled cells through the cell-local
evaluator that tests/test_local_stencil.py pins to the oracle.  The sampled
cells include corners, edges, faces and both sides of every tile-band boundary
(the banded grid, L2 prefetch and 32-bit offset paths of the kernels)."""
import numpy as np
import pytest
import torch

import paper_2407_09621_b200 as sf
from conftest import rel_l2
from local_stencil import LocalVmult, sample_cells
from oracle import port

pytestmark = pytest.mark.gpu
P = sf.PrecisionMode


@pytest.mark.parametrize("k,lvl", [(7, 4), (3, 5), (7, 5), (1, 6)])
def test_fp64_vmult_full_mesh_vs_oracle(k, lvl):
    """C1 = Q7 L4 (2.1 M DoF); Q3 L5 (2.1 M); Q7 L5 (16.8 M); Q1 L6 (2.1 M): every DoF <= 1e-12."""
    H = port.Hierarchy(lvl, k)
    u = np.random.default_rng(0).standard_normal(H.n_dofs(lvl))
    ref = port.apply_operator(H, lvl, u, threads=port.default_threads())
    v = sf.apply_operator(sf.build_hierarchy(lvl, k, max_dofs=2**31), lvl, u)
    assert rel_l2(v, ref) <= 1e-12
    # no single DoF far off either (relative to the operator scale)
    assert np.max(np.abs(v - ref)) <= 1e-11 * np.max(np.abs(ref))


def _device_u(n, dtype, seed=0):
    g = torch.Generator(device="cuda")
    g.manual_seed(seed)
    return torch.randn(n, dtype=torch.float64, device="cuda", generator=g).to(dtype)


def _sampled(k, lvl, v, u64, ncells, seed):
    """(GPU values, local fp64 values) on the sampled cells, flattened."""
    loc = LocalVmult(k, lvl)
    K = k + 1
    A = loc.n * K
    cells = sample_cells(loc.n, ncells, seed=seed, band=16)
    got, want = [], []
    vv = v.view(A, A, A)
    for (cz, cy, cx) in cells:
        idx = torch.from_numpy(loc.block_index(cz, cy, cx).reshape(-1)).cuda()
        blk = u64[idx].cpu().numpy().reshape(loc.block_index(cz, cy, cx).shape)
        want.append(loc.apply_cell(blk, cz, cy, cx).reshape(-1))
        got.append(vv[cz * K:(cz + 1) * K, cy * K:(cy + 1) * K, cx * K:(cx + 1) * K]
                   .double().cpu().numpy().reshape(-1))
    return np.concatenate(got), np.concatenate(want), len(cells)


@pytest.mark.parametrize("k,lvl", [(7, 7), (3, 8), (7, 6), (3, 7)])
def test_fp64_vmult_values_at_bench_size(k, lvl):
    """The bench meshes (1.07e9 DoF) and the 1.34e8 solve meshes: >= 1,500 sampled cells <= 1e-12."""
    hier = sf.build_hierarchy(lvl, k, max_dofs=2**31)
    n = hier.n_dofs(lvl)
    u = _device_u(n, torch.float64)
    v = sf.apply_operator(hier, lvl, u)
    torch.cuda.synchronize()
    got, want, nc = _sampled(k, lvl, v, u, 1500, seed=lvl)
    assert nc >= 1500
    assert rel_l2(got, want) <= 1e-12
    assert np.max(np.abs(got - want)) <= 1e-11 * np.max(np.abs(want))
    del u, v
    torch.cuda.empty_cache()


# reference error bands at C1 (measured with the reference: u ~ N(0,1), seed 0):
# Q7 L4 fp32 1.29e-7, fp16 4.22e-4, fp16_ec 1.63e-7.  Ours must stay within 4x at 1e9 DoF.
REF_BAND = {P.FP32: 1.29e-7, P.FP16: 4.22e-4, P.FP16_EC: 1.63e-7}


@pytest.mark.parametrize("mode", [P.FP32, P.FP16, P.FP16_EC])
def test_low_precision_vmult_band_at_bench_size(mode):
    k, lvl = 7, 7
    hier = sf.build_hierarchy(lvl, k, max_dofs=2**31)
    n = hier.n_dofs(lvl)
    u64 = _device_u(n, torch.float64)
    u32 = u64.float()
    v = sf.apply_operator(hier, lvl, u32, mode)
    assert v.dtype == torch.float32
    torch.cuda.synchronize()
    # the reference demotes the input to the storage dtype first: compare against A float32(u)
    got, want, _ = _sampled(k, lvl, v, u32.double(), 600, seed=11)
    err = rel_l2(got, want)
    assert err <= 4 * REF_BAND[mode], err
    del u64, u32, v
    torch.cuda.empty_cache()
