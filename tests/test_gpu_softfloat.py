"""binary16 primitives (precision.py:60-197) on the GPU, bit-exact against fixtures made by the reference itself
(tools/make_golden.py softfloat): the reference's 20,107-pair RNE fixture (tests/data/half_reference.txt), NaN
payloads and range edges, all 65,536 half patterns, ec_split and ec_matmul."""
import numpy as np
import pytest
import torch

import paper_2407_09621_b200 as sf

pytestmark = pytest.mark.gpu


def test_to_half_matches_reference_fixture(gold):
    g = gold("softfloat")
    got = sf.to_half(g["fix_x"].view(np.float32))
    assert got.dtype == np.uint16 and np.array_equal(got, g["fix_h"])


def test_to_half_nan_payloads_and_edges(gold):
    g = gold("softfloat")
    assert np.array_equal(sf.to_half(g["edge_x"]), g["edge_h"])
    assert sf.to_half(np.float32(1.0)) == np.uint16(0x3C00)  # scalar in, scalar out


def test_from_half_all_patterns(gold):
    g = gold("softfloat")
    got = sf.from_half(np.arange(65536, dtype=np.uint32).astype(np.uint16))
    assert np.array_equal(got.view(np.uint32), g["from_half_all"])


def test_demote16_matches_reference_and_roundtrip(gold):
    g = gold("half")
    got = sf.demote16(g["x"])
    assert np.array_equal(got.view(np.uint32), g["demoted"].view(np.uint32))
    x = g["x"][np.isfinite(g["x"])]
    assert np.array_equal(sf.from_half(sf.to_half(x)).view(np.uint32), sf.demote16(x).view(np.uint32))
    # device tensors stay on the device
    t = torch.from_numpy(g["x"]).cuda()
    assert sf.demote16(t).is_cuda and np.array_equal(sf.demote16(t).cpu().numpy().view(np.uint32),
                                                     g["demoted"].view(np.uint32))


def test_ec_split_matches_reference(gold):
    g = gold("softfloat")
    pr = sf.ec_split(g["ec_x"])
    assert np.array_equal(pr.main, g["ec_main"]) and np.array_equal(pr.residual, g["ec_resid"])
    rec, x = pr.reconstruct(), g["ec_x"]
    big = np.abs(x) > 1e-2  # residual half still normal: ~22 significant bits
    assert np.max(np.abs(rec[big] - x[big]) / np.abs(x[big])) < 2.0**-20
    with pytest.raises(sf.HalfRangeError):
        sf.ec_split(np.array([1.0, 7e4], dtype=np.float32))
    with pytest.raises(sf.HalfRangeError):
        sf.ec_split(np.array([np.nan], dtype=np.float32))


@pytest.mark.parametrize("refine", ["both", "left", "right"])
def test_ec_matmul_matches_reference(gold, refine):
    g = gold("softfloat")
    A, B = g["mm_a"], g["mm_b"]
    ea, eb = sf.ec_split(A), sf.ec_split(B)
    got = sf.ec_matmul(ea, eb, refine=refine)
    ref = g[f"mm_{refine}"]
    assert got.shape == ref.shape
    # fp32 accumulation; the reference's einsum may sum in another order
    assert np.max(np.abs(got - ref)) <= 4 * np.finfo(np.float32).eps * np.max(np.abs(ref)) * A.shape[1]
    with pytest.raises(ValueError):
        sf.ec_matmul(ea, eb, refine="middle")
    with pytest.raises(ValueError):
        sf.ec_matmul(eb, eb)
