"""Time the grid transfers at the fine level (CUDA events, mean of 10 after warm-up): prolongation+add and the
fused residual+restriction per mode, with the algorithmic HBM bytes and the fraction of the HBM roofline."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2407_09621_b200 as sf  # noqa: E402
from paper_2407_09621_b200.multigrid import prolongate_add_device, restrict_device  # noqa: E402

P = sf.PrecisionMode
HBM = 6547.5e9


def timeit(fn, reps=10):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


out = {}
cases = [(7, 6), (3, 7)] if len(sys.argv) < 2 else [tuple(map(int, a.split(","))) for a in sys.argv[1:]]
for k, L in cases:
    hier = sf.build_hierarchy(L, k, max_dofs=2**34, min_level=L - 1)
    nf, nc = hier.n_dofs(L), hier.n_dofs(L - 1)
    for m in (P.FP64, P.FP16_EC):
        dt = m.torch_dtype
        es = torch.tensor([], dtype=dt).element_size()
        e = torch.randn(nc, dtype=torch.float64, device="cuda").to(dt)
        x = torch.randn(nf, dtype=torch.float64, device="cuda").to(dt)
        b = torch.randn(nf, dtype=torch.float64, device="cuda").to(dt)
        rc = torch.empty(nc, dtype=dt, device="cuda")
        ms = timeit(lambda: prolongate_add_device(hier, L - 1, e, x, m))
        byt = (2 * nf + nc) * es
        out[f"prolong_q{k}l{L}_{m.value}"] = {"ms": ms, "GBs": byt / ms / 1e6, "frac": byt / ms / 1e-3 / HBM}
        ms = timeit(lambda: restrict_device(hier, L, b, rc, m, x=x))
        byt = (2 * nf + nc) * es
        out[f"resid_restrict_q{k}l{L}_{m.value}"] = {"ms": ms, "GBs": byt / ms / 1e6, "frac": byt / ms / 1e-3 / HBM}
print(json.dumps(out))
