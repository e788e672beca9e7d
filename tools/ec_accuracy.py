"""Low-precision accuracy report (FP16 / FP16-EC vs fp64 on the same fp32 input): vmult at several (k, L),
one smoothing step, one V-cycle and the solve's iterations / L2 error.  Prints one JSON line."""
import json
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2407_09621_b200 as sf  # noqa: E402
from paper_2407_09621_b200.discretization import assemble_rhs_separable, vmult_device  # noqa: E402

P = sf.PrecisionMode
out = {}


def rel(a, b):
    return (torch.linalg.norm(a.double() - b.double()) / torch.linalg.norm(b.double())).item()


g = torch.Generator(device="cuda").manual_seed(5)
for k, L in ((7, 5), (7, 6), (3, 6), (1, 7)):
    hier = sf.build_hierarchy(L, k, max_dofs=2**34, min_level=L)
    n = hier.n_dofs(L)
    u = torch.randn(n, dtype=torch.float64, device="cuda", generator=g).float()
    ref = torch.empty(n, dtype=torch.float64, device="cuda")
    vmult_device(hier, L, u.double(), ref, P.FP64)
    for m in (P.FP16, P.FP16_EC):
        v = torch.empty(n, dtype=torch.float32, device="cuda")
        vmult_device(hier, L, u, v, m)
        out[f"vmult_q{k}l{L}_{m.value}"] = rel(v, ref)
for k, L in ((7, 5), (3, 6)):
    hier = sf.build_hierarchy(L, k, max_dofs=2**34)
    n = hier.n_dofs(L)
    b = torch.randn(n, dtype=torch.float64, device="cuda", generator=g)
    x = torch.randn(n, dtype=torch.float64, device="cuda", generator=g)
    res = {}
    for m in (P.FP64, P.FP16, P.FP16_EC):
        mg = sf.MultigridPreconditioner(hier, sf.VCycleConfig(mode=m))
        res[m] = (mg.smooth(L, x.to(m.torch_dtype), b.to(m.torch_dtype)), mg.apply(b, L))
    for m in (P.FP16, P.FP16_EC):
        out[f"smooth_q{k}l{L}_{m.value}"] = rel(res[m][0], res[P.FP64][0])
        out[f"vcycle_q{k}l{L}_{m.value}"] = rel(res[m][1], res[P.FP64][1])
for k, L in ((7, 5), (3, 6)):
    for m in (P.FP64, P.FP16_EC):
        r = sf.run_solve(k, L, m)
        out[f"solve_q{k}l{L}_{m.value}"] = [r.report.iterations, r.l2]
print(json.dumps(out))
