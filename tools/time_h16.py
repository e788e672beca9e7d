"""Time the binary16 Q7 kernels (vmult at L7, colour pass at L6, EC solve at L6); SUMFACT_UMMA selects the path."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2407_09621_b200 as sf  # noqa: E402
from paper_2407_09621_b200.discretization import vmult_device  # noqa: E402


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


out = {"umma": os.environ.get("SUMFACT_UMMA", "0")}
P = sf.PrecisionMode
h7 = sf.build_hierarchy(7, 7, max_dofs=2**34, min_level=7)
u = torch.randn(h7.n_dofs(7), dtype=torch.float32, device="cuda")
v = torch.empty_like(u)
for m in (P.FP16, P.FP16_EC):
    ms = timeit(lambda: vmult_device(h7, 7, u, v, m))
    out[f"vmult_l7_{m.value}_ms"] = ms
    out[f"vmult_l7_{m.value}_gdofs"] = h7.n_dofs(7) / ms / 1e6
del u, v
h6 = sf.build_hierarchy(6, 7, max_dofs=2**34)
D6 = h6.n_dofs(6)
for m in (P.FP16, P.FP16_EC):
    mg = sf.MultigridPreconditioner(h6, sf.VCycleConfig(mode=m))
    x = torch.zeros(D6, dtype=torch.float32, device="cuda")
    b = torch.randn(D6, dtype=torch.float32, device="cuda")
    out[f"smooth_step_l6_{m.value}_ms"] = timeit(lambda: mg._smooth_device(6, x, b, m), reps=3)
print(json.dumps(out))
