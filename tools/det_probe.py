"""Bitwise reproducibility probe: every mode's vmult twice on the same input (hash + max |diff|)."""
import hashlib
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2407_09621_b200 as sf  # noqa: E402
from paper_2407_09621_b200.discretization import vmult_device  # noqa: E402

P = sf.PrecisionMode
g = torch.Generator(device="cuda").manual_seed(5)
cases = [(7, 2), (7, 3), (3, 4), (1, 5), (7, 5), (3, 6), (1, 7)] if len(sys.argv) < 2 else \
    [tuple(map(int, c.split(","))) for c in sys.argv[1:]]
for k, L in cases:
    hier = sf.build_hierarchy(L, k, max_dofs=2**34, min_level=L)
    n = hier.n_dofs(L)
    u = torch.randn(n, dtype=torch.float64, device="cuda", generator=g).float()
    hs = []
    for m in (P.FP64, P.FP32, P.FP16, P.FP16_EC):
        outs = []
        for rep in range(3):
            v = torch.empty(n, dtype=m.torch_dtype, device="cuda")
            vmult_device(hier, L, u.to(m.torch_dtype), v, m)
            outs.append(v)
        d = max(float((o - outs[0]).abs().max()) for o in outs[1:]) / float(outs[0].abs().max())
        nd = max(int((o != outs[0]).sum()) for o in outs[1:])
        hs.append(f"{m.value}:{'ok' if nd == 0 else f'DIFF n={nd} rel={d:.1e}'}")
    print(k, L, " ".join(hs), flush=True)
