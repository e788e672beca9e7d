"""One small binary16 vmult + colour pass for a single compute-sanitizer tool run: python tools/sanitize_one.py k L mode"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2407_09621_b200 as sf  # noqa: E402

k, L, mode = int(sys.argv[1]), int(sys.argv[2]), sf.PrecisionMode.parse(sys.argv[3])
hier = sf.build_hierarchy(L, k)
n = hier.n_dofs(L)
u = torch.randn(n, dtype=torch.float64, device="cuda").to(mode.torch_dtype)
v = sf.apply_operator(hier, L, u, mode)
torch.cuda.synchronize()
print("vmult ok", flush=True)
mg = sf.MultigridPreconditioner(hier, sf.VCycleConfig(mode=mode))
x = mg.smooth(L, torch.zeros_like(u), u, mode)
torch.cuda.synchronize()
print("smooth ok", flush=True)
