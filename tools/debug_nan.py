"""Locate the first non-finite value in a low-precision V-cycle (diagnostics)."""
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2407_09621_b200 as sf  # noqa: E402
from paper_2407_09621_b200 import multigrid as M  # noqa: E402
from paper_2407_09621_b200.discretization import assemble_rhs_separable, vmult_device  # noqa: E402

k, lvl, mode = int(sys.argv[1]), int(sys.argv[2]), sf.PrecisionMode.parse(sys.argv[3])
hier = sf.build_hierarchy(lvl, k, max_dofs=2**34)
b64 = assemble_rhs_separable(hier, lvl, lambda x: np.sin(np.pi * x), 3 * math.pi**2)
b64 = b64 / torch.linalg.norm(b64)
mg = sf.MultigridPreconditioner(hier, sf.VCycleConfig(mode=mode))


def stat(name, t):
    t = t.double()
    fin = torch.isfinite(t)
    print(f"{name:40s} finite={bool(fin.all())} maxabs={float(t[fin].abs().max()) if fin.any() else float('nan'):.3e} "
          f"minabs_nz={float(t[fin & (t != 0)].abs().min()) if (fin & (t != 0)).any() else 0:.3e}", flush=True)


orig_smooth = mg._smooth_device


def smooth(level, x, b, m):
    stat(f"smooth in x L{level}", x)
    orig_smooth(level, x, b, m)
    stat(f"smooth out x L{level}", x)


mg._smooth_device = smooth
orig_coarse = mg._coarse_solve_device


def coarse(b, m):
    stat("coarse rhs", b)
    x = orig_coarse(b, m)
    stat("coarse x", x)
    return x


mg._coarse_solve_device = coarse
for L in range(lvl, 1, -1):
    u = torch.randn(hier.n_dofs(L), dtype=torch.float32, device="cuda") * 1e-4
    v = torch.empty_like(u)
    vmult_device(hier, L, u, v, mode)
    stat(f"vmult L{L} (u~1e-4)", v)
out = mg.apply(b64, lvl)
stat("vcycle out", out)
