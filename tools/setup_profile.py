"""Where the solve setup time goes (bench extras' setup_s): python tools/setup_profile.py k L mode"""
import cProfile
import io
import math
import os
import pstats
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2407_09621_b200 as sf  # noqa: E402
from paper_2407_09621_b200.discretization import assemble_rhs_separable  # noqa: E402

k, L, mode = int(sys.argv[1]), int(sys.argv[2]), sf.PrecisionMode.parse(sys.argv[3])
torch.zeros(1, device="cuda")
torch.cuda.synchronize()


def step(name, fn):
    torch.cuda.synchronize()
    t = time.perf_counter()
    r = fn()
    torch.cuda.synchronize()
    print(f"  {name:28s} {1e3 * (time.perf_counter() - t):9.2f} ms")
    return r


pr = cProfile.Profile()
pr.enable()
hier = step("build_hierarchy", lambda: sf.build_hierarchy(L, k, max_dofs=2**34))
sine = lambda x: np.sin(np.pi * x)
b = step("assemble_rhs_separable", lambda: assemble_rhs_separable(hier, L, sine, 3.0 * math.pi**2))
mg = step("MultigridPreconditioner()", lambda: sf.MultigridPreconditioner(hier, sf.VCycleConfig(mode=mode)))
step("setup() (coarse LU)", mg.setup)
step("first V-cycle", lambda: mg.apply(b, L))
step("second V-cycle", lambda: mg.apply(b, L))
pr.disable()
s = io.StringIO()
pstats.Stats(pr, stream=s).sort_stats("cumulative").print_stats(30)
print(s.getvalue()[-6000:])
