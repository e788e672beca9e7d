"""Warm kernel-time breakdown of one FGMRES+MG solve (torch.profiler / CUPTI): python tools/solve_profile.py k L mode"""
import collections
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2407_09621_b200 as sf  # noqa: E402
from paper_2407_09621_b200.discretization import assemble_rhs_separable  # noqa: E402
from paper_2407_09621_b200.experiments import make_operator  # noqa: E402

k, L, mode = int(sys.argv[1]), int(sys.argv[2]), sf.PrecisionMode.parse(sys.argv[3])
hier = sf.build_hierarchy(L, k, max_dofs=2**34)
b = assemble_rhs_separable(hier, L, lambda x: np.sin(np.pi * x), 3.0 * math.pi ** 2)
mg = sf.MultigridPreconditioner(hier, sf.VCycleConfig(mode=mode)).setup()
A = make_operator(hier, L)
M = lambda v: mg.apply(v, L)
for _ in range(2):
    sf.fgmres(A, M, b, tol=1e-8)
torch.cuda.synchronize()
with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA]) as prof:
    x, rep = sf.fgmres(A, M, b, tol=1e-8)
    torch.cuda.synchronize()
agg = collections.defaultdict(lambda: [0, 0.0])
for e in prof.events():
    if e.device_type == torch.autograd.DeviceType.CUDA:
        name = e.name.replace("void ", "").replace("(anonymous namespace)::", "")
        name = name.split("(")[0][:60] or e.name[:60]
        agg[name][0] += 1
        agg[name][1] += e.device_time_total / 1000.0 if hasattr(e, "device_time_total") else e.cuda_time_total / 1000.0
tot = sum(v[1] for v in agg.values())
print(f"k{k} L{L} {mode.value}: {rep.iterations} its, kernel time {tot:.2f} ms")
for n, (c, t) in sorted(agg.items(), key=lambda kv: -kv[1][1])[:14]:
    print(f"  {t:8.2f} ms {100 * t / tot:5.1f}%  x{c:<4d} {n}")
