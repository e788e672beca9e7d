"""Run a few vmults / colour passes for ncu captures (never timed).

python tools/profile_vmult.py --degree 7 --level 7 --mode fp64 --reps 3 [--what vmult|colour|vcycle]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2407_09621_b200 as sf  # noqa: E402
from paper_2407_09621_b200.discretization import vmult_device  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--degree", type=int, default=7)
ap.add_argument("--level", type=int, default=7)
ap.add_argument("--mode", default="fp64")
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--what", default="vmult")
a = ap.parse_args()
mode = sf.PrecisionMode.parse(a.mode)
hier = sf.build_hierarchy(a.level, a.degree, max_dofs=2**34, min_level=max(1, a.level - (0 if a.what == "vmult" else 9)))
D = hier.n_dofs(a.level)
u = torch.randn(D, dtype=mode.torch_dtype, device="cuda")
v = torch.empty_like(u)
if a.what == "vmult":
    for _ in range(a.reps):
        vmult_device(hier, a.level, u, v, mode)
elif a.what == "colour":
    mg = sf.MultigridPreconditioner(hier, sf.VCycleConfig(mode=mode))
    for _ in range(a.reps):
        mg._smooth_device(a.level, v.zero_(), u, mode)
else:
    mg = sf.MultigridPreconditioner(hier, sf.VCycleConfig(mode=mode)).setup()
    b = u.double()
    for _ in range(a.reps):
        mg.apply(b, a.level)
torch.cuda.synchronize()
print("ok")
