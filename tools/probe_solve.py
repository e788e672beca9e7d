"""Print FGMRES residual histories per precision mode and level (diagnostics)."""
import json
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2407_09621_b200 as sf  # noqa: E402
from paper_2407_09621_b200.discretization import assemble_rhs_separable, l2_error_separable  # noqa: E402
from paper_2407_09621_b200.experiments import make_operator  # noqa: E402

k = int(sys.argv[1])
for lvl in map(int, sys.argv[2].split(",")):
    hier = sf.build_hierarchy(lvl, k, max_dofs=2**34)
    sine = lambda x: np.sin(np.pi * x)
    b = assemble_rhs_separable(hier, lvl, sine, 3 * math.pi**2)
    for m in sys.argv[3].split(","):
        mode = sf.PrecisionMode.parse(m)
        mg = sf.MultigridPreconditioner(hier, sf.VCycleConfig(mode=mode))
        x, rep = sf.fgmres(make_operator(hier, lvl), lambda v: mg.apply(v, lvl), b, tol=1e-8, maxit=25)
        print(json.dumps({"k": k, "level": lvl, "mode": m, "its": rep.iterations,
                          "l2": l2_error_separable(hier, lvl, x, sine),
                          "hist": [f"{h / rep.residual_history[0]:.2e}" for h in rep.residual_history]}), flush=True)
        del mg, x, rep
        torch.cuda.empty_cache()
