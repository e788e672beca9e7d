"""Our FGMRES residual histories vs the reference's (tests/golden/solves.npz) per mode."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2407_09621_b200 as sf  # noqa: E402

g = np.load(os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "tests", "golden", "solves.npz"))
for k, lvl in [(3, 3), (3, 4), (7, 2), (7, 3)]:
    for m in ("fp64", "fp32", "fp16_ec"):
        sel = (g["k"] == k) & (g["level"] == lvl) & (g["mode"] == m) & (g["solver"] == "fgmres")
        i = int(np.flatnonzero(sel)[0])
        h = g["history"][i]
        h = h[~np.isnan(h)]
        out = sf.run_solve(k, lvl, mode=sf.PrecisionMode.parse(m))
        ours = np.array(out.report.residual_history)
        print(f"k{k} L{lvl} {m:8s} ref {np.array2string(h / h[0], precision=2)}  ours {np.array2string(ours / ours[0], precision=2)}")
for lvl in (4, 5):
    for m in ("fp64", "fp32", "fp16_ec"):
        out = sf.run_solve(7, lvl, mode=sf.PrecisionMode.parse(m), hier=sf.build_hierarchy(lvl, 7, max_dofs=2**31))
        ours = np.array(out.report.residual_history)
        print(f"k7 L{lvl} {m:8s} ours {np.array2string(ours / ours[0], precision=2)}")
