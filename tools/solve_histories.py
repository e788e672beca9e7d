"""Relative residual histories and L2 errors of the manufactured solve per mode (bench sizes)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2407_09621_b200 as sf  # noqa: E402

cases = [(7, 6), (7, 5), (3, 7)] if len(sys.argv) < 2 else [tuple(map(int, a.split(","))) for a in sys.argv[1:]]
for k, L in cases:
    hier = sf.build_hierarchy(L, k, max_dofs=2**34)
    for m in (sf.PrecisionMode.FP64, sf.PrecisionMode.FP16_EC, sf.PrecisionMode.FP32):
        r = sf.run_solve(k, L, m, hier=hier)
        h = r.report.residual_history
        print(k, L, m.value, r.report.iterations, " ".join(f"{x / h[0]:.2e}" for x in h), f"l2={r.l2:.3e}",
              flush=True)
