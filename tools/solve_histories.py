import sys, os, json
sys.path.insert(0, os.getcwd())
import paper_2407_09621_b200 as sf
for lvl in (5, 6):
    hier = sf.build_hierarchy(lvl, 7, max_dofs=2**34)
    for m in ("fp64", "fp32", "fp16_ec"):
        out = sf.run_solve(7, lvl, mode=sf.PrecisionMode.parse(m), hier=hier)
        h = out.report.residual_history
        print(lvl, m, out.report.iterations, [f"{x/h[0]:.2e}" for x in h], f"{out.l2:.3e}", flush=True)
