"""Small invocations of every hot kernel in every mode, for compute-sanitizer
(memcheck / racecheck / synccheck / initcheck): tools/sanitize.sh runs this
script under each tool and keeps the logs in profiles/.

Covers: vmult (every degree, all modes, tiled and generic grids), the smoother
colour pass (all 8 colours), fused residual+restriction, prolongation+add, the
V-cycle, the FGMRES vector kernels, the generic contraction and the binary16
primitives.  Sizes are the smallest that exercise tile neighbours (>= 2 tiles
per axis for the 16-point line kernels)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2407_09621_b200 as sf  # noqa: E402
from paper_2407_09621_b200 import device  # noqa: E402

P = sf.PrecisionMode
MODES = [P.FP64, P.FP32, P.FP16, P.FP16_EC]
quick = "--quick" in sys.argv
# (degree, level): Q7 2 / 4 tiles per axis; Q3/Q1 line tiles with 2 tiles per axis; CUDA-core degrees
CASES = [(7, 2), (7, 3), (3, 3), (3, 4), (1, 4), (1, 5), (2, 3), (5, 2)]
if quick:
    CASES = [(7, 3), (3, 4), (1, 5)]


def run():
    g = torch.Generator(device="cuda")
    g.manual_seed(0)
    for k, lvl in CASES:
        hier = sf.build_hierarchy(lvl, k)
        n = hier.n_dofs(lvl)
        for mode in MODES:
            u = torch.randn(n, dtype=torch.float64, device="cuda", generator=g).to(mode.torch_dtype)
            v = sf.apply_operator(hier, lvl, u, mode)
            mg = sf.MultigridPreconditioner(hier, sf.VCycleConfig(mode=mode))
            b = torch.randn(n, dtype=torch.float64, device="cuda", generator=g)
            x = mg.smooth(lvl, torch.zeros_like(b), b, mode)
            z = mg.apply(b, lvl)
            torch.cuda.synchronize()
            assert torch.isfinite(v).all() and torch.isfinite(x).all() and torch.isfinite(z).all(), (k, lvl, mode)
            print(f"k={k} L={lvl} {mode.value}: vmult/smooth/vcycle ok", flush=True)
    # FGMRES vector kernels (dots, fused MGS, lincomb, div) through one short solve
    out = sf.run_solve(3, 3, mode=P.FP16_EC)
    assert out.report.converged
    xs = [torch.randn(1000, dtype=torch.float64, device="cuda") for _ in range(3)]
    o = torch.empty(1, dtype=torch.float64, device="cuda")
    device.dot2(xs[0], xs[1], xs[2], o, o.clone())
    device.lincomb(xs, [1.0, 2.0, 3.0], torch.empty(1000, dtype=torch.float64, device="cuda"))
    # generic contraction + binary16 primitives
    m = np.random.default_rng(0).standard_normal((5, 6))
    w = np.random.default_rng(1).standard_normal((3, 6, 4))
    for mode in MODES:
        sf.contract_mode(m, w, 1, mode)
    sf.demote16(np.linspace(-1e5, 1e5, 1001, dtype=np.float32))
    torch.cuda.synchronize()
    print("sanitize cases done", flush=True)


if __name__ == "__main__":
    run()
