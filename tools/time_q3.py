"""Q3 level 7 (1.34e8 DoF) colour pass per mode + EC solve launch composition helper (CUDA events)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2407_09621_b200 as sf  # noqa: E402
from paper_2407_09621_b200 import _native, device as dev  # noqa: E402


def timeit(fn, reps=10):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


P = sf.PrecisionMode
k, L = int(sys.argv[1]) if len(sys.argv) > 1 else 3, int(sys.argv[2]) if len(sys.argv) > 2 else 7
h = sf.build_hierarchy(L, k, max_dofs=2**34)
D = h.n_dofs(L)
out = {"k": k, "level": L}
for mode in (P.FP64, P.FP16_EC):
    mg = sf.MultigridPreconditioner(h, sf.VCycleConfig(mode=mode))
    x = torch.zeros(D, dtype=mode.torch_dtype, device="cuda")
    b = torch.randn(D, dtype=mode.torch_dtype, device="cuda")
    xn = torch.empty_like(x)
    lm = h.matrices(L)
    for shift in ((0, 0, 0), (1, 1, 1)):
        sh = mg._shift_arrays[shift]

        def colour():
            _native.check(_native.lib().sf_smooth_colour(mode.code, k, h.grid(L), sh, _native.host_ptr(lm.cell_op),
                                                         _native.host_ptr(mg.solvers[L].table), dev.ptr(x),
                                                         dev.ptr(b), dev.ptr(xn), dev.stream_ptr()), "colour")
        out[f"colour_{mode.value}_{''.join(map(str, shift))}_ms"] = timeit(colour)
    out[f"smooth_step_{mode.value}_ms"] = timeit(lambda: mg._smooth_device(L, x, b, mode), reps=3)
    r = torch.empty_like(x)
    out[f"vmult_{mode.value}_ms"] = timeit(lambda: sf.discretization.vmult_device(h, L, x, r, mode))
print(json.dumps(out))
