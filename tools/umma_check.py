"""A/B of the tcgen05 binary16 kernels against the mma.sync ones and the fp64 vmult (run under gpurun).
python tools/umma_check.py            -> spawns SUMFACT_UMMA=0 / 1 children, prints relative differences"""
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
CASES = [(7, 2), (7, 3), (7, 4), (7, 6)]


def child(out):
    import numpy as np
    import torch

    import paper_2407_09621_b200 as sf

    res = {}
    for k, lvl in CASES:
        hier = sf.build_hierarchy(lvl, k, max_dofs=2**31)
        g = torch.Generator(device="cuda").manual_seed(lvl)
        u = torch.randn(hier.n_dofs(lvl), dtype=torch.float64, device="cuda", generator=g)
        res[f"k{k}_l{lvl}_fp64"] = sf.apply_operator(hier, lvl, u).cpu().numpy()
        for m in ("fp16", "fp16_ec"):
            res[f"k{k}_l{lvl}_{m}"] = sf.apply_operator(hier, lvl, u.float(), sf.PrecisionMode.parse(m)).cpu().numpy()
    np.savez(out, **res)


if __name__ == "__main__":
    if len(sys.argv) > 1:
        child(sys.argv[1])
        sys.exit(0)
    import numpy as np

    outs = {}
    for flag in ("0", "1"):
        path = f"/tmp/umma_{flag}.npz"
        r = subprocess.run([sys.executable, __file__, path], env=dict(os.environ, SUMFACT_UMMA=flag),
                           capture_output=True, text=True)
        if r.returncode:
            print("child failed", flag, r.stderr[-3000:])
            sys.exit(1)
        outs[flag] = np.load(path)
    a, b = outs["0"], outs["1"]
    for key in a.files:
        if key.endswith("fp64"):
            continue
        k64 = "_".join(key.split("_")[:2]) + "_fp64"
        r64 = a[k64]
        rel = lambda x, y: float(np.linalg.norm(x.astype(np.float64) - y) / np.linalg.norm(y))
        print(f"{key:18s} mma.sync vs fp64 {rel(a[key], r64):.3e}   tcgen05 vs fp64 {rel(b[key], r64):.3e}   "
              f"tcgen05 vs mma.sync {rel(b[key], a[key].astype(np.float64)):.3e}")
