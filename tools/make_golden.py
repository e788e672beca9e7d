"""Generate golden vectors for the hot path by importing the REFERENCE itself.

Run in the build container only (``/root/reference`` does not exist on the GPU
box):  ``python tools/make_golden.py``.  Imports ``sumfact`` from
``/root/reference/pkg/src`` with its numpy backend (``SUMFACT_PURE_PYTHON=1``,
the reference's own ``_core/fallback.py``), calls the reference's public API on
seeded inputs and writes ``tests/golden/*.npz``.  The committed fixtures pin
``oracle/port.py`` (tests/test_oracle_golden.py) and the GPU path
(tests/test_gpu_*.py).
"""
import os
import sys
import time

os.environ.setdefault("SUMFACT_PURE_PYTHON", "1")
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, "/root/reference/pkg/tests")

import numpy as np  # noqa: E402

import sumfact  # noqa: E402
from sumfact.basis import embedding_1d  # noqa: E402
from sumfact.discretization import apply_operator, build_hierarchy  # noqa: E402
from sumfact.experiments import run_solve  # noqa: E402
from sumfact.multigrid import MultigridPreconditioner, VCycleConfig, prolongate, restrict  # noqa: E402
from sumfact.precision import PrecisionMode, demote16  # noqa: E402

OUT = os.path.join(os.path.dirname(__file__), "..", "tests", "golden")
MODES = [PrecisionMode.FP64, PrecisionMode.FP32, PrecisionMode.FP16, PrecisionMode.FP16_EC]


def save(name, **arrays):
    path = os.path.join(OUT, name + ".npz")
    np.savez_compressed(path, **arrays)
    print(f"wrote {path} ({os.path.getsize(path) / 1024:.0f} KiB)", flush=True)


def matrices():
    out = {}
    for k in (1, 2, 3, 7):
        hier = build_hierarchy(3, k)
        out[f"k{k}_P"] = embedding_1d(k)
        for lvl in (1, 2, 3):
            lm = hier.matrices(lvl)
            for name in ("M_cell", "L_cell", "M_patch", "L_tile", "B_left", "B_right", "F_cross"):
                out[f"k{k}_l{lvl}_{name}"] = getattr(lm, name)
            for (lb, rb), L in lm.L_smooth.items():
                out[f"k{k}_l{lvl}_Ls{int(lb)}{int(rb)}"] = L
    save("matrices", **out)


VMULT_CASES = [(1, 1), (1, 2), (2, 2), (3, 2), (3, 3), (7, 1), (7, 2)]


def vmult():
    out = {}
    for k, lvl in VMULT_CASES:
        hier = build_hierarchy(lvl, k)
        u = np.random.default_rng(0).standard_normal(hier.n_dofs(lvl))
        for mode in MODES:
            out[f"k{k}_l{lvl}_{mode.value}"] = apply_operator(hier, lvl, u, mode)
    save("vmult", **out)


def dense():
    from sipg_oracle import assemble_sipg_dense
    save("sipg_dense", k1_l1=assemble_sipg_dense(1, 1, 3), k1_l2=assemble_sipg_dense(1, 2, 3),
         k2_l1=assemble_sipg_dense(2, 1, 3))


def smoother_transfers():
    out = {}
    for k, lvl in [(1, 2), (2, 2), (3, 2), (7, 2), (1, 3)]:
        hier = build_hierarchy(lvl, k)
        D = hier.n_dofs(lvl)
        # unit-norm inputs: the V-cycle only ever sees unit-scale vectors, and
        # N(0,1) entries overflow binary16 in the Q7 residual (reference -> inf)
        x = np.random.default_rng(1).standard_normal(D)
        x /= np.linalg.norm(x)
        b = np.random.default_rng(2).standard_normal(D)
        b /= np.linalg.norm(b)
        for mode in MODES:
            mg = MultigridPreconditioner(hier, VCycleConfig(mode=mode))
            out[f"smooth_k{k}_l{lvl}_{mode.value}"] = mg.smooth(lvl, x, b, mode)
            out[f"restrict_k{k}_l{lvl}_{mode.value}"] = restrict(hier, lvl, x, mode)
            e = np.random.default_rng(3).standard_normal(hier.n_dofs(lvl - 1))
            out[f"prolong_k{k}_l{lvl}_{mode.value}"] = prolongate(hier, lvl - 1, e, mode)
    save("smoother", **out)


def vcycles():
    out = {}
    for k, lvl in [(1, 3), (3, 3), (2, 2), (7, 2)]:
        hier = build_hierarchy(lvl, k)
        b = np.random.default_rng(4).standard_normal(hier.n_dofs(lvl))
        b /= np.linalg.norm(b)  # unit norm, like the Arnoldi vectors the V-cycle sees
        for mode in MODES:
            mg = MultigridPreconditioner(hier, VCycleConfig(mode=mode))
            out[f"vcycle_k{k}_l{lvl}_{mode.value}"] = mg.apply(b, lvl)
    save("vcycle", **out)


def solves():
    rows = []
    cases = [(1, 2), (1, 3), (1, 4), (2, 3), (3, 2), (3, 3), (3, 4), (7, 2), (7, 3)]
    for k, lvl in cases:
        for mode in MODES:
            for solver in ("fgmres", "gmres"):
                if solver == "gmres" and mode is not PrecisionMode.FP16:
                    continue
                t0 = time.perf_counter()
                o = run_solve(k, lvl, mode=mode, solver=solver)
                r = o.report
                rows.append((k, lvl, mode.value, solver, r.iterations, o.l2, o.h1,
                             r.final_relative_residual, list(map(float, r.residual_history))))
                print(f"  solve k={k} L={lvl} {mode.value} {solver}: its={r.iterations} "
                      f"l2={o.l2:.6e} ({time.perf_counter() - t0:.1f}s)", flush=True)
    hist = np.full((len(rows), 101), np.nan)
    for i, row in enumerate(rows):
        hist[i, :len(row[8])] = row[8]
    save("solves", k=np.array([r[0] for r in rows]), level=np.array([r[1] for r in rows]),
         mode=np.array([r[2] for r in rows]), solver=np.array([r[3] for r in rows]),
         iterations=np.array([r[4] for r in rows]), l2=np.array([r[5] for r in rows]),
         h1=np.array([r[6] for r in rows]), final_rel=np.array([r[7] for r in rows]),
         history=hist)


def half():
    rng = np.random.default_rng(5)
    specials = np.array([0.0, -0.0, 65504.0, 65519.99, 65520.0, 6.1035156e-05, 6.0e-05, 5.96e-08,
                         2.98e-08, 2.99e-08, 1.0, 1.0004883, 1.0009766, 1.00073242, -2.5e-06,
                         np.inf, -np.inf, 1e-30, 7e4], dtype=np.float32)
    x = np.concatenate([specials,
                        rng.standard_normal(4000).astype(np.float32),
                        (rng.standard_normal(4000) * 1e-5).astype(np.float32),
                        (rng.standard_normal(2000) * 3e4).astype(np.float32),
                        np.float32(2.0) ** rng.integers(-30, 17, 2000).astype(np.float32)
                        * rng.uniform(1, 2, 2000).astype(np.float32)])
    save("half", x=x, demoted=demote16(x))


def softfloat():
    """precision.py:60-197 through the reference itself: its binary16 fixture (tests/data/half_reference.txt,
    fp32 bits -> fp16 bits), to_half on NaN payloads / edge values, from_half of all 65536 patterns, ec_split
    and ec_matmul (all three refine choices)."""
    from sumfact.precision import ec_matmul, ec_split, from_half, to_half

    lines = open("/root/reference/pkg/tests/data/half_reference.txt").read().splitlines()
    pairs = [ln.split() for ln in lines if not ln.startswith("#")]
    fix_x = np.array([int(a, 16) for a, _ in pairs], dtype=np.uint32)
    fix_h = np.array([int(b, 16) for _, b in pairs], dtype=np.uint16)
    nan_bits = np.array([0x7FC00000, 0xFFC00000, 0x7F800001, 0xFF800001, 0x7FA00000, 0x7F802000, 0x7FFFFFFF,
                         0x00000001, 0x80000001, 0x007FFFFF, 0x33000000, 0x33000001, 0x33800000, 0x477FEFFF,
                         0x477FF000, 0x7F7FFFFF], dtype=np.uint32)
    edge_x = np.concatenate([nan_bits, fix_x[:64]]).view(np.float32)
    all_h = np.arange(65536, dtype=np.uint32).astype(np.uint16)
    rng = np.random.default_rng(9)
    ec_x = np.concatenate([(rng.standard_normal(3000) * 10.0 ** rng.uniform(-6, 4, 3000)).astype(np.float32),
                           np.array([65504.0, -65504.0, 0.0, -0.0, 6e-8, 1.0 / 3.0], dtype=np.float32)])
    pr = ec_split(ec_x)
    A = (rng.standard_normal((19, 23)) * 3).astype(np.float32)
    B = (rng.standard_normal((23, 17)) * 0.1).astype(np.float32)
    ea, eb = ec_split(A.ravel()), ec_split(B.ravel())
    ea = type(ea)(main=ea.main.reshape(A.shape), residual=ea.residual.reshape(A.shape))
    eb = type(eb)(main=eb.main.reshape(B.shape), residual=eb.residual.reshape(B.shape))
    save("softfloat", fix_x=fix_x, fix_h=fix_h, edge_x=edge_x, edge_h=to_half(edge_x),
         from_half_all=from_half(all_h).view(np.uint32), ec_x=ec_x, ec_main=pr.main, ec_resid=pr.residual,
         mm_a=A, mm_b=B, **{f"mm_{r}": ec_matmul(ea, eb, refine=r) for r in ("both", "left", "right")})


def error_profiles():
    """Reference experiments.error_profile(7, 4, (fp32, fp16, fp16_ec), seed=0) -> JSON rows
    (acceptance criterion 9 inputs, tests/test_gpu_acceptance.py)."""
    import json

    from sumfact.experiments import error_profile

    rows = error_profile(7, 4, (PrecisionMode.FP32, PrecisionMode.FP16, PrecisionMode.FP16_EC), seed=0)
    path = os.path.join(OUT, "error_profile_k7_l4.json")
    with open(path, "w") as fh:
        json.dump(rows, fh, indent=0)
    print(f"wrote {path}", flush=True)


def quadrature():
    """Pre/post-processing with general (non-separable) data: assemble_rhs with a boundary term g,
    l2_error and h1_seminorm_error of a seeded DoF vector (discretization.py:317-459)."""
    from sumfact.discretization import assemble_rhs, h1_seminorm_error, l2_error

    f = lambda x, y, z: np.exp(x) * np.cos(2.0 * y + z) + x * y * z
    g = lambda x, y, z: np.sin(3.0 * x + y) - z * z + 0.5
    ex = lambda x, y, z: np.cos(x * y) + np.exp(z) * x
    gr = lambda x, y, z: (-y * np.sin(x * y) + np.exp(z), -x * np.sin(x * y), np.exp(z) * x)
    out = {}
    for k, lvl in [(1, 2), (2, 2), (3, 2), (7, 1), (7, 2)]:
        hier = build_hierarchy(lvl, k)
        out[f"k{k}_l{lvl}_rhs_f"] = assemble_rhs(hier, lvl, f)
        out[f"k{k}_l{lvl}_rhs_fg"] = assemble_rhs(hier, lvl, f, g)
        u = np.random.default_rng(5).standard_normal(hier.n_dofs(lvl))
        out[f"k{k}_l{lvl}_l2"] = np.array(l2_error(hier, lvl, u, ex))
        out[f"k{k}_l{lvl}_h1"] = np.array(h1_seminorm_error(hier, lvl, u, gr))
    save("quadrature", **out)


if __name__ == "__main__" and len(sys.argv) > 1:
    globals()[sys.argv[1]]()
    sys.exit(0)

if __name__ == "__main__":
    os.makedirs(OUT, exist_ok=True)
    print("reference sumfact", sumfact.__version__, "compiled core:", sumfact.HAVE_COMPILED)
    which = sys.argv[1:] or ["matrices", "vmult", "dense", "smoother_transfers", "vcycles", "half", "solves", "softfloat"]
    for w in which:
        globals()[w]()
