"""CPU baseline of the reference path as BASELINE.md §3 defines it (TEST/MEASUREMENT INFRASTRUCTURE).

The reference as shipped is single-threaded (pkg/README.md:85-87, src/cli.py:7-9): every case below runs
in a child process pinned to ONE core (sched_setaffinity, BLAS threads 1) with both of the reference's
contraction backends -- its compiled Cython kernel (oracle/_ref, built from the reference's own sources)
and its numpy einsum fallback -- best of 3 after a warm-up, and reports the faster; plus an all-cores
figure (the same algorithm with the contractions as threaded BLAS GEMMs).  Cases:
  C1  vmult Q7 L4 (16^3 cells, 2.1 M DoF), fp64          -- BASELINE configs[0]
  C1b vmult Q3 L5 (2.1 M DoF), fp64
  C3  one smooth() step (8 colours), Q3 L4 and Q7 L3, fp64 (reduced sizes: Q3 L7 takes ~10 min per step)
  C4  run_solve (FGMRES + V-cycle), Q3 L4 fp64, setup (hierarchy, eigh, coarse LU) excluded
python -m oracle.cpu_timing [--quick] [--out profiles/r02_cpu_baseline.json]
Only bench.py (cpu_baseline / --impl reference) and this CLI use it; the product never does.
"""
import argparse
import json
import multiprocessing as mp
import os
import platform
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return platform.processor() or "unknown"


def _child(case, backend, reps, q):
    import numpy as np
    from threadpoolctl import threadpool_limits

    os.sched_setaffinity(0, {sorted(os.sched_getaffinity(0))[0]})
    from oracle import port

    try:
        port.set_backend(backend)
    except RuntimeError as exc:
        q.put({"error": str(exc)})
        return
    kind, k, lvl = case
    with threadpool_limits(limits=1):
        H = port.Hierarchy(lvl, k)
        n = H.n_dofs(lvl)
        if kind == "vmult":
            u = np.random.default_rng(0).standard_normal(n)
            fn = lambda: port.apply_operator(H, lvl, u)
        elif kind == "smooth":
            mg = port.VCycle(H)
            x = np.random.default_rng(1).standard_normal(n)
            b = np.random.default_rng(2).standard_normal(n)
            fn = lambda: mg.smooth(lvl, x, b)
        else:  # solve: setup (hierarchy, eigh, coarse LU) outside the timed region
            mg = port.VCycle(H)
            mg._factor("fp64")
            bvec = port.assemble_rhs(H, lvl, port.sine_rhs)
            fn = lambda: port.gmres_driver(lambda v: port.apply_operator(H, lvl, v), lambda v: mg.apply(v, lvl),
                                           bvec, tol=1e-8, maxit=100, flexible=True)
        fn()  # warm-up
        best = float("inf")
        for _ in range(reps):
            t0 = time.perf_counter()
            fn()
            best = min(best, time.perf_counter() - t0)
    q.put({"seconds": best, "dofs": n})


def time_case(case, backend, reps=3):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    p = ctx.Process(target=_child, args=(case, backend, reps, q))
    p.start()
    res = q.get()
    p.join()
    return res


def all_cores_vmult(k=7, lvl=5, reps=2):
    import numpy as np

    from oracle import port

    threads = port.default_threads()
    H = port.Hierarchy(lvl, k)
    u = np.random.default_rng(0).standard_normal(H.n_dofs(lvl))
    port.apply_operator(H, lvl, u, "fp64", threads)
    best = float("inf")
    for _ in range(reps):
        t0 = time.perf_counter()
        port.apply_operator(H, lvl, u, "fp64", threads)
        best = min(best, time.perf_counter() - t0)
    return {"seconds": best, "dofs": H.n_dofs(lvl), "threads": threads, "case": f"vmult Q{k} L{lvl}"}


def run(cases, reps=3, verbose=False):
    out = {"cpu_model": cpu_model(), "nproc": os.cpu_count(), "cores_used": 1,
           "method": "child process pinned to one core (sched_setaffinity), BLAS threads 1, best of "
                     f"{reps} after a warm-up; backends: reference compiled kernel (oracle/_ref) and numpy "
                     "einsum fallback; 'best' = the faster", "cases": {}}
    for case in cases:
        name = f"{case[0]} Q{case[1]} L{case[2]}"
        r = {b: time_case(case, b, reps) for b in ("compiled", "einsum")}
        ok = {b: v for b, v in r.items() if "seconds" in v}
        best = min(ok, key=lambda b: ok[b]["seconds"])
        out["cases"][name] = {"seconds": {b: v.get("seconds") for b, v in r.items()}, "best_backend": best,
                              "dofs": ok[best]["dofs"],
                              "mdofs_per_s": ok[best]["dofs"] / ok[best]["seconds"] / 1e6}
        if verbose:  # (bench.py prints exactly one JSON line: silent there)
            print(name, out["cases"][name], flush=True)
    return out


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--quick", action="store_true")
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    cases = [("vmult", 7, 4)] if a.quick else [("vmult", 7, 4), ("vmult", 3, 5), ("smooth", 3, 4), ("smooth", 7, 3),
                                               ("solve", 3, 4)]
    res = run(cases, verbose=True)
    res["all_cores"] = all_cores_vmult()
    print(json.dumps(res, indent=1))
    if a.out:
        json.dump(res, open(a.out, "w"), indent=1)
