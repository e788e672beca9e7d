"""One rank of the multi-process z-slab tests (launched by tests/test_slab_*.py via subprocess).

RANK / WORLD_SIZE / MASTER_ADDR / MASTER_PORT come from the environment; backend gloo.
``--case host``: CPU-only host logic (halo exchange, ghost refresh, reductions) -- no GPU needed.
``--case gpu``: every rank on cuda:0 (gloo stages through host memory), distributed vmult,
V-cycle and FGMRES checked against the single-GPU path.  Prints one JSON line per rank.
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402


def host_case(args):
    import paper_2407_09621_b200 as sf
    from paper_2407_09621_b200 import slab

    comm = slab.SlabComm()
    r, G = comm.rank, comm.world
    out = {"rank": r}
    hier = sf.build_hierarchy(args.level, args.degree)
    sls = slab.slab_levels(hier, r, G)
    out["levels"] = sorted(sls)
    sl = sls[args.level]
    D = hier.n_dofs(args.level)
    g = torch.arange(D, dtype=torch.float64)  # the global vector, known to every rank for checking
    # smoother halo: extended slab = global range [z0 - h_lo, z0 + nz + h_hi) cells
    x_ext = torch.full((sl.ext_dofs,), -1.0, dtype=torch.float64)
    x_ext[sl.local_slice] = g[sl.global_slice]
    slab.refresh_ghost_cells(comm, sl, x_ext)
    lo = (sl.z0 - sl.h_lo) * sl.cell_layer
    out["ghost_cells_ok"] = bool(torch.equal(x_ext, g[lo:lo + sl.ext_dofs]))
    # vmult halo: K planes below / above
    u = g[sl.global_slice].clone()
    Kp = sl.K * sl.plane
    glo, ghi = torch.zeros(Kp, dtype=torch.float64), torch.zeros(Kp, dtype=torch.float64)
    slab.exchange_face_planes(comm, sl, u, glo, ghi)
    a, b = sl.global_slice.start, sl.global_slice.stop
    ok = True
    if comm.lo is not None:
        ok &= bool(torch.equal(glo, g[a - Kp:a]))
    if comm.hi is not None:
        ok &= bool(torch.equal(ghi, g[b:b + Kp]))
    out["face_planes_ok"] = ok
    # reductions: sum of local dots == global dot; gather == global vector
    rng = np.random.default_rng(5)
    x = torch.from_numpy(rng.standard_normal(D))
    part = torch.tensor([float(x[a:b] @ x[a:b])], dtype=torch.float64)
    comm.allreduce_(part)
    out["dot_rel_err"] = abs(float(part) - float(x @ x)) / float(x @ x)
    out["gather_ok"] = bool(torch.equal(comm.allgather_cat(x[a:b].clone()), x))
    return out


def gpu_case(args):
    import paper_2407_09621_b200 as sf
    from paper_2407_09621_b200 import slab
    from paper_2407_09621_b200.discretization import vmult_device

    torch.cuda.set_device(args.device)
    comm = slab.SlabComm()
    r = comm.rank
    k, L = args.degree, args.level
    hier = sf.build_hierarchy(L, k, max_dofs=2**30)
    D = hier.n_dofs(L)
    out = {"rank": r}
    gen = np.random.default_rng(11)
    ug = torch.from_numpy(gen.standard_normal(D)).cuda()
    # reference: single-GPU vmult of the global vector
    vg = torch.empty_like(ug)
    vmult_device(hier, L, ug, vg, sf.PrecisionMode.FP64)
    op = slab.DistributedOperator(hier, L, comm)
    sl = op.slab
    vloc = op(ug[sl.global_slice].contiguous())
    ref = vg[sl.global_slice]
    out["vmult_rel_err"] = float((vloc - ref).norm() / ref.norm())
    # weak-scaling brick (bench.py --gpus N): rank cubes stacked along z vs one brick vmult
    from paper_2407_09621_b200 import _native

    n = hier.n_cells(L)
    G = comm.world
    ub = torch.from_numpy(gen.standard_normal(D * G)).cuda()
    vb = torch.empty_like(ub)
    vmult_device(hier, L, ub, vb, sf.PrecisionMode.FP64, grid=_native.SfGrid(n, n, n * G, None, None))
    wop = slab.DistributedOperator.weak(hier, L, comm)
    vw = wop(ub[r * D:(r + 1) * D].contiguous())
    refw = vb[r * D:(r + 1) * D]
    out["weak_vmult_rel_err"] = float((vw - refw).norm() / refw.norm())
    # V-cycle: distributed vs single-GPU
    mode = sf.PrecisionMode.parse(args.mode)
    cfg = sf.VCycleConfig(mode=mode)
    mg1 = sf.MultigridPreconditioner(hier, cfg)
    bg = ug / ug.norm()
    z1 = mg1.apply(bg, L)
    dm = slab.DistributedMultigrid(hier, sf.VCycleConfig(mode=mode), comm).setup()
    zl = dm.apply(bg[sl.global_slice].contiguous())
    ref = z1[sl.global_slice]
    out["vcycle_rel_err"] = float((zl - ref).norm() / ref.norm())
    out["agglomerated_below"] = dm.lowest
    # FGMRES on slabs vs single GPU (manufactured sine problem)
    if args.solve:
        import math

        from paper_2407_09621_b200.discretization import assemble_rhs_separable
        from paper_2407_09621_b200.experiments import make_operator

        sine = lambda x: np.sin(np.pi * x)
        b = assemble_rhs_separable(hier, L, sine, 3.0 * math.pi**2)
        x1, rep1 = sf.fgmres(make_operator(hier, L), lambda v: mg1.apply(v, L), b, tol=1e-8)
        xl, repl = slab.fgmres_distributed(op, dm, b[sl.global_slice].contiguous(), comm, tol=1e-8)
        out["its_single"], out["its_dist"] = rep1.iterations, repl.iterations
        ref = x1[sl.global_slice]
        out["solve_rel_err"] = float((xl - ref).norm() / ref.norm())
        out["hist_single"] = [float(h) for h in rep1.residual_history]
        out["hist_dist"] = [float(h) for h in repl.residual_history]
        # the public distributed driver: same iterations, same L2 error as run_solve
        ref = sf.run_solve(k, L, mode=mode, hier=hier)
        _, rep_d, l2_d = slab.run_solve_distributed(k, L, comm, mode=mode, hier=hier)
        out["run_solve_its"], out["run_solve_dist_its"] = ref.report.iterations, rep_d.iterations
        out["run_solve_l2"], out["run_solve_dist_l2"] = ref.l2, l2_d
    return out


def memory_case(args):
    """Peak device memory of one rank's distributed solve (O(local DoF): slab-local load vector, slab
    V-cycle buffers, slab Krylov bases; only the agglomerated coarse levels are replicated)."""
    import paper_2407_09621_b200 as sf
    from paper_2407_09621_b200 import slab

    torch.cuda.set_device(args.device)
    comm = slab.SlabComm()
    k, L = args.degree, args.level
    hier = sf.build_hierarchy(L, k, max_dofs=2**30)
    mode = sf.PrecisionMode.parse(args.mode)
    torch.cuda.synchronize()
    torch.cuda.reset_peak_memory_stats()
    base = torch.cuda.memory_allocated()
    _, rep, l2 = slab.run_solve_distributed(k, L, comm, mode=mode, hier=hier)
    torch.cuda.synchronize()
    return {"rank": comm.rank, "peak_bytes": torch.cuda.max_memory_allocated() - base, "its": rep.iterations,
            "l2": l2, "global_dofs": hier.n_dofs(L)}


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--case", default="host")
    ap.add_argument("--degree", type=int, default=1)
    ap.add_argument("--level", type=int, default=3)
    ap.add_argument("--mode", default="fp64")
    ap.add_argument("--solve", action="store_true")
    ap.add_argument("--backend", default="gloo")
    a = ap.parse_args()
    a.device = 0
    if a.backend == "nccl":  # one GPU per rank (the driver's multi-GPU boxes)
        a.device = int(os.environ.get("LOCAL_RANK", 0))
        torch.cuda.set_device(a.device)
        dist.init_process_group("nccl", device_id=torch.device("cuda", a.device))
    else:
        dist.init_process_group("gloo")
    res = {"host": host_case, "gpu": gpu_case, "memory": memory_case}[a.case](a)
    print("RESULT " + json.dumps(res), flush=True)
    dist.barrier()
    dist.destroy_process_group()
