"""Benchmark of the B200 SIPG hot path (driver contract: one JSON line on rank 0).

Headline workload (N=1): FP64 Q7 DG-SIPG Laplace vmult on the 128^3-cell unit
cube, 1,073,741,824 DoF (BASELINE.json configs[1], "~1e9 DoF on 1 B200").
value = GDoF/s with u and v resident in HBM (8.6 GB each, far larger than the
126 MB L2, so no flush is needed between steps).  e2e = the same vmult through
the public API ``apply_operator`` with pinned HOST buffers, H2D + D2H inside
the timed region.

N>1 (torchrun): weak scaling -- every rank owns a 128^3-cell z-slab of a
128 x 128 x (128 N) brick, exchanges its K-plane ghost layers with the z
neighbours over NCCL each step, then runs the vmult with ghost pointers.

--impl reference: the reference algorithm's CPU implementation (the numpy
oracle port of src/discretization.py:216-266, all host threads) on a bounded
sample of the same workload (Q7 level 5, 16.8 M DoF), rank 0 only.
"""
from __future__ import annotations

import argparse
import datetime
import json
import math
import os
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "Laplace vmult GDoF/s & TFLOPS (FP64/FP16); FGMRES+MG time-to-solution"
UNIT = "GDoF/s"
FP64_PEAK_TFLOPS = 37.1  # measured DMMA.8x8x4 peak, profiles/r01_microbench_fp64.md (MEASURED_PEAKS has no fp64)


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            m = json.load(fh)
        return float(m["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def ref_flops_per_dof(k, level):
    """the reference schedule, 36N + 18N/p flop/DoF (N = 2(k+1), p = 2^(l-1))."""
    N = 2 * (k + 1)
    return 36 * N + 18 * N / 2 ** (level - 1)


def kernel_flops_per_dof(k):
    """Tensor-pipe flops the FP64 vmult kernel executes per DoF: one 16^3-point tile
    (4096 DoF) issues 1376 DMMA.8x8x4 (512 flop each): x stage 384, y stage 512, z stage 384, trace-plane
    masses 96 -- for Q7 (2x2x2-cell tiles) and for Q3/Q1 (16-point line tiles of 4 / 8 cells) alike.
    This is the figure ncu's DMMA-pipe utilisation measures, so frac and the pipe % agree."""
    if k in (1, 3, 7):
        return 1376 * 512 / 4096
    K = k + 1  # CUDA-core tile engine: line stages 7K + 9 - 3/K MACs + traces/masses
    return 2 * (7 * K + 9 - 3.0 / K + 3.0 * (K - 1) / K + 6.0) + 2


class ClockSampler:
    """nvidia-smi clocks and throttle reasons during the timed region: a background `nvidia-smi -lms 100` started
    (and waited for) before the warm-up, its samples kept only inside the host window of the timed region
    (timestamp field), plus one synchronous query issued while the timed steps are queued on the GPU -- so a short
    timed region still has samples."""

    Q = ("timestamp,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index):
        self.gpu = gpu_index
        self.path = tempfile.mktemp(suffix=".csv")
        self.fh = open(self.path, "w")
        self.extra = []
        self.t0 = self.t1 = None
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={gpu_index}", f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"], stdout=self.fh,
                                         stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def wait_ready(self, timeout=5.0):
        t = time.time()
        while self.proc is not None and time.time() - t < timeout:
            self.fh.flush()
            if os.path.getsize(self.path) > 0:
                return
            time.sleep(0.05)

    def start(self):
        self.t0 = time.time()

    def snapshot(self):
        """One synchronous query (call it while the timed work is queued on the GPU)."""
        try:
            out = subprocess.run(["nvidia-smi", f"--id={self.gpu}", f"--query-gpu={self.Q}",
                                  "--format=csv,noheader,nounits"], capture_output=True, text=True, timeout=20)
            self.extra += [l for l in out.stdout.splitlines() if l.strip()]
        except Exception:
            pass

    def stop(self):
        self.t1 = time.time()
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
        self.fh.close()
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]

        def when(stamp):
            try:
                return datetime.datetime.strptime(stamp.strip(), "%Y/%m/%d %H:%M:%S.%f").timestamp()
            except ValueError:
                return None
        try:
            lines = [(l, False) for l in open(self.path)] + [(l, True) for l in self.extra]
        except FileNotFoundError:
            lines = [(l, True) for l in self.extra]
        for line, inside in lines:
            f = [x.strip() for x in line.split(",")]
            if len(f) < 9:
                continue
            ts = when(f[0])
            if not inside and (ts is None or self.t0 is None or not (self.t0 - 0.05 <= ts <= self.t1 + 0.05)):
                continue
            try:
                sm.append(float(f[1]))
                mx = max(mx, float(f[2]))
            except ValueError:
                continue
            for name, val in zip(names, f[5:9]):
                if val.lower().startswith("active"):
                    reasons.add(name)
        if os.path.exists(self.path):
            os.unlink(self.path)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": mx or None,
                "reasons": sorted(reasons), "samples": len(sm)}


def cpu_baseline(reps=3):
    """The reference path on the host as BASELINE.md §3 defines it (oracle/cpu_timing.py): C1 = Q7 L4
    fp64 vmult on ONE pinned core, the reference's compiled kernel (oracle/_ref) vs its numpy einsum
    fallback, best of 3, the faster reported; plus the all-cores figure (threaded BLAS form, Q7 L5)."""
    from oracle import cpu_timing

    c1 = cpu_timing.run([("vmult", 7, 4)], reps=reps)
    case = c1["cases"]["vmult Q7 L4"]
    allc = cpu_timing.all_cores_vmult()
    best = case["best_backend"]
    return {"value": case["mdofs_per_s"] / 1e3, "unit": UNIT, "cores": 1,
            "kind": "reference" if best == "compiled" else "port",
            "sample": f"C1: Q7 level 4 (16^3 cells, {case['dofs']} DoF) fp64 vmult on one pinned core, best of "
                      f"{reps}; backend {best} (compiled oracle/_ref {case['seconds']['compiled']} s, numpy einsum "
                      f"{case['seconds']['einsum']} s per vmult)",
            "cpu_model": c1["cpu_model"], "nproc": c1["nproc"],
            "all_cores": {"value": allc["dofs"] / allc["seconds"] / 1e9, "unit": UNIT, "cores": allc["threads"],
                          "sample": f"{allc['case']} fp64 vmult, contractions as threaded BLAS GEMMs, best of 2"},
            "seconds_per_vmult": min(v for v in case["seconds"].values() if v)}


def run_reference(args, rank, world):
    """--impl reference: the reference's CPU path with all host threads (bounded sample per step),
    plus the single-core as-shipped C1 figure."""
    if rank != 0:
        return
    from oracle import cpu_timing

    steps = []
    res = None
    for _ in range(args.warmup):
        cpu_timing.all_cores_vmult(reps=1)
    for _ in range(args.steps):
        res = cpu_timing.all_cores_vmult(reps=1)
        steps.append(res["dofs"] / res["seconds"] / 1e9)
    value = float(np.median(steps))
    single = cpu_baseline()
    sample = (f"Q7 level 5 ({res['dofs']} DoF) fp64 vmult per step, the reference algorithm (oracle/port.py) "
              f"with its contractions as threaded BLAS GEMMs on {res['threads']} host threads")
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": res["dofs"] / value / 1e6, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "impl": "reference",
            "config": {"workload": "Q7 SIPG Laplace vmult, fp64 (bounded CPU sample: Q7 level 5, 16.8M DoF)",
                       "degree": 7, "level": 5, "dofs": res["dofs"]},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": res["threads"], "kind": "port",
                             "sample": sample, "cpu_model": single["cpu_model"], "nproc": single["nproc"],
                             "single_core_as_shipped": {k: single[k] for k in ("value", "unit", "cores", "kind",
                                                                               "sample")}},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--degree", type=int, default=7)
    ap.add_argument("--level", type=int, default=7)
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-extras", action="store_true")
    args = ap.parse_args()

    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    if args.impl == "reference":
        run_reference(args, rank, world)
        return

    import torch
    import torch.distributed as dist

    import paper_2407_09621_b200 as sf
    from paper_2407_09621_b200 import _native
    from paper_2407_09621_b200.discretization import vmult_device

    local = int(os.environ.get("LOCAL_RANK", 0))
    # SUMFACT_B200_SHARE_GPU=1, or more ranks than visible GPUs: every rank on cuda:0 over gloo (exercises the
    # N>1 path on a 1-GPU box; the throughput of such a run is not a scaling number)
    shared = os.environ.get("SUMFACT_B200_SHARE_GPU") == "1" or world > torch.cuda.device_count()
    if shared:
        local = 0
    torch.cuda.set_device(local)
    if world > 1:
        if shared:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    k, lvl = args.degree, args.level
    K = k + 1
    hier = sf.build_hierarchy(lvl, k, max_dofs=2**34, min_level=lvl)
    n = hier.n_cells(lvl)
    A = hier.axis_dofs(lvl)
    D = hier.n_dofs(lvl)
    P = sf.PrecisionMode
    gen = torch.Generator(device="cuda").manual_seed(1234 + rank)
    u = torch.randn(D, dtype=torch.float64, device="cuda", generator=gen)
    v = torch.empty_like(u)
    kernel_events = []  # (start, end) CUDA events around the vmult kernel of every timed step
    if world > 1:
        from paper_2407_09621_b200 import slab

        comm = slab.SlabComm()
        op = slab.DistributedOperator.weak(hier, lvl, comm)  # NCCL K-plane halo overlapped with the interior
        glo, ghi = op.ghosts(torch.float64)
        grid = _native.SfGrid(n, n, n, glo.data_ptr() if comm.lo is not None else None,
                              ghi.data_ptr() if comm.hi is not None else None)

        def step(timed=False):
            op.apply(u, v, P.FP64)

        def kernel_only(timed=False):  # the vmult kernel alone (ghost planes as left by the last exchange)
            ev = (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
            ev[0].record()
            vmult_device(hier, lvl, u, v, P.FP64, grid=grid)
            ev[1].record()
            kernel_events.append(ev)
    else:
        grid = hier.grid(lvl)

        def step(timed=False):
            vmult_device(hier, lvl, u, v, P.FP64, grid=grid)

    clocks = ClockSampler(local)
    clocks.wait_ready()
    for _ in range(max(args.warmup, 3)):
        step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    stream = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clocks.start()
    e0.record(stream)
    for _ in range(args.steps):
        step(timed=True)
    e1.record(stream)
    clocks.snapshot()  # the timed steps are queued on the GPU: this query samples them
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clk = clocks.stop()
    ms = e0.elapsed_time(e1) / args.steps
    halo_ms = None
    if world > 1:
        for _ in range(3):
            kernel_only()
        torch.cuda.synchronize()
        # the K-plane halo exchange alone (NCCL send/recv of 2 x K planes), CUDA events on the compute stream
        from paper_2407_09621_b200.slab import exchange_face_planes

        glo2, ghi2 = op.ghosts(torch.float64)
        hv = []
        for _ in range(4):
            ev = (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
            ev[0].record()
            exchange_face_planes(comm, op.slab, u, glo2, ghi2)
            ev[1].record()
            hv.append(ev)
        torch.cuda.synchronize()
        halo_ms = sum(a.elapsed_time(b) for a, b in hv[1:]) / 3
    if world > 1:
        t = torch.tensor([ms], dtype=torch.float64, device="cuda")
        if shared:
            t = t.cpu()
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    value = world * D / (ms * 1e-3) / 1e9

    # roofline of the dominant kernel (the vmult; the only one of ours in the step): executed DMMA-schedule
    # flops per launch over its average launch time (CUDA events on its stream; max over ranks)
    kms = ms
    if kernel_events:
        kms = sum(a.elapsed_time(b) for a, b in kernel_events) / len(kernel_events)
        t = torch.tensor([kms], dtype=torch.float64)
        if not shared:
            t = t.cuda()
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        kms = float(t.item())
    kflops = kernel_flops_per_dof(k) * D
    achieved_tf = kflops / (kms * 1e-3) / 1e12
    hbm, hbm_src = peaks()
    roofline = {"bound": "tensor", "achieved": achieved_tf, "peak": FP64_PEAK_TFLOPS, "unit": "TFLOP/s",
                "frac": (achieved_tf / FP64_PEAK_TFLOPS) if achieved_tf else None, "traffic": None,
                "kernel": {7: "sf::dm::k_vmult_dmma8", 3: "sf::dm::k_vmult_dmma_line<4>",
                           1: "sf::dm::k_vmult_dmma_line<2>"}.get(k, f"sf::k_vmult<{K},0>"),
                "kernel_ms": kms,
                "flops_per_dof": kernel_flops_per_dof(k),
                "peak_source": "measured DMMA microbenchmark (profiles/r01_microbench_fp64.md)",
                "hbm": {"achieved": 16 * D / (kms * 1e-3) / 1e9, "peak": hbm, "unit": "GB/s",
                        "frac": 16 * D / (kms * 1e-3) / 1e9 / hbm, "peak_source": hbm_src}}
    traffic = os.path.join(ROOT, "profiles", "vmult_traffic.json")
    if os.path.exists(traffic):  # ncu-measured bytes, used only while the kernel sources are unchanged
        try:
            sys.path.insert(0, os.path.join(ROOT, "tools"))
            from record_traffic import source_hash

            rec = json.load(open(traffic))
            if rec.get("source_hash") == source_hash() and rec.get(f"k{k}_l{lvl}_fp64"):
                roofline["traffic"] = rec[f"k{k}_l{lvl}_fp64"]
                roofline["traffic_source"] = "profiles/vmult_traffic.json (ncu dram bytes, same kernel sources)"
        except Exception:
            pass

    out = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
           "warmup": max(args.warmup, 3), "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
           "vs_baseline": None, "dtype": "f64", "data": "synthetic (u ~ N(0,1), seeded)",
           "config": {"workload": f"Q{k} DG-SIPG Laplace vmult, fp64, {n}x{n}x{n * world} cells "
                                  f"({world * D} DoF; {D} per GPU)",
                      "degree": k, "level": lvl, "dofs_per_gpu": D,
                      "parallelism": (f"z-slab x{world}" + (" (ranks sharing one GPU over gloo: not a scaling point)"
                                                             if shared else "")) if world > 1 else "single GPU",
                      "l2_flush": f"not needed: u, v = 2 x {8 * D / 1e9:.2f} GB per GPU >> 126 MB L2"},
           # the reference's patch schedule would need this many flop per DoF (src/discretization.py:240-264);
           # the kernel runs the cell-wise form (roofline.flops_per_dof), so this is a work-equivalence note only
           "reference_schedule_flop_per_dof": ref_flops_per_dof(k, lvl),
           "roofline": roofline, "clocks": clk,
           # our kernels per timed step: one vmult; at N > 1 the interior + two boundary tile layers
           "gpu_launches": args.steps * (3 if world > 1 and n >= 3 * (16 // K if K in (2, 4) else 2) else 1)}
    if halo_ms is not None:  # max over ranks; overlapped with the interior tiles inside the timed step
        t = torch.tensor([halo_ms], dtype=torch.float64)
        if not shared:
            t = t.cuda()
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        out["halo"] = {"exchange_ms_alone": float(t.item()), "bytes_per_rank": 2 * 8 * K * A * A,
                       "overlapped_with": "interior tile layers (sf_vmult_zrange) during the timed step"}

    # e2e: the public API with pinned HOST buffers, H2D + D2H inside the timed region, every step
    try:
        uh = torch.empty(D, dtype=torch.float64, pin_memory=True)
        uh.copy_(u)
        vh = torch.empty(D, dtype=torch.float64, pin_memory=True)
        if world == 1:
            api = "paper_2407_09621_b200.apply_operator(pinned host; z-slabs streamed)"

            def e2e_step():
                sf.apply_operator(hier, lvl, uh, out=vh)
        else:
            api = "slab.DistributedOperator.apply (per-rank pinned host slab -> HBM -> halo + vmult -> host)"

            def e2e_step():
                u.copy_(uh, non_blocking=True)
                op.apply(u, v, P.FP64)
                vh.copy_(v, non_blocking=True)
        e2e_step()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        for _ in range(args.e2e_steps):
            e2e_step()
        torch.cuda.synchronize()
        dt = (time.perf_counter() - t0) / args.e2e_steps
        if world > 1:
            t = torch.tensor([dt], dtype=torch.float64)
            if not shared:
                t = t.cuda()
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            dt = float(t.item())
        out["e2e"] = {"value": world * D / dt / 1e9, "unit": UNIT, "h2d_bytes_per_step": 8 * D * world,
                      "d2h_bytes_per_step": 8 * D * world, "api": api}
        del uh, vh
    except Exception as exc:  # pinned allocation can fail on small hosts
        out["e2e"] = {"value": None, "unit": UNIT, "error": repr(exc)[:200]}
    if rank == 0 and world == 1:
        if not args.no_cpu:
            out["cpu_baseline"] = {kk: vv for kk, vv in cpu_baseline().items() if kk != "seconds_per_vmult"}
        if not args.no_extras:
            out["extras"] = extras(sf, hier, lvl, k, u, v)
    if rank == 0:
        print(json.dumps(out), flush=True)
    if world > 1:
        dist.destroy_process_group()


SOLVE_KEYS = ("iterations", "solve_s", "solve_s_min", "solve_s_max", "solves_timed", "setup_s", "l2_error")


def extras(sf, hier, lvl, k, u, v):
    """Secondary measurements of the other configs (FP16 paths, Q3, smoother, solve)."""
    import torch

    from paper_2407_09621_b200.discretization import vmult_device

    P = sf.PrecisionMode
    res = {}

    def timeit(fn, reps=5):
        fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            fn()
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / reps

    D = hier.n_dofs(lvl)
    u32 = u.float()
    v32 = torch.empty_like(u32)
    for mode in (P.FP32, P.FP16, P.FP16_EC):
        ms = timeit(lambda: vmult_device(hier, lvl, u32, v32, mode))
        res[f"vmult_q{k}_l{lvl}_{mode.value}_gdofs"] = D / ms / 1e6
    # Q3 level 8 (1.07e9 DoF)
    h3 = sf.build_hierarchy(8, 3, max_dofs=2**34, min_level=8)
    ms = timeit(lambda: vmult_device(h3, 8, u, v, P.FP64))
    res["vmult_q3_l8_fp64_gdofs"] = h3.n_dofs(8) / ms / 1e6
    ms = timeit(lambda: vmult_device(h3, 8, u32, v32, P.FP32))
    res["vmult_q3_l8_fp32_gdofs"] = h3.n_dofs(8) / ms / 1e6
    del u32, v32
    # smoothing step (8 colour passes), Q7 level 6
    h6 = sf.build_hierarchy(6, k, max_dofs=2**34)
    D6 = h6.n_dofs(6)
    from paper_2407_09621_b200 import _native, device as dev

    hbm, _ = peaks()
    for mode in (P.FP64, P.FP32, P.FP16, P.FP16_EC):
        mg = sf.MultigridPreconditioner(h6, sf.VCycleConfig(mode=mode))
        x = torch.zeros(D6, dtype=mode.torch_dtype, device="cuda")
        b = torch.randn(D6, dtype=mode.torch_dtype, device="cuda")
        ms = timeit(lambda: mg._smooth_device(6, x, b, mode), reps=2)
        res[f"smooth_step_q{k}_l6_{mode.value}_ms"] = ms
        # one colour pass (shift 000: every DoF in a patch) -- the smoother's kernel, HBM roofline at
        # 3 vectors (read x, b; write x) of the storage dtype per DoF
        xn = torch.empty_like(x)
        lm = h6.matrices(6)

        def colour():
            rc = _native.lib().sf_smooth_colour(mode.code, k, h6.grid(6), mg._shift_arrays[(0, 0, 0)],
                                                _native.host_ptr(lm.cell_op), _native.host_ptr(mg.solvers[6].table),
                                                dev.ptr(x), dev.ptr(b), dev.ptr(xn), dev.stream_ptr())
            _native.check(rc, "sf_smooth_colour")
        ms1 = timeit(colour, reps=5)
        gbs = 3 * x.element_size() * D6 / (ms1 * 1e-3) / 1e9
        res[f"colour_pass_q{k}_l6_{mode.value}"] = {"ms": ms1, "gdofs": D6 / ms1 / 1e6, "hbm_gbs": gbs,
                                                   "hbm_frac": gbs / hbm}
        del xn
    del x, b, mg
    torch.cuda.empty_cache()  # the vmult benches above leave large cached blocks; solves allocate afresh
    # time-to-solution (BASELINE configs[3]): FGMRES(fp64) + V-cycle(fp64 | fp16_ec), Q7 level 6,
    # 1.34e8 DoF, setup excluded (tools/bench_solve.py)
    try:
        sys.path.insert(0, os.path.join(ROOT, "tools"))
        from bench_solve import solve_once

        for mode in (P.FP64, P.FP16_EC):
            r = solve_once(h6, 6, mode, reps=5)
            res[f"solve_q{k}_l6_{mode.value}"] = {kk: r[kk] for kk in SOLVE_KEYS}
        del h6
        h37 = sf.build_hierarchy(7, 3, max_dofs=2**34)  # Q3 level 7: the other 1.34e8-DoF solve config
        for mode in (P.FP64, P.FP16_EC):
            r = solve_once(h37, 7, mode, reps=5)
            res[f"solve_q3_l7_{mode.value}"] = {kk: r[kk] for kk in SOLVE_KEYS}
        for cfg in ("q7_l6", "q3_l7"):  # mixed-precision speed-up at the same tolerance (BASELINE configs[3])
            a, b = res.get(f"solve_{cfg}_fp64"), res.get(f"solve_{cfg}_fp16_ec")
            if a and b:
                res[f"solve_{cfg}_fp16_ec_speedup_vs_fp64"] = a["solve_s"] / b["solve_s"]
    except Exception as exc:  # secondary measurement only
        res["solve_error"] = repr(exc)[:200]
    return res


if __name__ == "__main__":
    main()
