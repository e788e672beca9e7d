"""z-slab domain decomposition of the hot path over torch.distributed (one process per GPU).

The reference is single-process ("Parallelism strategies: none"); this module adds the
decomposition SURVEY.md §8e prescribes, with NCCL over NVLink on the B200 box and gloo for the
host-logic tests on CPU:

* the global cube of n^3 cells is cut along z (the slowest axis, so every slab -- and every ghost
  layer -- is one contiguous range of the reference's flat (z, y, x) vector);
* ``DistributedOperator``: the SIPG vmult (discretization.py:216-266) after exchanging the K dof
  planes adjacent to each slab face; the kernel reads the neighbour's face traces from the ghost
  planes (``sf_grid.ghost_lo/ghost_hi``);
* ``DistributedMultigrid``: the V-cycle (multigrid.py:243-270) with level vectors kept in an
  *extended* slab (2 ghost cells per interior side), refreshed before every smoother colour;
  straddling vertex patches are solved redundantly by both owners; levels whose slab would be
  thinner than 2 cells are agglomerated (all-gather of the restricted residual, replicated coarse
  V-cycle, identical on every rank);
* ``fgmres_distributed``: krylov.fgmres with every dot product / norm all-reduced.

The numerics per rank are the single-GPU kernels; only the data movement is added here.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _native, device
from .discretization import MeshHierarchy, vmult_device
from .multigrid import MultigridPreconditioner, VCycleConfig
from .precision import PrecisionMode

GHOST_CELLS = 2  # smoother halo: a cell's colour update depends on x at most 2 cells away


class SlabComm:
    """Neighbour exchange and reductions of a z-slab decomposition.

    Rank r owns the r-th slab (rank order = z order).  NCCL moves CUDA tensors directly; with the
    gloo backend CUDA tensors are staged through host memory (tests / single-GPU emulation only).
    """

    def __init__(self, group=None):
        import torch.distributed as dist

        self.dist = dist
        self.group = group
        if dist.is_available() and dist.is_initialized():
            self.rank = dist.get_rank(group)
            self.world = dist.get_world_size(group)
            self.backend = str(dist.get_backend(group))
        else:
            self.rank, self.world, self.backend = 0, 1, "none"
        self.lo = self.rank - 1 if self.rank > 0 else None
        self.hi = self.rank + 1 if self.rank < self.world - 1 else None

    def _global(self, r):
        return r if self.group is None else self.dist.get_global_rank(self.group, r)

    def _staged(self, tensors):
        return self.backend == "gloo" and any(t.is_cuda for t in tensors)

    def exchange_start(self, send_lo=None, recv_lo=None, send_hi=None, recv_hi=None):
        """Post the neighbour exchange (send_lo -> rank-1's recv_hi, send_hi -> rank+1's recv_lo).

        NCCL: the transfers run on NCCL's stream once the current stream's prior work is done, so
        kernels enqueued after this call overlap them.  Returns a handle for exchange_finish."""
        if self.world == 1:
            return None
        pairs = []
        if self.lo is not None:
            pairs.append((send_lo, recv_lo, self.lo))
        if self.hi is not None:
            pairs.append((send_hi, recv_hi, self.hi))
        staged = self._staged([t for p in pairs for t in p[:2]])
        ops, back = [], []
        for snd, rcv, peer in pairs:
            if staged:
                s, r = snd.cpu(), torch.empty(rcv.shape, dtype=rcv.dtype)
                back.append((r, rcv))
            else:
                s, r = snd.contiguous(), rcv
            ops.append(self.dist.P2POp(self.dist.isend, s, self._global(peer), self.group))
            ops.append(self.dist.P2POp(self.dist.irecv, r, self._global(peer), self.group))
        return self.dist.batch_isend_irecv(ops), back

    def exchange_finish(self, handle):
        """Make the current stream wait for a posted exchange (and land host-staged receives)."""
        if handle is None:
            return
        reqs, back = handle
        for req in reqs:
            req.wait()
        for r, rcv in back:
            rcv.copy_(r)

    def exchange(self, send_lo=None, recv_lo=None, send_hi=None, recv_hi=None):
        """send_lo -> rank-1 (lands in its recv_hi); send_hi -> rank+1 (lands in its recv_lo)."""
        self.exchange_finish(self.exchange_start(send_lo, recv_lo, send_hi, recv_hi))

    def allreduce_(self, t: torch.Tensor) -> torch.Tensor:
        """In-place SUM over ranks (fixed NCCL/gloo reduction order for a fixed world: deterministic)."""
        if self.world == 1:
            return t
        if self._staged([t]):
            h = t.cpu()
            self.dist.all_reduce(h, group=self.group)
            t.copy_(h)
        else:
            self.dist.all_reduce(t, group=self.group)
        return t

    def allgather_cat(self, t: torch.Tensor) -> torch.Tensor:
        """Concatenate every rank's (equal-sized) tensor in rank (= z) order."""
        if self.world == 1:
            return t.clone()
        if self._staged([t]):
            h = t.cpu()
            parts = [torch.empty_like(h) for _ in range(self.world)]
            self.dist.all_gather(parts, h, group=self.group)
            return torch.cat(parts).to(t.device)
        parts = [torch.empty_like(t) for _ in range(self.world)]
        self.dist.all_gather(parts, t.contiguous(), group=self.group)
        return torch.cat(parts)


@dataclass
class SlabLevel:
    """Geometry of one level's slab on one rank (cells along z; x and y are global)."""

    level: int
    K: int
    n: int          # global cells per axis
    nz: int         # local cells along z
    z0: int         # first local cell (global index)
    h_lo: int       # ghost cells below in the extended layout (0 on the bottom rank)
    h_hi: int       # ghost cells above (0 on the top rank)

    @property
    def plane(self) -> int:
        return (self.n * self.K) ** 2

    @property
    def cell_layer(self) -> int:
        return self.K * self.plane

    @property
    def local_dofs(self) -> int:
        return self.nz * self.cell_layer

    @property
    def ext_dofs(self) -> int:
        return (self.nz + self.h_lo + self.h_hi) * self.cell_layer

    @property
    def local_slice(self) -> slice:
        a = self.h_lo * self.cell_layer
        return slice(a, a + self.local_dofs)

    @property
    def global_slice(self) -> slice:
        return slice(self.z0 * self.cell_layer, (self.z0 + self.nz) * self.cell_layer)


def slab_levels(hier: MeshHierarchy, rank: int, world: int, ghost_cells: int = GHOST_CELLS) -> dict:
    """Levels that shard: n_l divisible by 2*world (every slab an even number >= 2 of cells).

    Returns {level: SlabLevel} for the contiguous range of distributable levels ending at
    max_level (empty if the finest level cannot be sharded).
    """
    out = {}
    K = hier.degree + 1
    for lvl in range(hier.max_level, hier.min_level - 1, -1):
        n = hier.n_cells(lvl)
        if n % (2 * world) != 0:
            break
        nz = n // world
        if world > 1 and nz < ghost_cells:
            break
        out[lvl] = SlabLevel(lvl, K, n, nz, rank * nz, ghost_cells if rank > 0 else 0,
                             ghost_cells if rank < world - 1 else 0)
    return out


def exchange_face_planes(comm: SlabComm, sl: SlabLevel, u: torch.Tensor, ghost_lo, ghost_hi):
    """vmult halo: the K dof planes of the neighbour cell layer below (above) the slab land in
    ghost_lo (ghost_hi) -- exactly what sf_grid.ghost_lo/hi expect (include/sumfact_b200.h)."""
    Kp = sl.K * sl.plane
    comm.exchange(send_lo=u[:Kp], recv_lo=ghost_lo, send_hi=u[u.numel() - Kp:], recv_hi=ghost_hi)


def refresh_ghost_cells(comm: SlabComm, sl: SlabLevel, x_ext: torch.Tensor):
    """Smoother halo: fill the h_lo / h_hi ghost cells of an extended-slab vector with the
    neighbours' adjacent local cells (afterwards x_ext equals the global vector's matching range)."""
    if comm.world == 1:
        return
    L = sl.cell_layer
    loc = x_ext[sl.local_slice]
    comm.exchange(send_lo=loc[:GHOST_CELLS * L], recv_lo=x_ext[:sl.h_lo * L],
                  send_hi=loc[loc.numel() - GHOST_CELLS * L:], recv_hi=x_ext[x_ext.numel() - sl.h_hi * L:])


def refresh_ghost_cells_start(comm: SlabComm, sl: SlabLevel, x_ext: torch.Tensor):
    """refresh_ghost_cells posted asynchronously (NCCL: on its stream); finish with comm.exchange_finish."""
    if comm.world == 1:
        return None
    L = sl.cell_layer
    loc = x_ext[sl.local_slice]
    return comm.exchange_start(send_lo=loc[:GHOST_CELLS * L], recv_lo=x_ext[:sl.h_lo * L],
                               send_hi=loc[loc.numel() - GHOST_CELLS * L:],
                               recv_hi=x_ext[x_ext.numel() - sl.h_hi * L:])


# Q7 smoother on z-slabs: the ghost-cell refresh of each colour overlaps the colour's interior tiles
# (sf_smooth_colour_zrange), the boundary tiles run once the cells have landed
OVERLAP_SMOOTHER = True


def _grid(n: int, nz: int, lo=None, hi=None) -> _native.SfGrid:
    return _native.SfGrid(n, n, nz, lo, hi)


class DistributedOperator:
    """fp64 (or storage-dtype) vmult on this rank's slab with a K-plane halo (discretization.py:216-266)."""

    def __init__(self, hier: MeshHierarchy, level: int, comm: SlabComm):
        self.hier, self.level, self.comm = hier, level, comm
        sl = slab_levels(hier, comm.rank, comm.world, ghost_cells=1).get(level)
        if sl is None:
            raise ValueError(f"level {level} ({hier.n_cells(level)} cells/axis) does not split into "
                             f"{comm.world} even z-slabs")
        self.slab = sl
        self._ghosts = {}

    @classmethod
    def weak(cls, hier: MeshHierarchy, level: int, comm: SlabComm) -> "DistributedOperator":
        """Weak-scaling brick: every rank owns a full n^3-cell cube of the level, stacked along z
        (global domain n x n x (n * world) cells with the level's h; bench.py --gpus N)."""
        self = cls.__new__(cls)
        self.hier, self.level, self.comm = hier, level, comm
        n = hier.n_cells(level)
        self.slab = SlabLevel(level, hier.degree + 1, n, n, comm.rank * n, 1 if comm.lo is not None else 0,
                              1 if comm.hi is not None else 0)
        self._ghosts = {}
        return self

    def ghosts(self, dtype):
        g = self._ghosts.get(dtype)
        if g is None:
            K, p = self.slab.K, self.slab.plane
            g = (torch.empty(K * p, dtype=dtype, device="cuda"), torch.empty(K * p, dtype=dtype, device="cuda"))
            self._ghosts[dtype] = g
        return g

    def apply(self, u: torch.Tensor, v: torch.Tensor, mode: PrecisionMode = PrecisionMode.FP64):
        """v = A u on the slab.  With neighbours, the ghost-plane exchange overlaps the interior:
        post the exchange, run the tiles that never read a ghost plane (sf_vmult_zrange over
        [t, nz - t)), then -- once the planes have landed -- the two boundary tile layers."""
        sl, c = self.slab, self.comm
        glo, ghi = self.ghosts(u.dtype)
        grid = _grid(sl.n, sl.nz, glo.data_ptr() if c.lo is not None else None,
                     ghi.data_ptr() if c.hi is not None else None)
        t = 16 // sl.K if sl.K in (2, 4) else 2  # tile height in cells (DMMA line tiles for Q1/Q3)
        if c.world == 1 or sl.nz < 3 * t:
            exchange_face_planes(c, sl, u, glo, ghi)
            vmult_device(self.hier, self.level, u, v, mode, grid=grid)
            return v
        Kp = sl.K * sl.plane
        handle = c.exchange_start(send_lo=u[:Kp], recv_lo=glo, send_hi=u[u.numel() - Kp:], recv_hi=ghi)
        self._zrange(grid, t, sl.nz - t, u, v, mode)
        c.exchange_finish(handle)
        self._zrange(grid, 0, t, u, v, mode)
        self._zrange(grid, sl.nz - t, sl.nz, u, v, mode)
        return v

    def _zrange(self, grid, z0, z1, u, v, mode):
        lm = self.hier.matrices(self.level)
        rc = _native.lib().sf_vmult_zrange(mode.code, self.hier.degree, grid, z0, z1, _native.host_ptr(lm.cell_op),
                                           device.ptr(u), device.ptr(v), device.stream_ptr())
        _native.check(rc, "sf_vmult_zrange")

    def __call__(self, u: torch.Tensor) -> torch.Tensor:
        v = torch.empty_like(u)
        return self.apply(u, v)


class DistributedMultigrid:
    """V-cycle on z-slabs (multigrid.py:243-270); fp64 local slab in, fp64 local slab out."""

    def __init__(self, hier: MeshHierarchy, config: VCycleConfig | None, comm: SlabComm, level: int | None = None):
        self.hier, self.comm = hier, comm
        self.config = config or VCycleConfig()
        self.level = hier.max_level if level is None else level
        self.mg = MultigridPreconditioner(hier, self.config)  # patch tables, coarse LU, replicated levels
        allslabs = slab_levels(hier, comm.rank, comm.world)
        self.slabs = {l: s for l, s in allslabs.items() if self.config.coarse_level < l <= self.level}
        if self.level not in self.slabs:
            raise ValueError(f"level {self.level} does not split into {comm.world} z-slabs of >= "
                             f"{GHOST_CELLS} (even) cells")
        self.lowest = min(self.slabs)  # levels below are agglomerated (replicated on every rank)
        self._bufs = {}

    def setup(self):
        self.mg.setup()
        return self

    # ---------------------------------------------------------------- buffers
    def _buf(self, name, level, mode, size=None):
        key = (name, level, mode)
        t = self._bufs.get(key)
        if t is None:
            t = torch.zeros(self.slabs[level].ext_dofs if size is None else size, dtype=mode.torch_dtype,
                            device="cuda")
            self._bufs[key] = t
        return t

    def _refresh(self, sl: SlabLevel, x_ext: torch.Tensor):
        refresh_ghost_cells(self.comm, sl, x_ext)

    def _ext_grid(self, sl):
        return _grid(sl.n, sl.nz + sl.h_lo + sl.h_hi)

    def _local_grid(self, sl, x_ext):
        """Local slab grid whose ghost pointers are the K planes adjacent to it inside x_ext."""
        es = x_ext.element_size()
        base = x_ext.data_ptr() + sl.local_slice.start * es
        Kp = sl.K * sl.plane
        lo = base - Kp * es if self.comm.lo is not None else None
        hi = base + sl.local_dofs * es if self.comm.hi is not None else None
        return _grid(sl.n, sl.nz, lo, hi)

    # ---------------------------------------------------------------- smoother
    def smooth(self, level: int, x_ext: torch.Tensor, b_ext: torch.Tensor, mode: PrecisionMode):
        """One multiplicative sweep over the 8 colours (multigrid.py:172-204); b_ext ghosts must be fresh."""
        sl = self.slabs[level]
        hier = self.hier
        lm = hier.matrices(level)
        table = self.mg.solvers[level].table
        tmp = self._buf("pingpong", level, mode)
        cur, nxt = x_ext, tmp
        lib = _native.lib()
        g = self._ext_grid(sl)
        nz_ext = sl.nz + sl.h_lo + sl.h_hi
        overlap = self.comm.world > 1 and hier.degree == 7 and OVERLAP_SMOOTHER
        for shift in self.config.smoother_ordering:
            if min(sl.n // 2 - s for s in shift) < 1:
                continue
            sh = self.mg._shift_arrays[shift]
            args = (_native.host_ptr(lm.cell_op), _native.host_ptr(table), device.ptr(cur), device.ptr(b_ext),
                    device.ptr(nxt), device.stream_ptr())
            sz = shift[2]
            # interior tiles (first cell c): read x on cells c-1..c+2, none of them a ghost cell
            lo = sl.h_lo + 1 + ((sl.h_lo + 1 - sz) & 1)
            hi = nz_ext - sl.h_hi - 3
            hi -= (hi - sz) & 1
            if overlap and hi >= lo:
                handle = refresh_ghost_cells_start(self.comm, sl, cur)
                rc = lib.sf_smooth_colour_zrange(mode.code, hier.degree, g, sh, lo, hi + 2, *args)
                _native.check(rc, "sf_smooth_colour_zrange")
                self.comm.exchange_finish(handle)
                for z0, z1 in ((sz, lo), (hi + 2, nz_ext - sz)):
                    rc = lib.sf_smooth_colour_zrange(mode.code, hier.degree, g, sh, z0, z1, *args)
                    _native.check(rc, "sf_smooth_colour_zrange")
                rc = lib.sf_copy_uncovered(mode.code, hier.degree, g, sh, device.ptr(cur), device.ptr(nxt),
                                           device.stream_ptr())
                _native.check(rc, "sf_copy_uncovered")
            else:
                self._refresh(sl, cur)
                rc = lib.sf_smooth_colour(mode.code, hier.degree, g, sh, *args)
                _native.check(rc, "sf_smooth_colour")
            cur, nxt = nxt, cur
        if cur is not x_ext:
            x_ext.copy_(cur)

    # ---------------------------------------------------------------- V-cycle
    def _vcycle(self, level: int, x_ext: torch.Tensor, b_ext: torch.Tensor):
        cfg, mode, hier = self.config, self.config.mode, self.hier
        sl = self.slabs[level]
        for _ in range(cfg.pre_smooth_steps):
            self.smooth(level, x_ext, b_ext, mode)
        self._refresh(sl, x_ext)  # ghost planes of the residual inside the restriction
        lm = hier.matrices(level)
        coarse = level - 1
        b_loc = b_ext[sl.local_slice]
        if coarse in self.slabs:
            csl = self.slabs[coarse]
            rc_ext = self._buf("rhs", coarse, mode)
            rc_loc = rc_ext[csl.local_slice]
        else:
            rc_loc = self._buf("agglomerate_rhs", level, mode, size=sl.local_dofs // 8)
        rc = _native.lib().sf_residual_restrict(mode.code, hier.degree, self._local_grid(sl, x_ext),
                                                _native.host_ptr(lm.cell_op), _native.host_ptr(hier.embedding_c),
                                                device.ptr(x_ext) + sl.local_slice.start * x_ext.element_size(),
                                                device.ptr(b_loc), device.ptr(rc_loc), device.stream_ptr())
        _native.check(rc, "sf_residual_restrict")
        if coarse in self.slabs:
            self._refresh(csl, rc_ext)
            e_ext = self._buf("x", coarse, mode)
            e_ext.zero_()
            self._vcycle(coarse, e_ext, rc_ext)
            e_loc = e_ext[csl.local_slice]
        else:
            # agglomerate: every rank solves the coarse sub-hierarchy on the gathered residual
            rhs = self.comm.allgather_cat(rc_loc)
            e = self.mg._buf("x", coarse, mode)
            e.zero_()
            self.mg._vcycle_device(coarse, e, rhs)
            n = rc_loc.numel()
            e_loc = e[self.comm.rank * n:(self.comm.rank + 1) * n]
        cg = _grid(sl.n // 2, sl.nz // 2)
        rc = _native.lib().sf_prolongate_add(mode.code, hier.degree, cg, _native.host_ptr(hier.embedding_c),
                                             device.ptr(e_loc), device.ptr(x_ext[sl.local_slice]),
                                             device.stream_ptr())
        _native.check(rc, "sf_prolongate_add")
        for _ in range(cfg.post_smooth_steps):
            self.smooth(level, x_ext, b_ext, mode)

    def apply(self, b: torch.Tensor) -> torch.Tensor:
        """Preconditioner action on the local fp64 slab: one V-cycle from x = 0 (multigrid.py:257-270)."""
        mode = self.config.mode
        sl = self.slabs[self.level]
        b = b.reshape(-1)
        if b.numel() != sl.local_dofs:
            raise ValueError(f"expected {sl.local_dofs} local entries, got {b.numel()}")
        x_ext = self._buf("x", self.level, mode)
        b_ext = self._buf("rhs", self.level, mode)
        x_ext.zero_()
        device.convert(b.contiguous(), b_ext[sl.local_slice])
        self._refresh(sl, b_ext)
        self._vcycle(self.level, x_ext, b_ext)
        out = torch.empty(sl.local_dofs, dtype=torch.float64, device="cuda")
        device.convert(x_ext[sl.local_slice], out)
        return out

    __call__ = apply


def fgmres_distributed(apply_A, apply_M, b: torch.Tensor, comm: SlabComm, tol=1e-8, maxit=100):
    """krylov.fgmres (krylov.py:140-151) on slab-local vectors with every inner product all-reduced."""
    from .krylov import _gmres_driver

    if not 0.0 < tol < 1.0:
        raise ValueError("tol must lie in (0, 1)")
    return _gmres_driver(apply_A, apply_M, b, tol, maxit, True, False, reduce=comm.allreduce_)


def run_solve_distributed(degree: int, level: int, comm: SlabComm, mode: PrecisionMode = PrecisionMode.FP64,
                          tol: float = 1e-8, maxit: int = 100, coarse_level: int = 1, pre_smooth: int = 1,
                          post_smooth: int = 1, hier: MeshHierarchy | None = None):
    """experiments.run_solve (experiments.py:57-103) on z-slabs: every rank assembles its slab of the
    manufactured problem's load vector on the device, FGMRES runs on slab vectors with all-reduced inner
    products, the preconditioner is the slab V-cycle, and the L2 error is an all-reduced sum of squares.
    Returns (x_local, SolveReport, l2) on every rank."""
    import math

    from .discretization import _separable_error_sq, assemble_rhs_separable, build_hierarchy
    from .basis import gauss_rule, lagrange_values

    hier = hier or build_hierarchy(level, degree, max_dofs=2**34)
    cfg = VCycleConfig(pre_smooth_steps=pre_smooth, post_smooth_steps=post_smooth, coarse_level=coarse_level,
                       mode=mode)
    mg = DistributedMultigrid(hier, cfg, comm, level).setup()
    op = DistributedOperator(hier, level, comm)
    sl = mg.slabs[level]
    sine = lambda x: np.sin(np.pi * x)
    b = assemble_rhs_separable(hier, level, sine, 3.0 * math.pi**2, z_cells=(sl.z0, sl.nz))  # slab-local
    x, rep = fgmres_distributed(op, mg, b, comm, tol=tol, maxit=maxit)
    # L2 error: the separable quadrature over this rank's z cells, all-reduced
    rule = gauss_rule(hier.degree + 3)
    S = lagrange_values(hier.basis.nodes, rule.points)
    n, h = hier.n_cells(level), hier.h(level)
    f = sine((np.arange(n)[:, None] + rule.points[None, :]) * h)
    part = _separable_error_sq(hier, level, x, (S, S, S), (f, f, f[sl.z0:sl.z0 + sl.nz]), nz=sl.nz).reshape(1)
    comm.allreduce_(part)
    l2 = float(torch.sqrt(part))
    rep.l2_error = l2
    return x, rep, l2


def scatter_slab(x_global, comm: SlabComm, sl: SlabLevel) -> torch.Tensor:
    """This rank's slab of a global vector (numpy or tensor) as a CUDA tensor."""
    t = x_global if isinstance(x_global, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(x_global))
    return t.reshape(-1)[sl.global_slice].to("cuda").contiguous()


__all__ = ["SlabComm", "SlabLevel", "slab_levels", "DistributedOperator", "DistributedMultigrid",
           "fgmres_distributed", "run_solve_distributed", "scatter_slab", "exchange_face_planes", "refresh_ghost_cells",
           "refresh_ghost_cells_start", "GHOST_CELLS", "OVERLAP_SMOOTHER"]

