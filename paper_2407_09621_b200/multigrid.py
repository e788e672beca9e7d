"""Geometric V-cycle with the multiplicative vertex-patch smoother, on the B200.

Mirror of the reference's src/multigrid.py API (default_ordering,
VCycleConfig, PatchSolver, patch_inverse_apply, restrict, prolongate,
MultigridPreconditioner).  Every sweep runs in sm_100a kernels:

* smoother colour = one ``sf_smooth_colour`` launch (residual on the colour's
  patches, fast-diagonalisation solve, update) with ping-pong x buffers;
* ``r = b - A x; restrict(r)`` = one ``sf_residual_restrict`` launch;
* ``x + prolongate(e)`` = one ``sf_prolongate_add`` launch;
* the coarse solve is a dense LU factored once on the device (torch.linalg /
  cuSOLVER -- setup-time library code, like scipy in the reference).
"""
from __future__ import annotations

import itertools
from dataclasses import dataclass

import numpy as np
import scipy.linalg
import torch

from . import _native, device
from .discretization import MeshHierarchy, materialize_device, vmult_device
from .precision import PrecisionMode


def default_ordering(dim: int) -> tuple:
    """multigrid.py:27-29 -- all tiling shifts, lexicographic; element i = tensor axis i."""
    return tuple(itertools.product((0, 1), repeat=dim))


@dataclass
class VCycleConfig:
    """multigrid.py:32-44."""

    pre_smooth_steps: int = 1
    post_smooth_steps: int = 1
    coarse_level: int = 1
    mode: PrecisionMode = PrecisionMode.FP64
    smoother_ordering: tuple = None

    def __post_init__(self):
        if self.pre_smooth_steps < 1 or self.post_smooth_steps < 1:
            raise ValueError("smoothing steps must be at least 1")
        if self.coarse_level < 1:
            raise ValueError("coarse level must be at least 1")


_KIND_INDEX = {(False, False): 0, (False, True): 1, (True, False): 2, (True, True): 3}  # 2*lb + rb


class PatchSolver:
    """Fast-diagonalisation inverse of the separable patch operator (multigrid.py:47-89).

    eig[kind] = scipy.linalg.eigh(L_kind, M) (host setup, as the reference);
    ``table`` packs V and lambda for the kernels (kind index 2*left + right).
    """

    def __init__(self, M: np.ndarray, L_by_kind: dict):
        self.eig = {}
        for kind, L in L_by_kind.items():
            lam, V = scipy.linalg.eigh(L, M)
            self.eig[kind] = (lam, V)
        self.B = M.shape[0]
        self.table = None
        if all(k in self.eig for k in _KIND_INDEX):
            Vs = np.zeros((4, self.B, self.B))
            lams = np.zeros((4, self.B))
            for kind, q in _KIND_INDEX.items():
                lams[q], Vs[q] = self.eig[kind]
            self.table = np.ascontiguousarray(np.concatenate([Vs.ravel(), lams.ravel()]))

    def lambda_sum(self, kinds) -> np.ndarray:
        total = np.zeros((1,) * len(kinds))
        for d, kind in enumerate(kinds):
            shape = [1] * len(kinds)
            shape[d] = len(self.eig[kind][0])
            total = total + self.eig[kind][0].reshape(shape)
        return total

    def apply_batch(self, w, kinds, mode: PrecisionMode = PrecisionMode.FP64):
        """Solve on a batch (counts..., B, B, B) sharing one kind per numpy block axis (z, y, x)."""
        if self.table is None:
            raise NotImplementedError("the kernel tables need the four boundary kinds")
        host = not isinstance(w, torch.Tensor)
        arr = np.asarray(w) if host else w
        shape = tuple(arr.shape)
        B = self.B
        if len(shape) < 3 or shape[-3:] != (B, B, B):
            raise ValueError(f"patch batch must end in {(B, B, B)}")
        count = int(np.prod(shape[:-3], dtype=np.int64))
        device.require_cuda()
        t, _ = device.as_device(arr, mode.torch_dtype)
        out = torch.empty_like(t)
        # reference kinds are per numpy block axis (z, y, x); the ABI takes tensor axes (x, y, z)
        arr3 = _c_int3(_native_kinds(kinds[2]), _native_kinds(kinds[1]), _native_kinds(kinds[0]))
        k = B // 2 - 1
        rc = _native.lib().sf_patch_apply(mode.code, k, count, arr3, _native.host_ptr(self.table), device.ptr(t),
                                          device.ptr(out), device.stream_ptr())
        _native.check(rc, "sf_patch_apply")
        return device.to_host(out, mode.storage_dtype).reshape(shape) if host else out.reshape(shape)

    def apply_single(self, r, kinds, mode: PrecisionMode = PrecisionMode.FP64):
        r = np.asarray(r) if not isinstance(r, torch.Tensor) else r
        return self.apply_batch(r[(None,) * 3], kinds, mode)[0, 0, 0]


import ctypes as _ctypes  # noqa: E402

_c_int3 = _ctypes.c_int * 3


def _native_kinds(kind) -> int:
    return _KIND_INDEX[tuple(bool(b) for b in kind)]


def patch_inverse_apply(solver: PatchSolver, r, kinds):
    """multigrid.py:86-89."""
    return solver.apply_single(np.asarray(r, dtype=np.float64), kinds)


# ---------------------------------------------------------------- transfers


def restrict_device(hier, level, r: torch.Tensor, coarse: torch.Tensor, mode: PrecisionMode,
                    x: torch.Tensor | None = None):
    """coarse = R r  (x None) or R (r - A x) (fused residual)."""
    lm = hier.matrices(level)
    rc = _native.lib().sf_residual_restrict(mode.code, hier.degree, hier.grid(level), _native.host_ptr(lm.cell_op),
                                            _native.host_ptr(hier.embedding_c),
                                            device.ptr(x) if x is not None else None, device.ptr(r),
                                            device.ptr(coarse), device.stream_ptr())
    _native.check(rc, "sf_residual_restrict")


def prolongate_add_device(hier, coarse_level, e: torch.Tensor, fine: torch.Tensor, mode: PrecisionMode):
    rc = _native.lib().sf_prolongate_add(mode.code, hier.degree, hier.grid(coarse_level),
                                         _native.host_ptr(hier.embedding_c), device.ptr(e), device.ptr(fine),
                                         device.stream_ptr())
    _native.check(rc, "sf_prolongate_add")


def restrict(hier: MeshHierarchy, level: int, r, mode: PrecisionMode = PrecisionMode.FP64):
    """Transpose of the embedding, fine level -> level-1 (multigrid.py:112-125)."""
    device.require_cuda()
    t, host = device.as_device(r, mode.torch_dtype, hier.n_dofs(level))
    coarse = torch.empty(hier.n_dofs(level - 1), dtype=mode.torch_dtype, device="cuda")
    restrict_device(hier, level, t, coarse, mode)
    return device.to_host(coarse, mode.storage_dtype) if host else coarse


def prolongate(hier: MeshHierarchy, coarse_level: int, e, mode: PrecisionMode = PrecisionMode.FP64):
    """Exact embedding of a coarse function into the next finer level (multigrid.py:128-143)."""
    device.require_cuda()
    t, host = device.as_device(e, mode.torch_dtype, hier.n_dofs(coarse_level))
    fine = torch.zeros(hier.n_dofs(coarse_level + 1), dtype=mode.torch_dtype, device="cuda")
    prolongate_add_device(hier, coarse_level, t, fine, mode)
    return device.to_host(fine, mode.storage_dtype) if host else fine


# ------------------------------------------------------------ preconditioner


COARSE_INVERSE_MAX = 16384  # coarse unknowns up to which the solve is a product with the explicit inverse


class MultigridPreconditioner:
    """V-cycle on a mesh hierarchy, usable as a right preconditioner (multigrid.py:146-270)."""

    def __init__(self, hier: MeshHierarchy, config: VCycleConfig | None = None):
        self.hier = hier
        self.config = config or VCycleConfig()
        if self.config.smoother_ordering is None:
            self.config.smoother_ordering = default_ordering(hier.dim)
        self._check_ordering()
        if self.config.coarse_level < hier.min_level:
            raise ValueError("coarse level below the hierarchy's minimum")
        self.solvers = {lvl: PatchSolver(hier.matrices(lvl).M_patch, hier.matrices(lvl).L_smooth)
                        for lvl in hier.levels()}
        self._coarse_cache = {}
        self._buffers = {}
        self._shift_arrays = {s: (_ctypes.c_int * 3)(*s) for s in self.config.smoother_ordering}

    def _check_ordering(self):
        expected = set(default_ordering(self.hier.dim))
        order = self.config.smoother_ordering
        if set(order) != expected or len(order) != len(expected):
            raise ValueError("smoother ordering must enumerate every tiling shift once")

    # ------------------------------------------------------------- buffers
    def _buf(self, name, level, mode):
        key = (name, level, mode)
        t = self._buffers.get(key)
        if t is None:
            t = torch.empty(self.hier.n_dofs(level), dtype=mode.torch_dtype, device="cuda")
            self._buffers[key] = t
        return t

    # ------------------------------------------------------------ smoother
    def _smooth_device(self, level: int, x: torch.Tensor, b: torch.Tensor, mode: PrecisionMode,
                       x_zero: bool = False):
        """One multiplicative sweep in place on device x (multigrid.py:172-204).  x_zero: x is known to be zero
        (a V-cycle's first pre-smoothing step); an unshifted first colour then runs the zero-iterate kernel
        (r = b: no operator application, no x_old reads), bitwise the same result."""
        hier = self.hier
        n = hier.n_cells(level)
        lm = hier.matrices(level)
        table = self.solvers[level].table
        tmp = self._buf("pingpong", level, mode)
        cur, nxt = x, tmp
        L = _native.lib()
        g = hier.grid(level)
        first = True
        for shift in self.config.smoother_ordering:
            if min(n // 2 - s for s in shift) < 1:
                continue
            args = (mode.code, hier.degree, g, self._shift_arrays[shift], _native.host_ptr(lm.cell_op),
                    _native.host_ptr(table))
            rc = _native.SF_EUNSUPPORTED
            if first and x_zero and not any(shift):
                rc = L.sf_smooth_colour(*args, None, device.ptr(b), device.ptr(nxt), device.stream_ptr())
            if rc == _native.SF_EUNSUPPORTED:
                rc = L.sf_smooth_colour(*args, device.ptr(cur), device.ptr(b), device.ptr(nxt), device.stream_ptr())
            _native.check(rc, "sf_smooth_colour")
            cur, nxt = nxt, cur
            first = False
        if cur is not x:
            x.copy_(cur)

    def smooth(self, level: int, x, b, mode: PrecisionMode | None = None):
        """One multiplicative sweep: every vertex patch, colour by colour (multigrid.py:172-204)."""
        mode = mode or self.config.mode
        device.require_cuda()
        n = self.hier.n_dofs(level)
        xt, host = device.as_device(x, mode.torch_dtype, n)
        xt = xt.clone()
        bt, _ = device.as_device(b, mode.torch_dtype, n)
        self._smooth_device(level, xt, bt, mode)
        return device.to_host(xt, mode.storage_dtype) if host else xt

    # --------------------------------------------------------- coarse solve
    def _coarse_matrix(self) -> torch.Tensor:
        if "dense" not in self._coarse_cache:
            self._coarse_cache["dense"] = materialize_device(self.hier, self.config.coarse_level)
        return self._coarse_cache["dense"]

    def _coarse_factor(self, mode: PrecisionMode):
        """multigrid.py:215-228 -- the coarse matrix with operands demoted per mode, factorised once.  Up to
        COARSE_INVERSE_MAX unknowns the setup also forms its explicit inverse (fp64, from the LU factors) so that
        every V-cycle's coarse solve is one sf_dense_apply launch instead of two triangular solves."""
        if mode not in self._coarse_cache:
            A = self._coarse_matrix()
            if mode is PrecisionMode.FP64:
                Ad = A
            elif mode is PrecisionMode.FP32:
                Ad = A.float()
            elif mode is PrecisionMode.FP16:
                Ad = A.float().half().float()
            else:
                A32 = A.float()
                main = A32.half().float()
                resid = ((A32 - main) * 2048.0).half().float()
                Ad = main + resid / 2048.0
            if Ad.shape[0] <= COARSE_INVERSE_MAX:
                LU, piv = torch.linalg.lu_factor(Ad.double())
                eye = torch.eye(Ad.shape[0], dtype=torch.float64, device=Ad.device)
                self._coarse_cache[mode] = ("inverse", torch.linalg.lu_solve(LU, piv, eye).contiguous())
            else:
                self._coarse_cache[mode] = ("lu",) + tuple(torch.linalg.lu_factor(Ad))
        return self._coarse_cache[mode]

    def setup(self):
        """Eagerly build what the reference builds lazily inside the first solve."""
        device.require_cuda()
        self._coarse_factor(self.config.mode)
        return self

    def _coarse_solve_device(self, b: torch.Tensor, mode: PrecisionMode) -> torch.Tensor:
        fac = self._coarse_factor(mode)
        bs = b.to(mode.torch_dtype).contiguous()
        if fac[0] == "inverse":
            x = torch.empty_like(bs)
            device.dense_apply(fac[1], bs, x, demote16=mode is PrecisionMode.FP16)
            return x
        _, LU, piv = fac
        if mode is PrecisionMode.FP16:
            bs = bs.half().float()
        x = torch.linalg.lu_solve(LU, piv, bs.to(LU.dtype).reshape(-1, 1)).reshape(-1)
        return x.to(mode.torch_dtype)

    def coarse_solve(self, b, mode: PrecisionMode | None = None):
        """Direct dense solve at the coarse level (multigrid.py:230-239)."""
        mode = mode or self.config.mode
        device.require_cuda()
        bt, host = device.as_device(b, mode.torch_dtype, self.hier.n_dofs(self.config.coarse_level))
        x = self._coarse_solve_device(bt, mode)
        return device.to_host(x, mode.storage_dtype) if host else x

    # --------------------------------------------------------------- V-cycle
    def _vcycle_device(self, level: int, x: torch.Tensor, b: torch.Tensor, x_zero: bool = False):
        """multigrid.py:243-255, in place on device x (storage dtype); x_zero: x is zero on entry."""
        cfg = self.config
        mode = cfg.mode
        if level == cfg.coarse_level:
            x.copy_(self._coarse_solve_device(b, mode))
            return
        for i in range(cfg.pre_smooth_steps):
            self._smooth_device(level, x, b, mode, x_zero=x_zero and i == 0)
        rc = self._buf("rhs", level - 1, mode)
        restrict_device(self.hier, level, b, rc, mode, x=x)
        e = self._buf("x", level - 1, mode)
        e.zero_()
        self._vcycle_device(level - 1, e, rc, x_zero=True)
        prolongate_add_device(self.hier, level - 1, e, x, mode)
        for _ in range(cfg.post_smooth_steps):
            self._smooth_device(level, x, b, mode)

    def vcycle_device(self, x64: torch.Tensor | None, b64: torch.Tensor, level: int, out64: torch.Tensor):
        """fp64 device in/out; conversion to the storage dtype only here (multigrid.py:257-266).  x64 = None:
        zero initial guess (the preconditioner's apply), written straight into the storage-dtype buffer."""
        mode = self.config.mode
        xs = self._buf("x", level, mode)
        if x64 is None:
            xs.zero_()
        elif mode is PrecisionMode.FP64:
            xs.copy_(x64)
        else:
            device.convert(x64, xs)
        if mode is PrecisionMode.FP64:
            bs = b64
        else:
            bs = self._buf("rhs", level, mode)
            device.convert(b64, bs)
        self._vcycle_device(level, xs, bs, x_zero=x64 is None)
        device.convert(xs, out64)
        return out64

    def vcycle(self, x, b, level: int | None = None):
        """Run one V-cycle; fp64 in, fp64 out (multigrid.py:257-266)."""
        level = self.hier.max_level if level is None else level
        if not self.hier.min_level <= level <= self.hier.max_level:
            raise ValueError(f"level {level} outside hierarchy range")
        device.require_cuda()
        n = self.hier.n_dofs(level)
        xt, host = device.as_device(x, torch.float64, n)
        bt, _ = device.as_device(b, torch.float64, n)
        out = torch.empty(n, dtype=torch.float64, device="cuda")
        self.vcycle_device(xt, bt, level, out)
        return out.cpu().numpy() if host else out

    def apply(self, b, level: int | None = None):
        """Preconditioner action: one V-cycle from a zero initial guess (multigrid.py:268-270)."""
        level = self.hier.max_level if level is None else level
        if isinstance(b, torch.Tensor) and b.is_cuda:
            bt = b.reshape(-1).to(torch.float64).contiguous()
            if self.use_graph:
                return self._apply_graph(bt, level)
            out = torch.empty_like(bt)
            return self.vcycle_device(None, bt, level, out)
        return self.vcycle(np.zeros(np.asarray(b).size), b, level)

    # ------------------------------------------------------- CUDA graph
    use_graph = False

    def enable_graph(self, on: bool = True):
        """Replay each (level) V-cycle from a captured CUDA graph: the ~40 launches per level (16
        colour passes, transfers, coarse solve) cost one graph launch; the preconditioner input is
        copied into a static buffer first.  Same kernels, same arithmetic."""
        self.use_graph = on
        return self

    def _apply_graph(self, b: torch.Tensor, level: int) -> torch.Tensor:
        key = ("graph", level, b.numel())
        ent = self._buffers.get(key)
        if ent is None:
            b_in = torch.empty_like(b)
            out = torch.empty_like(b)
            b_in.copy_(b)
            self.vcycle_device(None, b_in, level, out)  # warm-up: workspaces, tables, LU factors
            torch.cuda.synchronize()
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                self.vcycle_device(None, b_in, level, out)
            ent = (g, b_in, out)
            self._buffers[key] = ent
        g, b_in, out = ent
        b_in.copy_(b)
        g.replay()
        return out.clone()


__all__ = ["default_ordering", "VCycleConfig", "PatchSolver", "patch_inverse_apply", "restrict", "prolongate",
           "MultigridPreconditioner", "vmult_device"]
