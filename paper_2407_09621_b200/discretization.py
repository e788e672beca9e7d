"""Mesh hierarchy and the matrix-free SIPG Laplacian on the B200.

Mirror of the reference's src/discretization.py API (MeshHierarchy,
build_hierarchy, apply_operator, materialize_operator) with the vmult executed
by the sm_100a kernel ``sf_vmult`` (csrc/sf_ops.cu).  The reference evaluates
the operator patch-wise (aligned tiling + Nitsche rim + three shifted face
passes, discretization.py:216-266); the kernel evaluates the algebraically
identical cell-wise form one 2x2x2-cell tile per CTA.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _native, device
from .basis import (Basis1D, basis_1d, cell_matrices_1d, cellwise_operator, embedding_1d, face_pieces,
                    patch_matrices_1d, smoother_matrices_1d)
from .precision import PrecisionMode


@dataclass
class LevelMatrices:
    """Per-level 1-D matrices (discretization.py:42-55) plus the packed kernel blocks."""

    h: float
    n_cells: int
    M_cell: np.ndarray
    L_cell: np.ndarray
    M_patch: np.ndarray
    L_tile: np.ndarray
    B_left: np.ndarray
    B_right: np.ndarray
    F_cross: np.ndarray
    L_smooth: dict = field(default_factory=dict)
    cell_op: np.ndarray | None = None  # M | D | ucol | urow | bl | br  (include/sumfact_b200.h)


class MeshHierarchy:
    """Nested uniform DG levels on [0,1]^3 (discretization.py:58-166)."""

    def __init__(self, max_level: int, degree: int, dim: int = 3, min_level: int = 1, max_dofs: int = 2**24):
        if max_level < 1:
            raise ValueError("need max_level >= 1 (vertex patches want 2 cells per axis)")
        if degree < 1:
            raise ValueError("degree must be at least 1")
        if dim not in (2, 3):
            raise ValueError("dim must be 2 or 3")
        if dim != 3:
            raise NotImplementedError("the B200 path is three-dimensional (2-D is out of scope, DESIGN.md §7)")
        if degree > _native.MAX_DEGREE:
            raise NotImplementedError(f"kernels are compiled for degree 1..{_native.MAX_DEGREE}")
        if min_level < 1 or min_level > max_level:
            raise ValueError("need 1 <= min_level <= max_level")
        self.max_level, self.min_level, self.degree, self.dim = max_level, min_level, degree, dim
        if self.n_dofs(max_level) > max_dofs:
            raise ValueError(f"level {max_level} has {self.n_dofs(max_level)} DoFs, cap is {max_dofs}")
        self.basis: Basis1D = basis_1d(degree)
        self.embedding = embedding_1d(degree)
        self.embedding_c = np.ascontiguousarray(self.embedding, dtype=np.float64)
        self._levels = {lvl: self._build_level(lvl) for lvl in range(min_level, max_level + 1)}

    # geometry (discretization.py:86-106)
    def n_cells(self, level: int) -> int:
        return 2**level

    def h(self, level: int) -> float:
        return 2.0**-level

    def axis_dofs(self, level: int) -> int:
        return self.n_cells(level) * (self.degree + 1)

    def n_dofs(self, level: int) -> int:
        return self.axis_dofs(level) ** self.dim

    def shape(self, level: int):
        return (self.axis_dofs(level),) * self.dim

    def levels(self):
        return range(self.min_level, self.max_level + 1)

    def matrices(self, level: int) -> LevelMatrices:
        return self._levels[level]

    def grid(self, level: int) -> _native.SfGrid:
        n = self.n_cells(level)
        return _native.SfGrid(n, n, n, None, None)

    def _build_level(self, level: int) -> LevelMatrices:
        """discretization.py:108-131."""
        k, h = self.degree, self.h(level)
        M_cell, L_cell = cell_matrices_1d(k, h)
        interior = patch_matrices_1d(k, h, "interior")
        left = patch_matrices_1d(k, h, "left")
        right = patch_matrices_1d(k, h, "right")
        names = {(False, False): "interior", (True, False): "left", (False, True): "right", (True, True): "both"}
        smooth = {key: smoother_matrices_1d(k, h, kind).L for key, kind in names.items()}
        pieces = face_pieces(k, h)
        lm = LevelMatrices(h=h, n_cells=self.n_cells(level), M_cell=M_cell, L_cell=L_cell, M_patch=interior.M,
                           L_tile=interior.L, B_left=left.L - interior.L, B_right=right.L - interior.L,
                           F_cross=pieces.F_center, L_smooth=smooth)
        lm.cell_op = cellwise_operator(M_cell, smooth, pieces.F_center, pieces)
        return lm

    # index maps (discretization.py:135-166)
    def cell_dof_indices(self, level: int, cell) -> np.ndarray:
        K, A = self.degree + 1, self.axis_dofs(level)
        idx = np.zeros((K,) * 3, dtype=np.int64)
        for a in range(3):
            shp = [1, 1, 1]
            shp[2 - a] = K
            idx = idx + ((cell[a] * K + np.arange(K, dtype=np.int64)) * A**a).reshape(shp)
        return idx.reshape(-1)

    def patch_dof_indices(self, level: int, shift, patch) -> np.ndarray:
        K, A = self.degree + 1, self.axis_dofs(level)
        B = 2 * K
        idx = np.zeros((B,) * 3, dtype=np.int64)
        for a in range(3):
            shp = [1, 1, 1]
            shp[2 - a] = B
            idx = idx + (((2 * patch[a] + shift[a]) * K + np.arange(B, dtype=np.int64)) * A**a).reshape(shp)
        return idx.reshape(-1)

    def patch_counts(self, level: int, shift):
        return tuple(self.n_cells(level) // 2 - s for s in shift)


def build_hierarchy(max_level: int, degree: int, dim: int = 3, min_level: int = 1,
                    max_dofs: int = 2**24) -> MeshHierarchy:
    return MeshHierarchy(max_level, degree, dim=dim, min_level=min_level, max_dofs=max_dofs)


# ------------------------------------------------------------------ vmult


def vmult_device(hier: MeshHierarchy, level: int, u: torch.Tensor, v: torch.Tensor, mode: PrecisionMode,
                 batch: int = 1, grid: _native.SfGrid | None = None):
    """Enqueue v = A u on the current stream (device tensors of the storage dtype)."""
    lm = hier.matrices(level)
    g = grid if grid is not None else hier.grid(level)
    rc = _native.lib().sf_vmult(mode.code, hier.degree, g, _native.host_ptr(lm.cell_op), device.ptr(u),
                                device.ptr(v), batch, device.stream_ptr())
    _native.check(rc, "sf_vmult")


def apply_operator(hier: MeshHierarchy, level: int, u, mode: PrecisionMode = PrecisionMode.FP64, out=None):
    """Matrix-free interior-penalty Laplacian at one level (discretization.py:216-266).

    numpy in -> numpy out (storage dtype of ``mode``); CUDA tensor in -> CUDA
    tensor out.  ``out`` (optional) receives the result: a host tensor (e.g.
    pinned, for streaming host buffers through the GPU) or a CUDA tensor.
    Host inputs of at least ``STREAM_MIN_DOFS`` entries are streamed through the
    GPU in z-slabs (copy-in, vmult and copy-out of consecutive slabs overlap).
    Raises ValueError on a length mismatch, like the reference.
    """
    n = hier.n_dofs(level)
    size = u.numel() if isinstance(u, torch.Tensor) else np.asarray(u).size
    if size != n:
        raise ValueError(f"expected {n} entries, got {size}")
    device.require_cuda()
    on_host = not (isinstance(u, torch.Tensor) and u.is_cuda)
    if on_host and n >= STREAM_MIN_DOFS and (out is None or not out.is_cuda):
        src = u if isinstance(u, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(np.asarray(u).reshape(-1)))
        if src.dtype != mode.torch_dtype:
            src = src.to(mode.torch_dtype)
        src = src.reshape(-1).contiguous()
        if out is None:
            dst_np = np.empty(n, dtype=mode.storage_dtype)
            _stream_vmult(hier, level, src, torch.from_numpy(dst_np), mode)
            return dst_np if not isinstance(u, torch.Tensor) else torch.from_numpy(dst_np)
        _stream_vmult(hier, level, src, out.reshape(-1), mode)
        return out
    if isinstance(u, torch.Tensor) and not u.is_cuda:
        t = u.reshape(-1).to(device="cuda", dtype=mode.torch_dtype, non_blocking=True)
        host = True
    else:
        t, host = device.as_device(u, mode.torch_dtype, n)
    if out is not None and out.is_cuda:
        vmult_device(hier, level, t, out, mode)
        return out
    v = torch.empty_like(t)
    vmult_device(hier, level, t, v, mode)
    if out is not None:
        out.copy_(v, non_blocking=True)
        torch.cuda.current_stream().synchronize()
        return out
    return device.to_host(v, mode.storage_dtype) if host else v


STREAM_MIN_DOFS = 1 << 24
_STREAM_BUFS: dict = {}  # device staging buffers + streams of the streamed host vmult (one set per device)


def _stream_vmult(hier: MeshHierarchy, level: int, u: torch.Tensor, v: torch.Tensor, mode: PrecisionMode,
                  slab_cells: int | None = None):
    """v = A u for HOST u, v: z-slabs of the vector flow host -> HBM -> host on three streams.

    Every cell layer of u crosses the host link exactly once, into a device-resident copy of u: slab i's
    copy-in brings its layers up to and including the first layer of slab i + 1 (its upper ghost), so its
    lower ghost is already resident from slab i - 1.  Slab i's vmult (sf_vmult with ghost_lo / ghost_hi
    pointing at the neighbouring layers -- the same mechanism as the multi-GPU halo) and its copy-out run on
    separate streams, so the transfers in both directions overlap each other and the kernel; the output
    is double buffered.
    """
    n, K = hier.n_cells(level), hier.degree + 1
    layer = K * (n * K) ** 2  # one cell layer of dofs
    if slab_cells is None:
        # 2 cells at level 7: tools/e2e_time.py 5.89-5.91 GDoF/s (4 cells: 5.77-5.88; 8: 5.51-5.89; 16: 5.60)
        # against the 5.7-6.1 GDoF/s the boxes' host links allow (tools/link_probe.py: 46-49 GB/s each way with
        # both directions busy)
        slab_cells = max(2, (n // 64) & ~1)
    slab_cells = min(slab_cells, n)
    dt = mode.torch_dtype
    key = (torch.cuda.current_device(), dt, slab_cells, layer, n)
    bufs = _STREAM_BUFS.get(key)
    if bufs is None:
        for k_old in [k for k in _STREAM_BUFS if k[0] == key[0]]:  # keep one set per device
            del _STREAM_BUFS[k_old]
        bufs = {"in": torch.empty(n * layer, dtype=dt, device="cuda"),
                "out": [torch.empty(slab_cells * layer, dtype=dt, device="cuda") for _ in range(2)],
                "streams": [torch.cuda.Stream() for _ in range(3)]}
        _STREAM_BUFS[key] = bufs
    s_in, s_run, s_out = bufs["streams"]
    main = torch.cuda.current_stream()
    for s in (s_in, s_run, s_out):
        s.wait_stream(main)
    out_free = [None, None]  # copy-out finished reading out[b]
    lm = hier.matrices(level)
    L = _native.lib()
    dev = bufs["in"]
    es = dev.element_size()
    base = dev.data_ptr()
    copied_to = 0  # cell layers of u resident on the device
    for i, z0 in enumerate(range(0, n, slab_cells)):
        b = i & 1
        z1 = min(n, z0 + slab_cells)
        obuf = bufs["out"][b]
        need = min(n, z1 + 1)  # this slab and its upper ghost layer
        with torch.cuda.stream(s_in):
            dev[copied_to * layer:need * layer].copy_(u[copied_to * layer:need * layer], non_blocking=True)
            loaded = torch.cuda.Event()
            loaded.record(s_in)
        copied_to = need
        s_run.wait_event(loaded)
        if out_free[b] is not None:
            s_run.wait_event(out_free[b])
        loc = base + z0 * layer * es
        ghost_lo = base + (z0 - 1) * layer * es if z0 > 0 else None
        ghost_hi = base + z1 * layer * es if z1 < n else None
        grid = _native.SfGrid(n, n, z1 - z0, ghost_lo, ghost_hi)
        rc = L.sf_vmult(mode.code, hier.degree, grid, _native.host_ptr(lm.cell_op), loc, obuf.data_ptr(), 1,
                        s_run.cuda_stream)
        _native.check(rc, "sf_vmult (streamed)")
        done = torch.cuda.Event()
        done.record(s_run)
        with torch.cuda.stream(s_out):
            s_out.wait_event(done)
            v[z0 * layer:z1 * layer].copy_(obuf[: (z1 - z0) * layer], non_blocking=True)
            copied = torch.cuda.Event()
            copied.record(s_out)
            out_free[b] = copied
    main.wait_stream(s_out)
    s_out.synchronize()
    return v


def materialize_device(hier: MeshHierarchy, level: int, mode: PrecisionMode = PrecisionMode.FP64,
                       chunk: int = 1024) -> torch.Tensor:
    """Dense operator on the device: column j = A e_j via batched vmults (discretization.py:269-279)."""
    device.require_cuda()
    n = hier.n_dofs(level)
    A = torch.empty((n, n), dtype=mode.torch_dtype, device="cuda")
    for j0 in range(0, n, chunk):
        m = min(chunk, n - j0)
        E = torch.zeros((m, n), dtype=mode.torch_dtype, device="cuda")
        E[torch.arange(m, device="cuda"), torch.arange(j0, j0 + m, device="cuda")] = 1.0
        out = torch.empty_like(E)
        vmult_device(hier, level, E, out, mode, batch=m)
        A[:, j0:j0 + m] = out.T
    return A


def materialize_operator(hier: MeshHierarchy, level: int, mode: PrecisionMode = PrecisionMode.FP64) -> np.ndarray:
    """Dense fp64 operator matrix (small levels only), discretization.py:269-279."""
    return materialize_device(hier, level, mode).double().cpu().numpy()


# ----------------------------------------------------- pre/post-processing
# Load vector, interpolation, error norms and the manufactured problem
# (discretization.py:317-531).  These are setup/reporting steps outside the
# hot path (SURVEY.md §8f "next"); round 1 evaluates them on the host with the
# same sum-factorised quadrature as the reference.


def _axis_points(hier, level, pts):
    n, h = hier.n_cells(level), hier.h(level)
    return ((np.arange(n)[:, None] + np.asarray(pts)[None, :]) * h).ravel()


def _coords(axis_pts):
    Z, Y, X = np.meshgrid(axis_pts, axis_pts, axis_pts, indexing="ij")
    return X, Y, Z


# ------------------------------------------- device pre/post-processing, general data
# The reference evaluates f, g and the exact solution on the full Gauss-point grid and contracts with
# numpy (discretization.py:317-459).  Here the contractions are the library's own sum-factorised
# kernels (csrc/sf_quad.cu) and the data are tabulated one z-chunk of cells at a time: on the device
# when the callable accepts CUDA tensors (torch operations), else on the host for that chunk only.


def _eval_chunk(fn, X, Y, Z, shape):
    """fn at the broadcast coordinates X (1,1,nx), Y (1,ny,1), Z (nz,1,1) -> contiguous fp64 CUDA tensor."""
    try:
        v = fn(X, Y, Z)
        if isinstance(v, torch.Tensor) and v.is_cuda:
            return v.to(torch.float64).expand(shape).contiguous()
    except Exception:  # numpy-only callable (the reference's convention): evaluate this chunk on the host
        pass
    Xh, Yh, Zh = (t.cpu().numpy() for t in (X, Y, Z))
    v = np.broadcast_to(np.asarray(fn(Xh, Yh, Zh), dtype=np.float64), shape)
    return torch.from_numpy(np.ascontiguousarray(v)).cuda()


def _eval_chunk_vec(fn, X, Y, Z, shape):
    """a vector-valued callable (the gradient): 3 components as CUDA tensors."""
    try:
        v = fn(X, Y, Z)
        if all(isinstance(c, torch.Tensor) and c.is_cuda for c in v):
            return [c.to(torch.float64).expand(shape).contiguous() for c in v]
    except Exception:
        pass
    Xh, Yh, Zh = (t.cpu().numpy() for t in (X, Y, Z))
    return [torch.from_numpy(np.ascontiguousarray(np.broadcast_to(np.asarray(c, dtype=np.float64), shape))).cuda()
            for c in fn(Xh, Yh, Zh)]


class _QuadLevel:
    """Gauss rule, evaluation matrices and device copies for one (level, q)."""

    def __init__(self, hier, level, q):
        from .basis import gauss_rule, lagrange_derivatives, lagrange_values

        self.n, self.h, self.K, self.k = hier.n_cells(level), hier.h(level), hier.degree + 1, hier.degree
        self.rule = gauss_rule(q)
        self.q = q
        self.S = lagrange_values(hier.basis.nodes, self.rule.points)             # (q, K)
        self.D = lagrange_derivatives(hier.basis.nodes, self.rule.points) / self.h
        self.ax = _axis_points(hier, level, self.rule.points)                    # (n q,)
        cu = lambda a: torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64)).cuda()
        self.ax_d = cu(self.ax)
        self.w_d = cu(np.tile(self.rule.weights, self.n) * self.h)
        self.ST_d = cu(self.S.T)
        self.mats_d = {None: cu(np.concatenate([self.S.ravel()] * 3))}
        for a in range(3):
            self.mats_d[a] = cu(np.concatenate([(self.D if b == a else self.S).ravel() for b in range(3)]))

    def chunk_cells(self, limit_points=1 << 27):
        return max(1, limit_points // ((self.n * self.q) ** 2 * self.q))

    def coords(self, z0, nz):
        nq = self.n * self.q
        X = self.ax_d.view(1, 1, nq)
        Y = self.ax_d.view(1, nq, 1)
        Z = self.ax_d[z0 * self.q:(z0 + nz) * self.q].view(nz * self.q, 1, 1)
        return X, Y, Z, (nz * self.q, nq, nq)


def _zrange(hier, level, z_cells):
    n = hier.n_cells(level)
    z0, nz = (0, n) if z_cells is None else (int(z_cells[0]), int(z_cells[1]))
    if z0 < 0 or nz < 1 or z0 + nz > n:
        raise ValueError(f"z-cell range {z_cells} outside [0, {n})")
    return z0, nz


def assemble_rhs_device(hier: MeshHierarchy, level: int, f, g=None, quad_points: int | None = None,
                        z_cells=None) -> torch.Tensor:
    """Load vector (discretization.py:317-394) on the device: cell integrals of f v by sf_quad_load, the
    Nitsche data terms of g by sf_face_load.  z_cells = (z0, nz): only that z-slab of cells (slab-local
    vector, what a multi-GPU rank owns); default the whole level."""
    from .basis import lagrange_derivatives, lagrange_values, penalty

    device.require_cuda()
    k = hier.degree
    Q = _QuadLevel(hier, level, quad_points or (k + 2))
    n, K, q = Q.n, Q.K, Q.q
    z0, nz = _zrange(hier, level, z_cells)
    b = torch.empty(nz * K * (n * K) ** 2, dtype=torch.float64, device="cuda")
    L = _native.lib()
    step = Q.chunk_cells()
    layer = K * (n * K) ** 2
    for c0 in range(z0, z0 + nz, step):
        c1 = min(c0 + step, z0 + nz)
        X, Y, Z, shape = Q.coords(c0, c1 - c0)
        fq = _eval_chunk(f, X, Y, Z, shape)
        rc = L.sf_quad_load(k, q, n, c0, c1 - c0, device.ptr(fq), device.ptr(Q.ST_d), device.ptr(Q.w_d),
                            device.ptr(b) + (c0 - z0) * layer * 8, device.stream_ptr())
        _native.check(rc, "sf_quad_load")
    if g is not None:
        nodes, h = hier.basis.nodes, Q.h
        gamma = penalty(k, h, h)
        coef = {0: gamma * lagrange_values(nodes, [0.0])[0] + lagrange_derivatives(nodes, [0.0])[0] / h,
                1: gamma * lagrange_values(nodes, [1.0])[0] - lagrange_derivatives(nodes, [1.0])[0] / h}
        nq = n * q
        A = Q.ax_d
        for a in range(3):  # tensor axis of the face normal
            for side in (0, 1):
                if a == 2 and not (z0 <= (0 if side == 0 else n - 1) < z0 + nz):
                    continue  # z face outside this slab
                pin = torch.full((1, 1), float(side), dtype=torch.float64, device="cuda")
                slow, fast = A.view(nq, 1), A.view(1, nq)  # face grid (slow, fast) = tangential axes (z|y, y|x)
                if a == 0:
                    gv = _eval_chunk(g, pin, fast, slow, (nq, nq))
                elif a == 1:
                    gv = _eval_chunk(g, fast, pin, slow, (nq, nq))
                else:
                    gv = _eval_chunk(g, fast, slow, pin, (nq, nq))
                cf = torch.from_numpy(np.ascontiguousarray(coef[side], dtype=np.float64)).cuda()
                rc = L.sf_face_load(k, q, n, z0, nz, a, side, device.ptr(gv), device.ptr(Q.ST_d),
                                    device.ptr(Q.w_d), device.ptr(cf), device.ptr(b), device.stream_ptr())
                _native.check(rc, "sf_face_load")
    return b


def _quad_error_sq(hier, level, u_h: torch.Tensor, fn, deriv_axis, quad_points, z_cells, vector=False):
    """device scalar: sum over the z-slab of w (I u_h - fn)^2 (per gradient component when vector)."""
    k = hier.degree
    Q = _QuadLevel(hier, level, quad_points or (k + 3))
    n, K, q = Q.n, Q.K, Q.q
    z0, nz = _zrange(hier, level, z_cells)
    u = u_h.reshape(-1)
    if u.numel() != nz * K * (n * K) ** 2:
        raise ValueError(f"expected {nz * K * (n * K) ** 2} entries, got {u.numel()}")
    u = u.to(torch.float64).contiguous()
    L = _native.lib()
    step = Q.chunk_cells()
    layer = K * (n * K) ** 2
    part = torch.empty(n * n * step, dtype=torch.float64, device="cuda")
    total = torch.zeros(1, dtype=torch.float64, device="cuda")
    out = torch.empty(1, dtype=torch.float64, device="cuda")
    axes = (0, 1, 2) if vector else (deriv_axis,)
    for c0 in range(z0, z0 + nz, step):
        c1 = min(c0 + step, z0 + nz)
        X, Y, Z, shape = Q.coords(c0, c1 - c0)
        vals = _eval_chunk_vec(fn, X, Y, Z, shape) if vector else [_eval_chunk(fn, X, Y, Z, shape)]
        for a, fq in zip(axes, vals):
            rc = L.sf_quad_error(k, q, n, c0, c1 - c0, device.ptr(u) + (c0 - z0) * layer * 8,
                                 device.ptr(Q.mats_d[a]), device.ptr(fq), device.ptr(Q.w_d), device.ptr(part),
                                 device.ptr(out), device.stream_ptr())
            _native.check(rc, "sf_quad_error")
            total += out
    return total


def l2_error_device(hier: MeshHierarchy, level: int, u_h, exact, quad_points: int | None = None,
                    z_cells=None) -> torch.Tensor:
    """Sum of squares of the L2 error over a z-slab (device scalar; sqrt of the all-slab sum = l2_error)."""
    return _quad_error_sq(hier, level, device.as_device(u_h, torch.float64)[0], exact, None, quad_points, z_cells)


def h1_error_device(hier: MeshHierarchy, level: int, u_h, grad_exact, quad_points: int | None = None,
                    z_cells=None) -> torch.Tensor:
    """Sum of squares of the broken H1-seminorm error over a z-slab (device scalar)."""
    return _quad_error_sq(hier, level, device.as_device(u_h, torch.float64)[0], grad_exact, None, quad_points,
                          z_cells, vector=True)


def assemble_rhs(hier: MeshHierarchy, level: int, f, g=None, quad_points: int | None = None) -> np.ndarray:
    """Load vector: cell integrals of f v (+ Nitsche data terms for g), discretization.py:317-394.
    Computed on the device (assemble_rhs_device); returned as numpy like the reference."""
    return assemble_rhs_device(hier, level, f, g, quad_points).cpu().numpy()


def interpolate(hier: MeshHierarchy, level: int, func) -> np.ndarray:
    """Nodal interpolant on the Gauss-Lobatto product grid (discretization.py:397-402)."""
    ax = _axis_points(hier, level, hier.basis.nodes)
    return np.broadcast_to(np.asarray(func(*_coords(ax)), dtype=np.float64), hier.shape(level)).reshape(-1).copy()


def l2_error(hier: MeshHierarchy, level: int, u_h, exact, quad_points: int | None = None) -> float:
    """L2 distance between a DoF vector and a callable (discretization.py:431-441), on the device."""
    return float(torch.sqrt(l2_error_device(hier, level, u_h, exact, quad_points)))


def h1_seminorm_error(hier: MeshHierarchy, level: int, u_h, grad_exact, quad_points: int | None = None) -> float:
    """Broken H1-seminorm distance (discretization.py:444-459), on the device."""
    return float(torch.sqrt(h1_error_device(hier, level, u_h, grad_exact, quad_points)))



# ---------------------------------------------------------- serialization (discretization.py:462-488)


def save_vector(path, u, fmt: str = "csv"):
    """discretization.py:465-476: CSV ``index,value`` rows (17 significant digits) or flat f64 binary.
    Accepts numpy arrays and torch tensors (CUDA tensors are read back once)."""
    if isinstance(u, torch.Tensor):
        u = u.detach().cpu().numpy()
    u = np.asarray(u, dtype=np.float64).ravel()
    if fmt == "csv":
        with open(path, "w") as fh:
            fh.write("index,value\n")
            if u.size:
                np.savetxt(fh, np.column_stack([np.arange(u.size, dtype=np.float64), u]), fmt="%d,%.17g")
    elif fmt == "bin":
        u.tofile(path)
    else:
        raise ValueError(f"unknown vector format {fmt!r}")


def load_vector(path, fmt: str = "csv") -> np.ndarray:
    """discretization.py:479-488: rows are put back in index order."""
    if fmt == "csv":
        data = np.genfromtxt(path, delimiter=",", skip_header=1)
        if data.ndim == 1:  # single row
            data = data.reshape(1, -1)
        order = np.argsort(data[:, 0], kind="stable")
        return data[order, 1].copy()
    if fmt == "bin":
        return np.fromfile(path, dtype=np.float64)
    raise ValueError(f"unknown vector format {fmt!r}")

@dataclass
class ModelProblem:
    exact: callable
    rhs: callable
    gradient: callable
    boundary: callable | None = None


def sine_product_problem(dim: int = 3) -> ModelProblem:
    """Product-of-sines solution, f = 3 pi^2 u, zero Dirichlet data (discretization.py:504-531)."""
    if dim != 3:
        raise NotImplementedError("the B200 path is three-dimensional")
    pi = np.pi
    exact = lambda x, y, z: np.sin(pi * x) * np.sin(pi * y) * np.sin(pi * z)
    rhs = lambda x, y, z: 3.0 * pi**2 * exact(x, y, z)

    def gradient(x, y, z):
        return (pi * np.cos(pi * x) * np.sin(pi * y) * np.sin(pi * z),
                pi * np.sin(pi * x) * np.cos(pi * y) * np.sin(pi * z),
                pi * np.sin(pi * x) * np.sin(pi * y) * np.cos(pi * z))

    return ModelProblem(exact=exact, rhs=rhs, gradient=gradient)


# ------------------------------------------- device pre/post-processing
# Separable data (the manufactured sine problem) never needs the host: the load
# vector is a tensor product of 1-D quadrature sums, and the L2 error is
# evaluated per z-slab of cells on the device.  Same quadrature as the
# reference (k+2 points for the load, k+3 for the error).


def _rhs_1d(hier, level, f1, q):
    from .basis import gauss_rule, lagrange_values

    n, h, K = hier.n_cells(level), hier.h(level), hier.degree + 1
    rule = gauss_rule(q)
    S = lagrange_values(hier.basis.nodes, rule.points)  # (q, K)
    pts = (np.arange(n)[:, None] + rule.points[None, :]) * h
    vals = f1(pts) * rule.weights[None, :] * h  # (n, q)
    return (vals @ S).reshape(n * K)  # (n*K,)


def assemble_rhs_separable(hier: MeshHierarchy, level: int, f1, scale: float = 1.0, z_cells=None) -> torch.Tensor:
    """Load vector of f = scale * f1(x) f1(y) f1(z) on the device (fp64, flat (z,y,x)); z_cells = (z0, nz):
    only that z-slab of cells (O(local DoF) memory on a multi-GPU rank)."""
    device.require_cuda()
    b1 = torch.from_numpy(_rhs_1d(hier, level, f1, hier.degree + 2)).cuda()
    z0, nz = _zrange(hier, level, z_cells)
    K = hier.degree + 1
    bz = b1[z0 * K:(z0 + nz) * K]
    return (scale * bz[:, None, None] * b1[None, :, None] * b1[None, None, :]).reshape(-1).contiguous()


def _separable_error_sq(hier, level, u_h, mats, factors, slab_cells=8, nz=None):
    """sum_q w_q (I u_h - scale * f_z f_y f_x)^2 over k+3-point Gauss points, slab by slab on the device.

    mats[a]: (q, K) evaluation matrix along tensor axis a (values or derivatives);
    factors[a]: the exact 1-D factor along axis a at the n*q points (scale folded into axis 0);
    nz: cells along z of u_h (a z-slab of the level; factors[2] then covers those nz cells).
    """
    from .basis import gauss_rule

    n, h, K = hier.n_cells(level), hier.h(level), hier.degree + 1
    rule = gauss_rule(hier.degree + 3)
    q = len(rule.points)
    Sx, Sy, Sz = (torch.from_numpy(np.ascontiguousarray(m)).cuda() for m in mats)
    fx, fy, fz = (torch.from_numpy(np.ascontiguousarray(f).reshape(-1)).cuda() for f in factors)
    w1 = torch.from_numpy(np.tile(rule.weights, n) * h).cuda()
    nzc = n if nz is None else nz
    U = u_h.reshape(nzc, K, n, K, n, K)
    total = torch.zeros((), dtype=torch.float64, device="cuda")
    for z0 in range(0, nzc, slab_cells):
        blk = U[z0:z0 + slab_cells]
        t = torch.einsum("qk,zkylxm->zqylxm", Sz, blk)
        t = torch.einsum("qk,zaykxm->zayqxm", Sy, t)
        t = torch.einsum("qk,zaybxk->zaybxq", Sx, t)
        nz = blk.shape[0]
        t = t.reshape(nz * q, n * q, n * q)
        zi = slice(z0 * q, (z0 + nz) * q)
        exact = fz[zi][:, None, None] * fy[None, :, None] * fx[None, None, :]
        W = w1[zi][:, None, None] * w1[None, :, None] * w1[None, None, :]
        total += (W * (t - exact) ** 2).sum()
    return total


def l2_error_separable(hier: MeshHierarchy, level: int, u_h: torch.Tensor, e1, scale: float = 1.0,
                       slab_cells: int = 8) -> float:
    """L2 distance between u_h (device) and scale * e1(x) e1(y) e1(z), k+3-point Gauss quadrature
    (the reference's l2_error, discretization.py:431-441, for separable exact solutions)."""
    from .basis import gauss_rule, lagrange_values

    n, h = hier.n_cells(level), hier.h(level)
    rule = gauss_rule(hier.degree + 3)
    S = lagrange_values(hier.basis.nodes, rule.points)
    pts = (np.arange(n)[:, None] + rule.points[None, :]) * h
    f = e1(pts)
    total = _separable_error_sq(hier, level, u_h, (S, S, S), (f, f, scale * f), slab_cells)
    return float(torch.sqrt(total))


def h1_seminorm_error_separable(hier: MeshHierarchy, level: int, u_h: torch.Tensor, e1, de1, scale: float = 1.0,
                                slab_cells: int = 8) -> float:
    """H1-seminorm distance to scale * e1 e1 e1 with d/dx e1 = de1 (discretization.py:444-459), on the device."""
    from .basis import gauss_rule, lagrange_derivatives, lagrange_values

    n, h = hier.n_cells(level), hier.h(level)
    rule = gauss_rule(hier.degree + 3)
    S = lagrange_values(hier.basis.nodes, rule.points)
    Dm = lagrange_derivatives(hier.basis.nodes, rule.points) / h
    pts = (np.arange(n)[:, None] + rule.points[None, :]) * h
    f, df = e1(pts), de1(pts)
    total = torch.zeros((), dtype=torch.float64, device="cuda")
    for a in range(3):
        mats = tuple(Dm if b == a else S for b in range(3))
        facs = [df if b == a else f for b in range(3)]
        facs[2] = scale * facs[2]
        total += _separable_error_sq(hier, level, u_h, mats, facs, slab_cells)
    return float(torch.sqrt(total))
