"""numpy restatement of the reference SIPG hot path (TEST INFRASTRUCTURE ONLY).

Every function cites the reference file:line it restates (paths relative to
``/root/reference/pkg/src/sumfact``).  The arithmetic follows the reference's
schedule -- the same 1-D matrices, the same patch-tiled operator passes, the
same contraction order (tensor x, then y, then z inside a Kronecker term), the
same precision demotion per contraction -- so that the port reproduces the
reference to rounding (checked against golden vectors from the reference in
``tests/test_oracle_golden.py``).  3-D only (the hot path's dimension).

Nothing in the product package imports this module.
"""

from __future__ import annotations

import itertools
import math
import os
from dataclasses import dataclass, field

import numpy as np
import scipy.linalg
from scipy.special import roots_jacobi

DIM = 3
EC_SCALE = np.float32(2048.0)  # precision.py:19
MODES = ("fp64", "fp32", "fp16", "fp16_ec")  # precision.py:29-33


def storage_dtype(mode: str):
    """precision.py:36-39 -- fp64 keeps f64 vectors, every other mode f32."""
    return np.float64 if mode == "fp64" else np.float32


# ------------------------------------------------------------ 1-D setup


def gauss_points_weights(q: int):
    """basis.py:34-39 -- Gauss-Legendre on [0, 1]."""
    x, w = np.polynomial.legendre.leggauss(q)
    return (x + 1.0) / 2.0, w / 2.0


def lobatto_nodes(k: int) -> np.ndarray:
    """basis.py:42-49 -- k+1 Gauss-Lobatto points on [0, 1]."""
    if k == 1:
        return np.array([0.0, 1.0])
    inner, _ = roots_jacobi(k - 1, 1.0, 1.0)
    return np.concatenate(([0.0], (inner + 1.0) / 2.0, [1.0]))


def lagrange_table(nodes, pts) -> np.ndarray:
    """basis.py:52-62 -- basis values, one row per point (product formula)."""
    nodes = np.asarray(nodes, dtype=float)
    pts = np.atleast_1d(np.asarray(pts, dtype=float))
    tab = np.ones((pts.size, nodes.size))
    for j in range(nodes.size):
        for m in range(nodes.size):
            if m != j:
                tab[:, j] *= (pts - nodes[m]) / (nodes[j] - nodes[m])
    return tab


def lagrange_slope_table(nodes, pts) -> np.ndarray:
    """basis.py:65-80 -- basis derivatives, one row per point."""
    nodes = np.asarray(nodes, dtype=float)
    pts = np.atleast_1d(np.asarray(pts, dtype=float))
    n = nodes.size
    tab = np.zeros((pts.size, n))
    for j in range(n):
        for l in range(n):
            if l == j:
                continue
            term = np.full(pts.size, 1.0 / (nodes[j] - nodes[l]))
            for m in range(n):
                if m != j and m != l:
                    term *= (pts - nodes[m]) / (nodes[j] - nodes[m])
            tab[:, j] += term
    return tab


def cell_mass_stiffness(k: int, h: float):
    """basis.py:123-132 -- h*S^T W S and (1/h)*D^T W D on a (k+1)-point Gauss rule."""
    pts, wts = gauss_points_weights(k + 1)
    nodes = lobatto_nodes(k)
    S = lagrange_table(nodes, pts)
    D = lagrange_slope_table(nodes, pts)
    return h * (S.T * wts) @ S, (1.0 / h) * (D.T * wts) @ D


def embedding(k: int) -> np.ndarray:
    """basis.py:243-252 -- (2K x K) coarse basis evaluated at both children's nodes."""
    nodes = lobatto_nodes(k)
    return np.vstack([lagrange_table(nodes, nodes / 2.0), lagrange_table(nodes, (nodes + 1.0) / 2.0)])


@dataclass
class Level1D:
    """discretization.py:42-55 -- the per-level 1-D matrices."""

    h: float
    n: int
    M_cell: np.ndarray
    L_cell: np.ndarray
    M_patch: np.ndarray
    L_tile: np.ndarray
    B_left: np.ndarray
    B_right: np.ndarray
    F_cross: np.ndarray
    L_smooth: dict = field(default_factory=dict)


def level_matrices(k: int, level: int) -> Level1D:
    """basis.py:149-231 + discretization.py:108-131 -- patch pieces and level matrices."""
    h = 2.0 ** -level
    K = k + 1
    nodes = lobatto_nodes(k)
    Mc, Lc = cell_mass_stiffness(k, h)
    Mp = np.zeros((2 * K, 2 * K))
    Mp[:K, :K] = Mc
    Mp[K:, K:] = Mc
    Lcells = np.zeros((2 * K, 2 * K))
    Lcells[:K, :K] = Lc
    Lcells[K:, K:] = Lc
    gamma = k * (k + 1) * (1.0 / h + 1.0 / h)  # basis.py:116-120
    slope = lambda x: lagrange_slope_table(nodes, [x])[0] / h
    value = lambda x: lagrange_table(nodes, [x])[0]

    jump = np.concatenate([value(1.0), -value(0.0)])
    avg = np.concatenate([0.5 * slope(1.0), 0.5 * slope(0.0)])
    F = gamma * np.outer(jump, jump) - np.outer(avg, jump) - np.outer(jump, avg)

    z = np.zeros(K)
    e0 = np.concatenate([value(0.0), z])
    d0 = np.concatenate([slope(0.0), z])
    e1 = np.concatenate([z, value(1.0)])
    d1 = np.concatenate([z, slope(1.0)])
    Bl = gamma * np.outer(e0, e0) + np.outer(d0, e0) + np.outer(e0, d0)
    Br = gamma * np.outer(e1, e1) - np.outer(d1, e1) - np.outer(e1, d1)
    Hl = gamma * np.outer(e0, e0) + 0.5 * (np.outer(d0, e0) + np.outer(e0, d0))
    Hr = gamma * np.outer(e1, e1) - 0.5 * (np.outer(d1, e1) + np.outer(e1, d1))

    tile = Lcells + F  # patch_matrices_1d(..., "interior")
    left = tile + Bl
    right = tile + Br
    smooth = {}
    for lb in (False, True):
        for rb in (False, True):
            base = Lcells + F
            base = base + (Bl if lb else Hl)
            base = base + (Br if rb else Hr)
            smooth[(lb, rb)] = base
    return Level1D(h=h, n=2 ** level, M_cell=Mc, L_cell=Lc, M_patch=Mp, L_tile=tile,
                   B_left=left - tile, B_right=right - tile, F_cross=F, L_smooth=smooth)


class Hierarchy:
    """discretization.py:58-166 -- nested cube levels min_level..max_level (3-D)."""

    def __init__(self, max_level: int, degree: int, min_level: int = 1):
        self.max_level, self.min_level, self.degree = max_level, min_level, degree
        self.P = embedding(degree)
        self.levels = {l: level_matrices(degree, l) for l in range(min_level, max_level + 1)}

    def A(self, level):
        return 2 ** level * (self.degree + 1)

    def n_dofs(self, level):
        return self.A(level) ** DIM

    def shape(self, level):
        return (self.A(level),) * DIM


# ----------------------------------------------------------- contraction


# Single-threaded contraction backend (_core/__init__.py:12-24 picks one at import time):
# "einsum" = the reference's numpy fallback (_core/fallback.py:10-15), "compiled" = the
# reference's own Cython kernel contract_f8/_f4 built from its sources into oracle/_ref
# (oracle/build_ref.py) -- both exactly as the reference ships them.
BACKEND = "einsum"
_REF_KERNEL = None


def set_backend(name: str) -> str:
    """Select "einsum" or "compiled" (needs oracle/_ref); returns the previous backend."""
    global BACKEND, _REF_KERNEL
    if name not in ("einsum", "compiled"):
        raise ValueError(name)
    if name == "compiled" and _REF_KERNEL is None:
        from oracle import build_ref

        _REF_KERNEL = build_ref.load()
        if _REF_KERNEL is None:
            raise RuntimeError("oracle/_ref is not built (python oracle/build_ref.py)")
    prev, BACKEND = BACKEND, name
    return prev


def contract(m: np.ndarray, w: np.ndarray, axis: int, threads: int = 1) -> np.ndarray:
    """_core/__init__.py:27-59 + _core/fallback.py:10-15: out[o,i,r] = sum_k m[i,k] w[o,k,r].

    threads == 1: numpy einsum without ``optimize`` -- the reference's own
    fallback backend, single-threaded, ascending k (the checker path); or, with
    set_backend("compiled"), the reference's compiled kernel from oracle/_ref.
    threads > 1: the same contraction as BLAS GEMMs (np.matmul) on ``threads``
    BLAS threads -- used only for the multi-core CPU *baseline* timing; it
    differs from einsum by summation order only (~1e-16 relative).
    """
    w = np.ascontiguousarray(w)
    m = np.ascontiguousarray(m, dtype=w.dtype)
    outer = int(np.prod(w.shape[:axis], dtype=np.int64))
    inner = int(np.prod(w.shape[axis + 1:], dtype=np.int64))
    w3 = w.reshape(outer, w.shape[axis], inner)
    shape = w.shape[:axis] + (m.shape[0],) + w.shape[axis + 1:]
    if threads <= 1:
        out = np.empty((outer, m.shape[0], inner), dtype=w.dtype)
        if BACKEND == "compiled":  # _core/__init__.py:53-58 -> _contract.pyx:14-45
            (_REF_KERNEL.contract_f8 if w.dtype == np.float64 else _REF_KERNEL.contract_f4)(w3, m, out)
        else:
            np.einsum("ik,okr->oir", m, w3, out=out)
        return out.reshape(shape)
    from threadpoolctl import threadpool_limits

    with threadpool_limits(limits=threads, user_api="blas"):
        if inner == 1:
            out = w3.reshape(outer, -1) @ m.T
        else:
            out = np.matmul(m, w3)
    return out.reshape(shape)


def demote16(x):
    """precision.py:130-137 -- round fp32 through binary16 (RNE, subnormals kept)."""
    with np.errstate(over="ignore"):
        return np.asarray(x, dtype=np.float32).astype(np.float16).astype(np.float32)


def ec_split(x32):
    """precision.py:168-174 -- main half and 2^11-scaled residual half, both as f32."""
    with np.errstate(over="ignore"):
        main = x32.astype(np.float16).astype(np.float32)
        resid = ((x32 - main) * EC_SCALE).astype(np.float16).astype(np.float32)
    return main, resid


def contract_mode(m, w, axis, mode, threads=1):
    """precision.py:206-230 -- one contraction under a precision mode."""
    if mode == "fp64":
        return contract(np.asarray(m, np.float64), np.asarray(w, np.float64), axis, threads)
    m32 = np.asarray(m, np.float32)
    w32 = np.asarray(w, np.float32)
    if mode == "fp32":
        return contract(m32, w32, axis, threads)
    if mode == "fp16":
        return contract(demote16(m32), demote16(w32), axis, threads)
    if mode == "fp16_ec":
        mh, dm = ec_split(m32)
        wh, dw = ec_split(w32)
        main = contract(mh, wh, axis, threads)
        corr = contract(dm, wh, axis, threads) + contract(mh, dw, axis, threads)
        return main + corr / EC_SCALE
    raise ValueError(mode)


def _kron_block(w, mats, mode, threads=1):
    """discretization.py:201-210 -- mats[b] along numpy block axis b; x (axis 5) first."""
    out = w
    for b in (2, 1, 0):
        out = contract_mode(mats[b], out, DIM + b, mode, threads)
    return out


def patches(arr, starts, counts, B):
    """discretization.py:176-185 -- (cz,cy,cx,B,B,B) patch batch from a level array."""
    sub = arr[starts[0]:starts[0] + counts[0] * B,
              starts[1]:starts[1] + counts[1] * B,
              starts[2]:starts[2] + counts[2] * B]
    sub = sub.reshape(counts[0], B, counts[1], B, counts[2], B)
    return np.ascontiguousarray(sub.transpose(0, 2, 4, 1, 3, 5))


def add_patches(v, batch, starts, counts, B):
    """discretization.py:188-198 -- accumulate a patch batch back into a level array."""
    flat = batch.transpose(0, 3, 1, 4, 2, 5).reshape(counts[0] * B, counts[1] * B, counts[2] * B)
    v[starts[0]:starts[0] + counts[0] * B,
      starts[1]:starts[1] + counts[1] * B,
      starts[2]:starts[2] + counts[2] * B] += flat


# ------------------------------------------------------------- the vmult


def apply_operator(H: Hierarchy, level: int, u, mode="fp64", threads=1) -> np.ndarray:
    """discretization.py:216-266 -- aligned pass + Nitsche rim + 3 shifted face passes."""
    u = np.asarray(u)
    if u.size != H.n_dofs(level):
        raise ValueError(f"expected {H.n_dofs(level)} entries, got {u.size}")
    lm = H.levels[level]
    K = H.degree + 1
    B = 2 * K
    p = lm.n // 2
    dt = storage_dtype(mode)
    arr = u.reshape(H.shape(level)).astype(dt, copy=False)
    v = np.zeros(H.shape(level), dtype=dt)

    zero3, full = (0, 0, 0), (p, p, p)
    w = patches(arr, zero3, full, B)
    out = np.zeros_like(w)
    for t in range(DIM):
        out += _kron_block(w, [lm.L_tile if b == t else lm.M_patch for b in range(DIM)], mode, threads)
    for t in range(DIM):
        for lo, Bm in ((True, lm.B_left), (False, lm.B_right)):
            sel = [slice(None)] * (2 * DIM)
            sel[t] = slice(0, 1) if lo else slice(p - 1, p)
            sel = tuple(sel)
            out[sel] += _kron_block(w[sel], [Bm if b == t else lm.M_patch for b in range(DIM)],
                                    mode, threads)
    add_patches(v, out, zero3, full, B)

    if p >= 2:
        for t in range(DIM):
            st = tuple(K if d == t else 0 for d in range(DIM))
            ct = tuple(p - 1 if d == t else p for d in range(DIM))
            w = patches(arr, st, ct, B)
            add_patches(v, _kron_block(w, [lm.F_cross if b == t else lm.M_patch for b in range(DIM)],
                                       mode, threads), st, ct, B)
    return v.reshape(-1)


def materialize(H: Hierarchy, level: int) -> np.ndarray:
    """discretization.py:269-279 -- dense fp64 operator (column j = A e_j)."""
    n = H.n_dofs(level)
    A = np.empty((n, n))
    e = np.zeros(n)
    for j in range(n):
        e[j] = 1.0
        A[:, j] = apply_operator(H, level, e)
        e[j] = 0.0
    return A


# ------------------------------------------------------------- multigrid


class PatchInverse:
    """multigrid.py:47-83 -- fast-diagonalization inverse per boundary kind."""

    def __init__(self, M, L_by_kind):
        self.eig = {kind: scipy.linalg.eigh(L, M) for kind, L in L_by_kind.items()}

    def lam_sum(self, kinds):
        """multigrid.py:60-69 -- lambda_i + lambda_j + lambda_k over block axes."""
        tot = np.zeros((1, 1, 1))
        for d, kind in enumerate(kinds):
            shp = [1, 1, 1]
            lam = self.eig[kind][0]
            shp[d] = lam.size
            tot = tot + lam.reshape(shp)
        return tot

    def apply(self, w, kinds, mode, threads=1):
        """multigrid.py:71-83 -- V^T x3, divide, V x3 (x axis first each time)."""
        t = w
        for b in (2, 1, 0):
            t = contract_mode(np.ascontiguousarray(self.eig[kinds[b]][1].T), t, DIM + b, mode, threads)
        t = t / self.lam_sum(kinds).astype(t.dtype).reshape((1, 1, 1) + (t.shape[3], t.shape[4], t.shape[5]))
        for b in (2, 1, 0):
            t = contract_mode(self.eig[kinds[b]][1], t, DIM + b, mode, threads)
        return t


def axis_runs(count, shift, n):
    """multigrid.py:97-109 -- runs of constant (left_bnd, right_bnd) kind along one axis."""
    if count < 1:
        return []
    first_left = shift == 0
    last_right = 2 * (count - 1) + shift + 2 == n
    if count == 1:
        return [(slice(0, 1), (first_left, last_right))]
    runs = [(slice(0, 1), (first_left, False))]
    if count > 2:
        runs.append((slice(1, count - 1), (False, False)))
    runs.append((slice(count - 1, count), (False, last_right)))
    return runs


def colour_order():
    """multigrid.py:27-29 -- itertools.product((0,1), repeat=3); element i = tensor axis i."""
    return tuple(itertools.product((0, 1), repeat=DIM))


def restrict(H: Hierarchy, level, r, mode="fp64", threads=1):
    """multigrid.py:112-125 -- P^T on each axis of the (2K)^3 blocks -> coarse K^3."""
    K = H.degree + 1
    p = 2 ** level // 2
    arr = np.asarray(r).reshape(H.shape(level)).astype(storage_dtype(mode), copy=False)
    w = patches(arr, (0, 0, 0), (p, p, p), 2 * K)
    Pt = np.ascontiguousarray(H.P.T)
    for b in (2, 1, 0):
        w = contract_mode(Pt, w, DIM + b, mode, threads)
    coarse = np.zeros(H.shape(level - 1), dtype=w.dtype)
    add_patches(coarse, w, (0, 0, 0), (p, p, p), K)
    return coarse.reshape(-1)


def prolongate(H: Hierarchy, coarse_level, e, mode="fp64", threads=1):
    """multigrid.py:128-143 -- exact embedding P on each axis, K^3 -> (2K)^3."""
    K = H.degree + 1
    nc = 2 ** coarse_level
    arr = np.asarray(e).reshape(H.shape(coarse_level)).astype(storage_dtype(mode), copy=False)
    w = patches(arr, (0, 0, 0), (nc, nc, nc), K)
    P = np.ascontiguousarray(H.P)
    for b in (2, 1, 0):
        w = contract_mode(P, w, DIM + b, mode, threads)
    fine = np.zeros(H.shape(coarse_level + 1), dtype=w.dtype)
    add_patches(fine, w, (0, 0, 0), (nc, nc, nc), 2 * K)
    return fine.reshape(-1)


class VCycle:
    """multigrid.py:146-270 -- MultigridPreconditioner restated."""

    def __init__(self, H: Hierarchy, mode="fp64", pre=1, post=1, coarse_level=1,
                 ordering=None, threads=1):
        self.H, self.mode, self.pre, self.post = H, mode, pre, post
        self.coarse_level = coarse_level
        self.ordering = ordering or colour_order()
        self.threads = threads
        self.solvers = {l: PatchInverse(H.levels[l].M_patch, H.levels[l].L_smooth) for l in H.levels}
        self._cache = {}

    def smooth(self, level, x, b, mode=None):
        """multigrid.py:172-204 -- 8 multiplicative colours, residual refreshed per colour."""
        mode = mode or self.mode
        H = self.H
        K = H.degree + 1
        n = 2 ** level
        dt = storage_dtype(mode)
        x = np.asarray(x, dtype=dt).reshape(H.shape(level)).copy()
        b = np.asarray(b, dtype=dt).reshape(-1)
        solver = self.solvers[level]
        for shift in self.ordering:
            counts = tuple(n // 2 - shift[DIM - 1 - d] for d in range(DIM))
            if min(counts) < 1:
                continue
            starts = tuple(K * shift[DIM - 1 - d] for d in range(DIM))
            r = b - apply_operator(H, level, x.reshape(-1), mode, self.threads)
            w = patches(r.reshape(H.shape(level)), starts, counts, 2 * K)
            out = np.empty_like(w)
            runs = [axis_runs(counts[d], shift[DIM - 1 - d], n) for d in range(DIM)]
            for combo in itertools.product(*runs):
                sel = tuple(s for s, _ in combo) + (slice(None),) * DIM
                out[sel] = solver.apply(w[sel], tuple(k for _, k in combo), mode, self.threads)
            add_patches(x, out, starts, counts, 2 * K)
        return x.reshape(-1)

    def _dense(self):
        if "dense" not in self._cache:
            self._cache["dense"] = materialize(self.H, self.coarse_level)
        return self._cache["dense"]

    def _factor(self, mode):
        """multigrid.py:215-228 -- LU of the coarse matrix, operands demoted per mode."""
        if mode not in self._cache:
            A = self._dense()
            if mode == "fp64":
                Ad = A
            elif mode == "fp32":
                Ad = A.astype(np.float32)
            elif mode == "fp16":
                Ad = demote16(A.astype(np.float32))
            else:
                main, resid = ec_split(A.astype(np.float32))
                Ad = main + resid / EC_SCALE
            self._cache[mode] = scipy.linalg.lu_factor(Ad)
        return self._cache[mode]

    def coarse_solve(self, b, mode=None):
        """multigrid.py:230-239."""
        mode = mode or self.mode
        fac = self._factor(mode)
        bs = np.asarray(b, dtype=storage_dtype(mode))
        if mode == "fp16":
            bs = demote16(bs)
        return scipy.linalg.lu_solve(fac, bs.astype(fac[0].dtype)).astype(storage_dtype(mode))

    def _cycle(self, level, x, b):
        """multigrid.py:243-255 -- recursive V-cycle in storage precision."""
        if level == self.coarse_level:
            return self.coarse_solve(b)
        for _ in range(self.pre):
            x = self.smooth(level, x, b)
        r = b - apply_operator(self.H, level, x, self.mode, self.threads)
        rc = restrict(self.H, level, r, self.mode, self.threads)
        e = self._cycle(level - 1, np.zeros_like(rc), rc)
        x = x + prolongate(self.H, level - 1, e, self.mode, self.threads)
        for _ in range(self.post):
            x = self.smooth(level, x, b)
        return x

    def vcycle(self, x, b, level=None):
        """multigrid.py:257-266 -- fp64 in/out; storage conversion only here."""
        level = self.H.max_level if level is None else level
        dt = storage_dtype(self.mode)
        return self._cycle(level, np.asarray(x, dt).copy(), np.asarray(b, dt)).astype(np.float64)

    def apply(self, b, level=None):
        """multigrid.py:268-270."""
        return self.vcycle(np.zeros(np.asarray(b).size), b, level)


# ---------------------------------------------------------------- krylov


@dataclass
class Report:
    """krylov.py:21-42 (the fields the parity tests read)."""

    iterations: int
    residual_history: list
    final_relative_residual: float
    converged: bool
    breakdown: bool = False


def gmres_driver(apply_A, apply_M, b, tol=1e-8, maxit=100, flexible=True):
    """krylov.py:49-137 -- right-preconditioned (F)GMRES, MGS + one selective re-orth."""
    b = np.asarray(b, dtype=np.float64)
    beta = float(np.linalg.norm(b))
    if beta == 0.0:
        return np.zeros(b.size), Report(0, [0.0], 0.0, True)
    V = [b / beta]
    Z = []
    H = np.zeros((maxit + 1, maxit))
    cs, sn = np.zeros(maxit), np.zeros(maxit)
    g = np.zeros(maxit + 1)
    g[0] = beta
    hist = [beta]
    breakdown = False
    j = -1
    for j in range(maxit):
        z = apply_M(V[j])
        if flexible:
            Z.append(np.asarray(z, dtype=np.float64))
        w = np.asarray(apply_A(z), dtype=np.float64)
        nb = float(np.linalg.norm(w))
        for i in range(j + 1):
            H[i, j] = V[i] @ w
            w = w - H[i, j] * V[i]
        hn = float(np.linalg.norm(w))
        if hn < nb / np.sqrt(2.0):
            for i in range(j + 1):
                c = V[i] @ w
                H[i, j] += c
                w = w - c * V[i]
            hn = float(np.linalg.norm(w))
        H[j + 1, j] = hn
        for i in range(j):
            hij = cs[i] * H[i, j] + sn[i] * H[i + 1, j]
            H[i + 1, j] = -sn[i] * H[i, j] + cs[i] * H[i + 1, j]
            H[i, j] = hij
        den = np.hypot(H[j, j], H[j + 1, j])
        cs[j] = H[j, j] / den if den else 1.0
        sn[j] = H[j + 1, j] / den if den else 0.0
        H[j, j] = den
        H[j + 1, j] = 0.0
        g[j + 1] = -sn[j] * g[j]
        g[j] = cs[j] * g[j]
        hist.append(abs(g[j + 1]))
        if abs(g[j + 1]) / beta <= tol:
            break
        if hn <= 1e-14 * max(nb, 1.0):
            breakdown = True
            break
        V.append(w / hn)
    m = j + 1
    y = np.zeros(m)
    for i in range(m - 1, -1, -1):
        y[i] = (g[i] - H[i, i + 1:m] @ y[i + 1:m]) / H[i, i]
    if flexible:
        x = np.zeros(b.size)
        for i in range(m):
            x += y[i] * Z[i]
    else:
        comb = np.zeros(b.size)
        for i in range(m):
            comb += y[i] * V[i]
        x = np.asarray(apply_M(comb), dtype=np.float64)
    rel = hist[-1] / beta
    return x, Report(m, hist, rel, bool(rel <= tol), breakdown)


# ------------------------------------------------- rhs / errors / solve


def _cells(arr, n, q):
    w = arr.reshape(n, q, n, q, n, q)
    return np.ascontiguousarray(w.transpose(0, 2, 4, 1, 3, 5))


def _uncells(w, n, q):
    return w.transpose(0, 3, 1, 4, 2, 5).reshape(n * q, n * q, n * q)


def _axis_pts(n, h, pts):
    return ((np.arange(n)[:, None] + pts[None, :]) * h).ravel()


def sine_exact(x, y, z):
    """discretization.py:504-531 -- manufactured solution, f = 3 pi^2 u."""
    return np.sin(np.pi * x) * np.sin(np.pi * y) * np.sin(np.pi * z)


def sine_rhs(x, y, z):
    return 3.0 * np.pi ** 2 * sine_exact(x, y, z)


def sine_grad(x, y, z):
    pi = np.pi
    return (pi * np.cos(pi * x) * np.sin(pi * y) * np.sin(pi * z),
            pi * np.sin(pi * x) * np.cos(pi * y) * np.sin(pi * z),
            pi * np.sin(pi * x) * np.sin(pi * y) * np.cos(pi * z))


def assemble_rhs(H: Hierarchy, level, f):
    """discretization.py:317-345 -- volume load vector (g = None, as run_solve uses)."""
    k = H.degree
    n, h = 2 ** level, 2.0 ** -level
    q = k + 2
    pts, wts = gauss_points_weights(q)
    S = lagrange_table(lobatto_nodes(k), pts)
    ax = _axis_pts(n, h, pts)
    Z, Y, X = np.meshgrid(ax, ax, ax, indexing="ij")
    vals = np.asarray(f(X, Y, Z), dtype=np.float64) * np.ones((n * q,) * 3)
    wa = np.tile(wts, n) * h
    vals = vals * wa[:, None, None] * wa[None, :, None] * wa[None, None, :]
    w = _cells(vals, n, q)
    for b in (2, 1, 0):
        w = contract(np.ascontiguousarray(S.T), w, DIM + b)
    return _uncells(w, n, k + 1).reshape(-1)


def _qvalues(H, level, u, pts, deriv_axis=None):
    """discretization.py:405-419."""
    k = H.degree
    n, h = 2 ** level, 2.0 ** -level
    nodes = lobatto_nodes(k)
    S = lagrange_table(nodes, pts)
    D = lagrange_slope_table(nodes, pts) / h
    w = _cells(np.asarray(u, np.float64).reshape(H.shape(level)), n, k + 1)
    for b in (2, 1, 0):
        w = contract(np.ascontiguousarray(D if deriv_axis == 2 - b else S), w, DIM + b)
    return _uncells(w, n, len(pts))


def l2_error(H, level, u, exact):
    """discretization.py:431-441."""
    q = H.degree + 3
    pts, wts = gauss_points_weights(q)
    n, h = 2 ** level, 2.0 ** -level
    ax = _axis_pts(n, h, pts)
    Z, Y, X = np.meshgrid(ax, ax, ax, indexing="ij")
    diff = _qvalues(H, level, u, pts) - exact(X, Y, Z)
    wa = np.tile(wts, n) * h
    W = wa[:, None, None] * wa[None, :, None] * wa[None, None, :]
    return float(math.sqrt(np.sum(W * diff ** 2)))


def h1_error(H, level, u, grad):
    """discretization.py:444-459."""
    q = H.degree + 3
    pts, wts = gauss_points_weights(q)
    n, h = 2 ** level, 2.0 ** -level
    ax = _axis_pts(n, h, pts)
    Z, Y, X = np.meshgrid(ax, ax, ax, indexing="ij")
    wa = np.tile(wts, n) * h
    W = wa[:, None, None] * wa[None, :, None] * wa[None, None, :]
    g = grad(X, Y, Z)
    tot = 0.0
    for a in range(DIM):
        c = _qvalues(H, level, u, pts, deriv_axis=a) - g[a]
        tot += float(np.sum(W * c ** 2))
    return math.sqrt(tot)


def run_solve(degree, level, mode="fp64", solver="fgmres", tol=1e-8, maxit=100,
              coarse_level=1, pre=1, post=1, H=None, threads=1):
    """experiments.py:57-103 -- sine problem, V-cycle preconditioned (F)GMRES."""
    H = H or Hierarchy(level, degree)
    b = assemble_rhs(H, level, sine_rhs)
    mg = VCycle(H, mode=mode, pre=pre, post=post, coarse_level=coarse_level, threads=threads)
    x, rep = gmres_driver(lambda v: apply_operator(H, level, v, "fp64", threads),
                          lambda v: mg.apply(v, level), b, tol=tol, maxit=maxit,
                          flexible=(solver == "fgmres"))
    return x, rep, l2_error(H, level, x, sine_exact), h1_error(H, level, x, sine_grad)


def default_threads():
    return max(1, len(os.sched_getaffinity(0)))
