"""Cell-local evaluation of the reference vmult for spot checks at sizes the
full oracle cannot reach (TEST INFRASTRUCTURE).

The reference operator (`src/discretization.py:216-266`, restated by
``oracle.port.apply_operator``) is, on the uniform cube mesh, the Kronecker sum

    A = L1 (x) M1 (x) M1 + M1 (x) L1 (x) M1 + M1 (x) M1 (x) L1

of the 1-D global matrices built from the same per-level pieces the reference
uses: ``L1`` = blockdiag over patches of ``L_tile`` + ``B_left`` on the first
patch + ``B_right`` on the last + ``F_cross`` on every shifted patch pair
(`:244-264`), ``M1`` = blockdiag(``M_cell``).  Row block c of ``L1`` only touches
cells c-1..c+1, so ``v`` on one cell needs ``u`` on that cell and its six face
neighbours.  ``tests/test_local_stencil.py`` pins this evaluator to
``oracle.port.apply_operator`` on whole meshes; the GPU tests then use it on
sampled cells of the 1e9-DoF bench meshes.
"""
from __future__ import annotations

import numpy as np

from oracle import port


def global_1d(k: int, level: int):
    """(L1, M1) as dense A x A arrays (A = 2^level (k+1)) from the port's level pieces."""
    lm = port.level_matrices(k, level)
    K = k + 1
    n = 2 ** level
    A, B, p = n * K, 2 * K, n // 2
    L1 = np.zeros((A, A))
    M1 = np.zeros((A, A))
    for c in range(n):
        M1[c * K:(c + 1) * K, c * K:(c + 1) * K] = lm.M_cell
    for q in range(p):
        s = slice(q * B, (q + 1) * B)
        L1[s, s] += lm.L_tile
    L1[0:B, 0:B] += lm.B_left
    L1[A - B:A, A - B:A] += lm.B_right
    for q in range(p - 1):
        s = slice(q * B + K, q * B + K + B)
        L1[s, s] += lm.F_cross
    return L1, M1


class LocalVmult:
    """v restricted to chosen cells, from u gathered on the cell's 3-cell windows."""

    def __init__(self, k: int, level: int):
        self.k, self.level = k, level
        self.K = k + 1
        self.n = 2 ** level
        self.L1, self.M1 = global_1d(k, level)

    def window(self, c: int):
        """cells c-1..c+1 clipped to the mesh -> (first cell, count)."""
        lo, hi = max(c - 1, 0), min(c + 1, self.n - 1)
        return lo, hi - lo + 1

    def block_index(self, cz: int, cy: int, cx: int):
        """flat indices of the clipped 3x3x3-cell block around (cz, cy, cx)."""
        K, A = self.K, self.n * self.K
        (z0, nz), (y0, ny), (x0, nx) = self.window(cz), self.window(cy), self.window(cx)
        z = np.arange(z0 * K, (z0 + nz) * K)
        y = np.arange(y0 * K, (y0 + ny) * K)
        x = np.arange(x0 * K, (x0 + nx) * K)
        return (z[:, None, None] * A + y[None, :, None]) * A + x[None, None, :]

    def apply_cell(self, block: np.ndarray, cz: int, cy: int, cx: int) -> np.ndarray:
        """v on cell (cz, cy, cx) (K^3, numpy order z, y, x) from the u block of block_index."""
        K = self.K
        (z0, nz), (y0, ny), (x0, nx) = self.window(cz), self.window(cy), self.window(cx)
        rz = slice(cz * K, (cz + 1) * K)
        ry = slice(cy * K, (cy + 1) * K)
        rx = slice(cx * K, (cx + 1) * K)
        cz_ = slice(z0 * K, (z0 + nz) * K)
        cy_ = slice(y0 * K, (y0 + ny) * K)
        cx_ = slice(x0 * K, (x0 + nx) * K)
        oz, oy, ox = (cz - z0) * K, (cy - y0) * K, (cx - x0) * K
        u = np.asarray(block, dtype=np.float64)
        L, M = self.L1, self.M1
        # own-cell sub-blocks along the M directions
        uz = u[:, oy:oy + K, ox:ox + K]  # z window, own y, own x
        uy = u[oz:oz + K, :, ox:ox + K]
        ux = u[oz:oz + K, oy:oy + K, :]
        v = np.einsum("ab,cd,ef,bdf->ace", L[rz, cz_], M[ry, ry], M[rx, rx], uz)
        v += np.einsum("ab,cd,ef,bdf->ace", M[rz, rz], L[ry, cy_], M[rx, rx], uy)
        v += np.einsum("ab,cd,ef,bdf->ace", M[rz, rz], M[ry, ry], L[rx, cx_], ux)
        return v

    def apply_full(self, u: np.ndarray) -> np.ndarray:
        """every cell (small meshes only) -- used to pin the evaluator to the oracle."""
        K, n, A = self.K, self.n, self.n * self.K
        uf = np.asarray(u, dtype=np.float64).reshape(-1)
        v = np.zeros((A, A, A))
        for cz in range(n):
            for cy in range(n):
                for cx in range(n):
                    blk = uf[self.block_index(cz, cy, cx)]
                    v[cz * K:(cz + 1) * K, cy * K:(cy + 1) * K, cx * K:(cx + 1) * K] = \
                        self.apply_cell(blk, cz, cy, cx)
        return v.reshape(-1)


def sample_cells(n: int, count: int, seed: int = 0, band: int = 16):
    """Random cells plus every structurally special one: the 8 corners, edge and face
    cells, and cells on both sides of tile-band / tile-pair boundaries (multiples of
    ``band`` and of 2 cells) -- the places where the kernels change code path."""
    rng = np.random.default_rng(seed)
    cells = {tuple(int(c) for c in rng.integers(0, n, 3)) for _ in range(count)}
    edge = [0, 1, n - 2, n - 1]
    for z in edge:
        for y in edge:
            for x in edge:
                cells.add((z, y, x))
    specials = sorted({c for b in range(band, n, band) for c in (b - 1, b)} | {n // 2 - 1, n // 2})
    for s in specials:
        r = tuple(int(c) for c in rng.integers(0, n, 3))
        cells.add((s, r[1], r[2]))
        cells.add((r[0], s, r[2]))
        cells.add((r[0], r[1], s))
        cells.add((s, s, r[2]))
    return sorted(cells)
