// FP64 tensor-core (DMMA, mma.sync.m8n8k4.f64) tile toolkit for Q7 (K = 8):
// one 2x2x2-cell tile = 16^3 dofs per CTA, 8 warps, two CTAs per SM.
//
// Every line contraction of the tile is a small GEMM  Y[line][out] = X[line][k] Op^T[k][out]
// on 8-line groups: A = data (8 lines x 4 k) from shared memory, B = operator
// fragment in registers, C/D = 8 lines x 8 outputs in registers.  The 16x16
// line operators are the patch matrices themselves:
//   mass       M_patch = blockdiag(M_cell, M_cell)      (4 DMMA per group)
//   stiffness  L_smooth[kind]  (principal submatrix of the global 1-D operator,
//              Nitsche rows at domain-boundary ends)    (8 DMMA per group)
// and the coupling to the face neighbours outside the tile is the rank-2 U/U^T
// update from the neighbour's face traces (alpha, beta), added to the C
// fragment.  Schedule (cell-wise sum factorisation):
//   prologue: tile -> smem (cp.async), neighbour face traces straight from
//             L2/HBM (all loads in flight at once), tangential masses of the
//             y/z trace planes on DMMA
//   x:  a = Mx u,   b = Lx u (+ x halo)             -- warp owns z planes, in place
//   y:  c = My a,  dd = Ly a (+ y halo) + My b      -- same warp, same planes, in place
//   z:  v = Lz c (+ z halo) + Mz dd                 -- warp owns y rows, lines along x
// Shared-memory layouts are XOR swizzles (the paper's conflict-free idea,
// P:319), chosen per stage and then A/B-measured (profiles/r02_vmult_fp64.md):
//   U layout : z*256 + y*16 + 2((x/2) ^ (y&7)) + (x&1)   (the TMA 128-byte swizzle; see idxU)
//   A layout : z*256 + y*16 + (x ^ {0,8,4,12}[y&3])
//   C layout : z*256 + y*16 + (x ^ 4(((y>>1)+z)&3))
#pragma once
#include "sf_common.cuh"
#include "sf_tile.cuh"

namespace sf {
namespace dm {

constexpr int K = 8, B = 16, PLANE = 256, VOL = 4096;
constexpr int TRP = 320;   // one trace plane: 16 rows x pitch 20 (pitch = 4 mod 16)
constexpr int TRW = 20;
constexpr int kThreads = 256;
constexpr size_t kSmemTile = sizeof(double) * (2 * VOL + 12 * TRP + 4 * 8 * 32);

// U layout = the TMA 128-byte swizzle of a 16 x 16 x 16 fp64 box: 128-byte rows (z, y), 16-byte chunk x / 2
// XORed with the row index mod 8 -- conflict-free for the x stage's A-fragment loads, and what
// cp.async.bulk.tensor writes with CU_TENSOR_MAP_SWIZZLE_128B (the FP64 vmult loads its tile that way)
// (Q7 2-cell tiles; the 16-point line tiles of Q3 / Q1 keep the 32-byte XOR x ^ 4(y mod 4), which measured 1.3 %
// faster for them: profiles/r02_vmult_fp64.md)
template <int KK = 8>
__device__ __forceinline__ int idxU(int z, int y, int x) {
  if constexpr (KK == 8) return z * PLANE + y * 16 + ((((x >> 1) ^ (y & 7)) << 1) | (x & 1));
  else return z * PLANE + y * 16 + (x ^ ((y & 3) << 2));
}
__device__ __forceinline__ int swA(int y) { return ((y & 1) << 3) | ((y & 2) << 1); }  // {0,8,4,12}[y&3]
__device__ __forceinline__ int idxA(int z, int y, int x) { return z * PLANE + y * 16 + (x ^ swA(y)); }
__device__ __forceinline__ int idxC(int z, int y, int x) {
  return z * PLANE + y * 16 + (x ^ ((((y >> 1) + z) & 3) << 2));
}
// smoother layouts: T = C with the roles of y and z swapped; G = the U swizzle (was a Gray-code swizzle of
// 32-byte groups; measured 0.4 % slower per smoothing step)
__device__ __forceinline__ int idxT(int z, int y, int x) {
  return z * PLANE + y * 16 + (x ^ ((((z >> 1) + y) & 3) << 2));
}
__device__ __forceinline__ int idxG(int z, int y, int x) {
  return z * PLANE + y * 16 + ((((x >> 1) ^ (y & 7)) << 1) | (x & 1));
}

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  // not volatile: no side effects, so ptxas may interleave independent DMMAs of several groups
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async8(void* smem, const void* gmem) {
  unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;\n" ::); }

// Storage-precision demotion of a contraction output (FP32 mode on the FP64 tensor pipe: every
// stage result is rounded to fp32 where the reference stores it in the mode's dtype,
// precision.py:206-230); identity for fp64 storage.
template <class S>
__device__ __forceinline__ double rd(double x) {
  if constexpr (sizeof(S) == 4) return (double)__double2float_rn(x);
  else return x;
}

// Operator fragments held by one lane.
struct Frags {
  double m[2];     // M_cell[lane>>2][4*kc + (lane&3)], kc = 0,1 (both cells)
  double l[2][4];  // L[8nb + (lane>>2)][4kc + (lane&3)]
};

// acc[nb][2]: outputs 8nb + 2(lane&3) + {0,1} of line (lane>>2)
// k-chunk outer, output block inner: consecutive DMMAs are independent
__device__ __forceinline__ void mass_group(const Frags& f, const double* a, double (*acc)[2]) {
#pragma unroll
  for (int kc = 0; kc < 2; ++kc)
#pragma unroll
    for (int nb = 0; nb < 2; ++nb) dmma(acc[nb][0], acc[nb][1], a[2 * nb + kc], f.m[kc]);
}
__device__ __forceinline__ void stiff_group(const Frags& f, const double* a, double (*acc)[2]) {
#pragma unroll
  for (int kc = 0; kc < 4; ++kc)
#pragma unroll
    for (int nb = 0; nb < 2; ++nb) dmma(acc[nb][0], acc[nb][1], a[kc], f.l[nb][kc]);
}

// Shared state of one tile (pointers into the CTA's shared memory + geometry).
struct Tile {
  double* sU;   // u -> a -> c   (VOL)
  double* sB;   // b -> dd       (VOL)
  double* tr;   // 12 trace planes: (face*2 + {alpha,beta}) * TRP + p*TRW + q
  const double* sLf;  // L_smooth fragments [kind][nb*4+kc][lane] (shared or global)
  int cx, cy, cz;
  long long sy, sz;
  unsigned nbm;             // bit 2*axis+hi: face neighbour present (inside the array or ghost)
  int kind[3];
  int r, k4, c2, lane, warp;
  int b0;  // banded launch: first tile row of the band
  int skip[3];  // leading points per axis already written by the previous tile (clamped last line)
};

// 0: neighbour inside the local array, 1: ghost (z only), 2: domain boundary.
// A tile line spans 16 points = 16 / K cells (K = 8: 2 cells, K = 4: 4, K = 2: 8).
template <int K = 8>
__device__ __forceinline__ int face_src(const Geom& g, int axis, int hi, int c0) {
  int n = axis == 0 ? g.nx : (axis == 1 ? g.ny : g.nz);
  int c = hi ? c0 + 16 / K : c0 - 1;
  if (c >= 0 && c < n) return 0;
  if (hi ? g.bnd_hi[axis] : g.bnd_lo[axis]) return 2;
  return 1;
}

// Shifted Q7 colours leave the first / last cell layer of every shifted axis uncovered; the ping-pong copy
// keeps x_old there.  Fused into the colour kernels: the CTA of a tile at the start (end) of a shifted axis
// also copies the uncovered cells of its box extended by that layer (the extended boxes partition the grid,
// so every uncovered cell is copied exactly once), 16-byte chunks, threads strided.  S = storage type.
template <typename S, int NT>
__device__ __forceinline__ void copy_uncovered_ext(const Geom& g, int cx, int cy, int cz, const S* __restrict__ xo,
                                                   S* __restrict__ xn) {
  const int c[3] = {cx, cy, cz}, n[3] = {g.nx, g.ny, g.nz}, sh[3] = {g.tx0 & 1, g.ty0 & 1, g.tz0 & 1};
  int lo[3], ext[3];
  bool any = false;
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    lo[a] = c[a];
    ext[a] = 2;
    if (sh[a] && c[a] == 1) { lo[a] = 0; ++ext[a]; any = true; }
    if (sh[a] && c[a] + 2 == n[a] - 1) { ++ext[a]; any = true; }
  }
  if (!any) return;
  constexpr int VPR = 8 * (int)sizeof(S) / 16;  // 16-byte chunks per 8-point row
  const long long sy = (long long)g.nx * 8, sz = sy * g.ny * 8;
  const int total = ext[0] * ext[1] * ext[2] * 64 * VPR;
  for (int i = threadIdx.x; i < total; i += NT) {
    const int ch = i % VPR, r = i / VPR, row = r & 63, cell = r >> 6;
    const int X = lo[0] + cell % ext[0], Y = lo[1] + (cell / ext[0]) % ext[1], Z = lo[2] + cell / (ext[0] * ext[1]);
    if (X >= cx && X <= cx + 1 && Y >= cy && Y <= cy + 1 && Z >= cz && Z <= cz + 1) continue;  // this tile
    const long long o = (long long)(Z * 8 + (row >> 3)) * sz + (long long)(Y * 8 + (row & 7)) * sy + X * 8 +
                        ch * (16 / (int)sizeof(S));
    *reinterpret_cast<uint4*>(xn + o) = __ldg(reinterpret_cast<const uint4*>(xo + o));
  }
}

// Banded 3-D launch (replaces per-thread integer divisions of a linear tile id): grid =
// (ntx, band rows `by`, ntz * nbands [* batch]); launch order x, y-in-band, z, band -- the
// L2-aware order of tile_coords<K>.  Returns false for the idle CTAs of a partial last band.
struct Band {
  int by, zb;  // tile rows per band; ntz * nbands (z extent of one batch vector)
};
__host__ __forceinline__ Band make_band(const Geom& g) {
  int by = band_tiles<K>() / g.ntx;
  by = by < 1 ? 1 : (by > g.nty ? g.nty : by);
  const int nb = (g.nty + by - 1) / by;
  return Band{by, g.ntz * nb};
}
__device__ __forceinline__ bool band_tile(const Geom& g, const Band& bd, int& tx, int& ty, int& tz, int& batch) {
  int zz = blockIdx.z;
  batch = 0;
  if (gridDim.z > (unsigned)bd.zb) {
    batch = zz / bd.zb;
    zz -= batch * bd.zb;
  }
  const int band = zz / g.ntz;
  tz = zz - band * g.ntz;
  ty = band * bd.by + blockIdx.y;
  tx = blockIdx.x;
  return ty < g.nty;
}

template <int K = 8>
__device__ __forceinline__ void tile_fields(Tile& T, const Geom& g, int tx, int ty, int tz);


template <int K>
__device__ __forceinline__ void tile_fields(Tile& T, const Geom& g, int tx, int ty, int tz) {
  constexpr int CPL = 16 / K;
  T.cx = g.tx0 + CPL * tx;
  T.cy = g.ty0 + CPL * ty;
  T.cz = g.tz0 + CPL * tz;
  T.skip[0] = T.skip[1] = T.skip[2] = 0;
  if constexpr (K < 8) {  // shifted colour (odd offset): the last line ends at cell n-2 (overlaps its neighbour)
    const int ux = T.cx, uy = T.cy, uz = T.cz;
    if (g.tx0 & 1) T.cx = min(T.cx, g.nx - CPL - g.tx0);
    if (g.ty0 & 1) T.cy = min(T.cy, g.ny - CPL - g.ty0);
    if (g.tz0 & 1) T.cz = min(T.cz, g.nz - CPL - g.tz0);
    // the overlapped patches were written by the previous line, whose position along the line gave
    // them different (rounding-level) arithmetic: only one writer, so results are deterministic
    T.skip[0] = (ux - T.cx) * K;
    T.skip[1] = (uy - T.cy) * K;
    T.skip[2] = (uz - T.cz) * K;
  }
  T.sy = (long long)g.nx * K;
  T.sz = T.sy * (long long)g.ny * K;
  const int c0[3] = {T.cx, T.cy, T.cz};
  T.nbm = 0;
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    if (face_src<K>(g, a, 0, c0[a]) != 2) T.nbm |= 1u << (2 * a);
    if (face_src<K>(g, a, 1, c0[a]) != 2) T.nbm |= 1u << (2 * a + 1);
  }
#pragma unroll
  for (int a = 0; a < 3; ++a) {  // kind of the 16-point line: 2 * (domain boundary at its start) + (at its end)
    const int n = a == 0 ? g.nx : (a == 1 ? g.ny : g.nz);
    const int lb = (c0[a] == 0 && g.bnd_lo[a]) ? 1 : 0;
    const int rb = (c0[a] + CPL == n && g.bnd_hi[a]) ? 1 : 0;
    T.kind[a] = 2 * lb + rb;
  }
  T.lane = threadIdx.x & 31;
  T.warp = threadIdx.x >> 5;
  T.r = T.lane >> 2;
  T.k4 = T.lane & 3;
  T.c2 = 2 * T.k4;
}

// banded-grid variant of tile_setup; `batch` = vector index of a batched launch
template <int K = 8>
__device__ __forceinline__ bool tile_setup_band(Tile& T, double* smem, const Geom& g, const Band& bd, int& batch) {
  T.sU = smem;
  T.sB = smem + VOL;
  T.tr = T.sB + VOL;
  T.sLf = T.tr + 12 * TRP;
  int tx, ty, tz;
  if (!band_tile(g, bd, tx, ty, tz, batch)) return false;
  tile_fields<K>(T, g, tx, ty, tz);
  T.b0 = ty - blockIdx.y;  // first tile row of this band
  return true;
}

// L2 prefetch of the u rows of the tile two rows ahead in launch order (~2 ntx CTAs later):
// (tx, ty + 2) inside the band, else the wrapped row of the next z layer.
template <int K = 8, class S = double>
__device__ __forceinline__ void prefetch_ahead_l2(const Geom& g, const Band& bd, const Tile& T,
                                                  const S* __restrict__ u) {
  constexpr int CPL = 16 / K;
  const int ty = (T.cy - g.ty0) / CPL, tz = (T.cz - g.tz0) / CPL;
  const int b0 = T.b0;
  const int bh = min(bd.by, g.nty - b0);
  int ny = ty + 2, nz = tz;
  if (ny >= b0 + bh) {
    ny -= bh;
    if (++nz >= g.ntz) return;
  }
  if (ny < b0 || threadIdx.x >= 256) return;
  const int y = threadIdx.x & 15, z = threadIdx.x >> 4;
  const S* p = u + (long long)((g.tz0 + CPL * nz) * K + z) * T.sz + (long long)((g.ty0 + CPL * ny) * K + y) * T.sy +
                    T.cx * K;
  asm volatile("prefetch.global.L2 [%0];\n" ::"l"(p));
}

// L2 prefetch of this tile's rows of a second input (the right-hand side b the colour /
// restriction kernels read in their z stage): DRAM latency paid during the prologue, not there.
template <int K = 8, class S = double>
__device__ __forceinline__ void prefetch_tile_rows_l2(const Tile& T, const S* __restrict__ p0) {
  if (threadIdx.x >= 256) return;
  const int y = threadIdx.x & 15, z = threadIdx.x >> 4;
  const S* p = p0 + (long long)(T.cz * K + z) * T.sz + (long long)(T.cy * K + y) * T.sy + T.cx * K;
  asm volatile("prefetch.global.L2 [%0];\n" ::"l"(p));
}





__device__ __forceinline__ void load_l(const Tile& T, Frags& f, int kind) {
#pragma unroll
  for (int nb = 0; nb < 2; ++nb)
#pragma unroll
    for (int kc = 0; kc < 4; ++kc) f.l[nb][kc] = T.sLf[(kind * 8 + nb * 4 + kc) * 32 + T.lane];
}


// rank-2 halo update of a stiffness fragment (lo neighbour -> cell 0, hi -> cell 1)
struct Halo {
  double ur[2], uc[2];
  __device__ __forceinline__ void apply(const Tile& T, double (*acc)[2], int axis, int t) const {
    if ((T.nbm >> (2 * axis)) & 1) {
      const double* pl = T.tr + (2 * axis) * 2 * TRP;
      const double alo = pl[t], blo = pl[TRP + t];
      acc[0][0] = fma(ur[0], alo, acc[0][0]);
      acc[0][1] = fma(ur[1], alo, acc[0][1]);
      if (T.c2 == 0) acc[0][0] += blo;
    }
    if ((T.nbm >> (2 * axis + 1)) & 1) {
      const double* pl = T.tr + (2 * axis + 1) * 2 * TRP;
      const double ahi = pl[t], bhi = pl[TRP + t];
      acc[1][0] = fma(uc[0], ahi, acc[1][0]);
      acc[1][1] = fma(uc[1], ahi, acc[1][1]);
      if (T.c2 + 1 == K - 1) acc[1][1] += bhi;
    }
  }
};

// x and y stages on the warp's two z planes (in place: U <- a <- c, B <- b <- dd)
template <class S = double, int KK = 8>
__device__ __forceinline__ void xy_stages(const Tile& T, Frags& f, const Halo& h) {
  for (int zz = 0; zz < 2; ++zz) {
    const int z = 2 * T.warp + zz;
    load_l(T, f, T.kind[0]);
    double ra[2][2][2], rb[2][2][2];
#pragma unroll
    for (int g8 = 0; g8 < 2; ++g8) {
      const int y = 8 * g8 + T.r;
      double a[4];
#pragma unroll
      for (int kc = 0; kc < 4; ++kc) a[kc] = T.sU[idxU<KK>(z, y, 4 * kc + T.k4)];
#pragma unroll
      for (int nb = 0; nb < 2; ++nb) ra[g8][nb][0] = ra[g8][nb][1] = rb[g8][nb][0] = rb[g8][nb][1] = 0.0;
      h.apply(T, rb[g8], 0, z * TRW + y);  // halo first: the DFMAs need no DMMA result
      mass_group(f, a, ra[g8]);
      stiff_group(f, a, rb[g8]);
    }
    __syncwarp();
#pragma unroll
    for (int g8 = 0; g8 < 2; ++g8) {
      const int y = 8 * g8 + T.r;
#pragma unroll
      for (int nb = 0; nb < 2; ++nb) {
        const int i = idxA(z, y, 8 * nb + T.c2);
        *reinterpret_cast<double2*>(&T.sU[i]) = make_double2(rd<S>(ra[g8][nb][0]), rd<S>(ra[g8][nb][1]));
        *reinterpret_cast<double2*>(&T.sB[i]) = make_double2(rd<S>(rb[g8][nb][0]), rd<S>(rb[g8][nb][1]));
      }
    }
    __syncwarp();
    load_l(T, f, T.kind[1]);
#pragma unroll
    for (int g8 = 0; g8 < 2; ++g8) {
      const int x = 8 * g8 + T.r;
      double a[4], b[4];
#pragma unroll
      for (int kc = 0; kc < 4; ++kc) {
        a[kc] = T.sU[idxA(z, 4 * kc + T.k4, x)];
        b[kc] = T.sB[idxA(z, 4 * kc + T.k4, x)];
      }
#pragma unroll
      for (int nb = 0; nb < 2; ++nb) ra[g8][nb][0] = ra[g8][nb][1] = rb[g8][nb][0] = rb[g8][nb][1] = 0.0;
      h.apply(T, rb[g8], 1, z * TRW + x);  // (y halo)
      mass_group(f, a, ra[g8]);   // c = My a
      stiff_group(f, a, rb[g8]);  // d = Ly a
      mass_group(f, b, rb[g8]);   // dd = d + My b
    }
    __syncwarp();
#pragma unroll
    for (int g8 = 0; g8 < 2; ++g8) {
      const int x = 8 * g8 + T.r;
#pragma unroll
      for (int nb = 0; nb < 2; ++nb)
#pragma unroll
        for (int i = 0; i < 2; ++i) {
          const int j = idxC(z, 8 * nb + T.c2 + i, x);
          T.sU[j] = rd<S>(ra[g8][nb][i]);
          T.sB[j] = rd<S>(rb[g8][nb][i]);
        }
    }
    __syncwarp();
  }
}

// z stage for one group: lines x = x0 + r at row y; acc = (A u) C fragment [line][z]
__device__ __forceinline__ void z_group(const Tile& T, const Frags& f, const Halo& h, int y, int x0,
                                       double (*acc)[2]) {
  const int x = x0 + T.r;
  double cc[4], dd[4];
#pragma unroll
  for (int kc = 0; kc < 4; ++kc) {
    cc[kc] = T.sU[idxC(4 * kc + T.k4, y, x)];
    dd[kc] = T.sB[idxC(4 * kc + T.k4, y, x)];
  }
  acc[0][0] = acc[0][1] = acc[1][0] = acc[1][1] = 0.0;
  h.apply(T, acc, 2, y * TRW + x);  // (z halo)
  stiff_group(f, cc, acc);
  mass_group(f, dd, acc);
}

// Per-lane operator fragments: mass B fragment of the 16-point line operator blockdiag(M_cell)
// (chunk kc of the block: nonzero where output row r and input 4kc + k4 fall in one cell), and
// the halo coefficients of the line's first / last cell (zero for lanes whose outputs lie in
// another cell, so Halo::apply needs no cell test).
template <int K = 8, class OpT>
__device__ __forceinline__ void init_frags(const Tile& T, const OpT& op, Frags& f, Halo& h) {
#pragma unroll
  for (int kc = 0; kc < 2; ++kc) {
    const int kk = 4 * kc + T.k4;
    f.m[kc] = (T.r / K == kk / K) ? op.M[T.r % K][kk % K].h : 0.0;
  }
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    const int n0 = T.c2 + i;          // output within the first 8-block (cell 0 when n0 < K)
    const int n1 = T.c2 + i - (8 - K);  // output index within the last cell (second 8-block)
    h.ur[i] = n0 < K ? op.urow[n0].h : 0.0;
    h.uc[i] = n1 >= 0 ? op.ucol[n1].h : 0.0;
  }
}


// ---------------------------------------------------------------------------
// Prologue of the vmult / colour / residual-restriction kernels (profiles/r01_vmult_fp64.md).

// tangential mass along q (Mx) on trace planes [first, first + 4): one 8-row group per warp task
__device__ __forceinline__ void plane_mass_rows(const Tile& T, const Frags& f, int first) {
  for (int task = T.warp; task < 8; task += kThreads / 32) {
    const int plane = first + (task >> 1);
    if (!((T.nbm >> (plane >> 1)) & 1)) continue;
    double* P = T.tr + plane * TRP + (task & 1) * 8 * TRW;
    double a[4];
#pragma unroll
    for (int kc = 0; kc < 4; ++kc) a[kc] = P[T.r * TRW + 4 * kc + T.k4];
    double acc[2][2] = {{0.0, 0.0}, {0.0, 0.0}};
    mass_group(f, a, acc);
    __syncwarp();
#pragma unroll
    for (int nb = 0; nb < 2; ++nb) {
      P[T.r * TRW + 8 * nb + T.c2] = acc[nb][0];
      P[T.r * TRW + 8 * nb + T.c2 + 1] = acc[nb][1];
    }
  }
}
// tangential mass along p (My) on the z-face planes 8..11
__device__ __forceinline__ void plane_mass_cols(const Tile& T, const Frags& f) {
  for (int task = T.warp; task < 8; task += kThreads / 32) {
    const int plane = 8 + (task >> 1);
    if (!((T.nbm >> (plane >> 1)) & 1)) continue;
    double* P = T.tr + plane * TRP + (task & 1) * 8;
    double a[4];
#pragma unroll
    for (int kc = 0; kc < 4; ++kc) a[kc] = P[(4 * kc + T.k4) * TRW + T.r];
    double acc[2][2] = {{0.0, 0.0}, {0.0, 0.0}};
    mass_group(f, a, acc);
    __syncwarp();
#pragma unroll
    for (int nb = 0; nb < 2; ++nb) {
      P[(8 * nb + T.c2) * TRW + T.r] = acc[nb][0];
      P[(8 * nb + T.c2 + 1) * TRW + T.r] = acc[nb][1];
    }
  }
}

// The x-face neighbour layers are staged through shared memory: the two x neighbour cell
// layers (2 x 16 x 16 rows of K doubles) go to the still-unused B buffer by cp.async -- row
// segments, coalesced, no registers -- instead of per-lane K-double LDGs that touch 32 cache
// lines per warp instruction.  Chunk c of staged row i sits at a swizzled chunk so the 8 lanes
// of an LDS.128 quarter-warp hit 8 distinct bank groups (K = 8: c ^ ((i >> 1) & 3); K = 4:
// c ^ ((i >> 2) & 1); K = 2: one chunk per row, conflict-free as is).  y/z faces keep the
// register path (their loads are row-coalesced).
template <int K = 8>
__device__ __forceinline__ int xs_idx(int row, int c) {
  if constexpr (K == 8) return row * 8 + 2 * (c ^ ((row >> 1) & 3));
  else if constexpr (K == 4) return row * 4 + 2 * (c ^ ((row >> 2) & 1));
  else return row * K + 2 * c;
}

// Address arithmetic is strength-reduced: every thread's cp.async chunks and trace items share
// one (x, y) position and step only in z (or along the face normal), so each source/destination
// is one pointer plus a constant stride instead of a fresh 64-bit index computation per element
// (the prologue was half of the kernel's instructions).
template <int K = 8, class S = double, class OpT>
__device__ __forceinline__ void prologue_fast(Tile& T, const Geom& g, const OpT& op, const S* __restrict__ u,
                                              const Frags& f, const double* __restrict__ ltab = nullptr) {
  constexpr bool F32 = sizeof(S) == 4;
  const int tid = threadIdx.x;
  // optional: the L_smooth fragment table (4 kinds x 8 x 32 doubles) -> shared memory, so the
  // stage loops read it with LDS; loads issued here, stored after the trace loads are in flight
  double lt[4];
  if (ltab) {
#pragma unroll
    for (int i = 0; i < 4; ++i) lt[i] = __ldg(ltab + tid + kThreads * i);
  }
  // 32-bit element strides (host guarantees 24 * sz < 2^31): one IMAD.WIDE per address
  const int sy = (int)T.sy, sz = (int)T.sz;
  const long long txy = (long long)(T.cy * K) * sy + T.cx * K;  // tile origin within a z plane
  const S* ub = u + (long long)(T.cz * K) * sz + txy;
  // fp32 storage: tile and x-face rows are staged as floats in the still-unused B buffer by
  // cp.async (16-byte chunks; 8-byte for K = 2, whose shifted tiles are only 8-byte aligned) and
  // widened to fp64 after the wait; fp64 storage: cp.async straight into the tile / B buffer
  constexpr int VEC = K == 2 ? 2 : 4, NV = 16 / VEC, LGV = NV == 4 ? 2 : 3;
  float* stg = reinterpret_cast<float*>(T.sB);  // [0, 4096): tile z*256+y*16+x; then x rows (hi, z, y) x K
  const int p = (tid >> 4) & 15, q = tid & 15;
  if constexpr (F32) {
    const int x = VEC * (tid & (NV - 1)), y = (tid >> LGV) & 15, z0 = tid >> (LGV + 4);
    const S* src = ub + z0 * sz + y * sy + x;
    float* dst = stg + z0 * 256 + y * 16 + x;
#pragma unroll
    for (int i = 0; i < 16 / VEC; ++i) {
      if constexpr (VEC == 4) cp_async16(dst + (16 / NV) * i * 256, src + (16 / NV) * i * sz);
      else cp_async8(dst + (16 / NV) * i * 256, src + (16 / NV) * i * sz);
    }
    // x-neighbour rows: chunk ch of row (hi, z, y); K / VEC chunks per row
    constexpr int RC = K / VEC, LR = RC == 2 ? 1 : 0;
    const int ch = tid & (RC - 1), yy = (tid >> LR) & 15, zb = tid >> (LR + 4);
    constexpr int ZS = 256 / (16 * RC);  // z step per pass
#pragma unroll
    for (int hi = 0; hi < 2; ++hi) {
      if (!((T.nbm >> hi) & 1)) continue;
      const S* s0 = ub + zb * sz + yy * sy + (hi ? B : -K) + VEC * ch;
      float* d0 = stg + 4096 + ((hi * 16 + zb) * 16 + yy) * K + VEC * ch;
#pragma unroll
      for (int k = 0; k < 16 / ZS; ++k) {
        if constexpr (VEC == 4) cp_async16(d0 + ZS * k * 16 * K, s0 + ZS * k * sz);
        else cp_async8(d0 + ZS * k * 16 * K, s0 + ZS * k * sz);
      }
    }
  } else {
    {  // tile: chunk (x2 = tid & 7, y = (tid >> 3) & 15, z = (tid >> 7) + 2i)
      const int x2 = tid & 7, y = (tid >> 3) & 15, z0 = tid >> 7;
      const S* src = ub + z0 * sz + y * sy + 2 * x2;
      double* dst = &T.sU[idxU<K>(z0, y, 2 * x2)];
#pragma unroll
      for (int i = 0; i < 8; ++i) cp_async16(dst + i * 512, src + 2 * i * sz);
    }
    {  // x-neighbour layers: K/2 16-byte chunks per row (hi, z, y); chunk ch = tid % (K/2),
       // y = (tid / (K/2)) & 15, z = zb + (32/K) k  -- every k step is 512 staged doubles
      constexpr int KC = K / 2, LG = KC == 4 ? 2 : (KC == 2 ? 1 : 0);
      const int ch = tid & (KC - 1), y = (tid >> LG) & 15, zb = tid >> (LG + 4);
#pragma unroll
      for (int hi = 0; hi < 2; ++hi) {
        if (!((T.nbm >> hi) & 1)) continue;
        const S* src = ub + zb * sz + y * sy + (hi ? B : -K) + 2 * ch;
        double* dst = &T.sB[xs_idx<K>((hi * 16 + zb) * 16 + y, ch)];
#pragma unroll
        for (int k = 0; k < KC; ++k) cp_async16(dst + k * 512, src + (32 / K) * k * sz);
      }
    }
  }
  // y and z faces: item (hi = j, p = (tid >> 4) & 15, q = tid & 15); K values along the normal
  double w1[2][K], w2[2][K];
#pragma unroll
  for (int hi = 0; hi < 2; ++hi) {
    if ((T.nbm >> (2 + hi)) & 1) {  // y faces: Z = p, X = q, Y = hi ? 16 : -8
      const S* b1 = ub + p * sz + q + (hi ? B : -K) * sy;
#pragma unroll
      for (int c = 0; c < K; ++c) w1[hi][c] = __ldg(b1 + c * sy);
    }
    if ((T.nbm >> (4 + hi)) & 1) {  // z faces: Y = p, X = q, Z = hi ? 16 : -8 (ghost planes past the slab)
      const S* b2;
      const bool inside = hi ? (T.cz + 16 / K < g.nz) : (T.cz > 0);
      if (inside) b2 = ub + (hi ? B : -K) * sz + p * sy + q;
      else b2 = reinterpret_cast<const S*>(hi ? g.ghost_hi : g.ghost_lo) + txy + p * sy + q;
#pragma unroll
      for (int c = 0; c < K; ++c) w2[hi][c] = __ldg(b2 + c * sz);
    }
  }
  auto trace = [&](const double* w, int hi, double* pl) {
    double alpha, beta = 0.0;
    if (hi) {
      alpha = w[0];
#pragma unroll
      for (int c = 1; c < K; ++c) beta = fma(op.urow[c].h, w[c], beta);
    } else {
      alpha = w[K - 1];
#pragma unroll
      for (int c = 0; c < K - 1; ++c) beta = fma(op.ucol[c].h, w[c], beta);
    }
    pl[0] = alpha;
    pl[TRP] = rd<S>(beta);
  };
#pragma unroll
  for (int hi = 0; hi < 2; ++hi) {
#pragma unroll
    for (int axis = 1; axis < 3; ++axis) {
      if (!((T.nbm >> (2 * axis + hi)) & 1)) continue;
      trace(axis == 1 ? w1[hi] : w2[hi], hi, T.tr + (2 * axis + hi) * 2 * TRP + p * TRW + q);
    }
  }
  if (ltab) {
    double* dst = const_cast<double*>(T.sLf);
#pragma unroll
    for (int i = 0; i < 4; ++i) dst[tid + kThreads * i] = lt[i];
  }
  if constexpr (!F32) {
    cp_async_wait_all();
    __syncthreads();
    // x traces from the staged layers: item (hi, p = z, q = y) -> one staged row
#pragma unroll
    for (int hi = 0; hi < 2; ++hi) {
      if (!((T.nbm >> hi) & 1)) continue;
      const int row = (hi * 16 + p) * 16 + q;
      double w[K];
#pragma unroll
      for (int ch = 0; ch < K / 2; ++ch) {
        const double2 v2 = *reinterpret_cast<const double2*>(&T.sB[xs_idx<K>(row, ch)]);
        w[2 * ch] = v2.x;
        w[2 * ch + 1] = v2.y;
      }
      trace(w, hi, T.tr + hi * 2 * TRP + p * TRW + q);
    }
  } else {
    cp_async_wait_all();
    __syncthreads();
    {  // widen the staged tile into the U layout
      const int x = VEC * (tid & (NV - 1)), y = (tid >> LGV) & 15, z0 = tid >> (LGV + 4);
#pragma unroll
      for (int i = 0; i < 16 / VEC; ++i) {
        const int z = z0 + (16 / NV) * i;
        const float* src = stg + z * 256 + y * 16 + x;
#pragma unroll
        for (int j = 0; j < VEC; j += 2) {
          const float2 v2 = *reinterpret_cast<const float2*>(src + j);
          *reinterpret_cast<double2*>(&T.sU[idxU<K>(z, y, x + j)]) = make_double2(v2.x, v2.y);
        }
      }
    }
#pragma unroll
    for (int hi = 0; hi < 2; ++hi) {
      if (!((T.nbm >> hi) & 1)) continue;
      const float* row = stg + 4096 + ((hi * 16 + p) * 16 + q) * K;
      double w[K];
#pragma unroll
      for (int c = 0; c < K; c += 2) {
        const float2 v2 = *reinterpret_cast<const float2*>(row + c);
        w[c] = v2.x;
        w[c + 1] = v2.y;
      }
      trace(w, hi, T.tr + hi * 2 * TRP + p * TRW + q);
    }
  }
  plane_mass_rows(T, f, 4);
  plane_mass_rows(T, f, 8);
  __syncthreads();  // also: staged layers consumed before the x stage writes B
  plane_mass_cols(T, f);
  __syncthreads();
}


}  // namespace dm
}  // namespace sf
