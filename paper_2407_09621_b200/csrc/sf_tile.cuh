// The tile engine: one CTA evaluates the SIPG Laplacian on TPC tiles of
// 2x2x2 cells ((2K)^3 dofs each) with sum factorisation on CUDA cores.
//
// Schedule per tile, x = fastest axis:
//   stage 0  load u tile -> smem (coalesced rows)
//   stage 1  face traces of the 6 neighbouring cell layers (alpha = face value,
//            beta = the U-row dot product over the neighbour's K nodes); domain
//            boundary faces are skipped (the line stages apply Nitsche instead)
//   stage 1b tangential masses on the y-face (Mx) and z-face (My Mx) trace planes
//   stage 2  x lines:  a = Mx u,  b = Dx* u
//   stage 3  y lines:  c = My a,  dd = Dy* a + My b
//   stage 4  z lines:  v = Dz* c + Mz dd
// where Dt* is the block-tridiagonal 1-D operator along t restricted to the
// tile's 2K-line plus the rank-2 couplings to the face neighbours (or the
// Nitsche boundary correction).  Every contraction follows the mode's operand
// semantics (sf_common.cuh).
#pragma once
#include "sf_common.cuh"

namespace sf {

template <int K, int MODE>
__device__ __forceinline__ void mass_line(const LevelOp<K, MODE>& op, const Op<MODE>* w, Acc<MODE>* acc) {
#pragma unroll
  for (int c = 0; c < 2; ++c)
#pragma unroll
    for (int i = 0; i < K; ++i)
#pragma unroll
      for (int j = 0; j < K; ++j) acc[c * K + i].fma(op.M[i][j], w[c * K + j]);
}

// Line operator along one axis over the tile's two cells (2K values).
// lo side of cell 0: neighbour (alpha_lo prepared, beta_lo finished value) or Nitsche;
// hi side of cell 1 likewise.
template <int K, int MODE>
__device__ __forceinline__ void stiff_line(const LevelOp<K, MODE>& op, const Op<MODE>* w, Acc<MODE>* acc,
                                           bool lo_bnd, const Op<MODE>& a_lo, typename MT<MODE>::C b_lo,
                                           bool hi_bnd, const Op<MODE>& a_hi, typename MT<MODE>::C b_hi) {
  // diagonal blocks
#pragma unroll
  for (int c = 0; c < 2; ++c)
#pragma unroll
    for (int i = 0; i < K; ++i)
#pragma unroll
      for (int j = 0; j < K; ++j) acc[c * K + i].fma(op.D[i][j], w[c * K + j]);
  // the face inside the tile: cell 0 <- U w1, cell 1 <- U^T w0
#pragma unroll
  for (int i = 0; i < K; ++i) acc[i].fma(op.ucol[i], w[K]);
#pragma unroll
  for (int j = 1; j < K; ++j) acc[K - 1].fma(op.urow[j], w[K + j]);
#pragma unroll
  for (int i = 0; i < K; ++i) acc[K + i].fma(op.urow[i], w[K - 1]);
#pragma unroll
  for (int j = 0; j < K - 1; ++j) acc[K].fma(op.ucol[j], w[j]);
  // low end of cell 0
  if (lo_bnd) {
#pragma unroll
    for (int i = 0; i < K; ++i) acc[i].fma(op.bl[i], w[0]);
#pragma unroll
    for (int j = 1; j < K; ++j) acc[0].fma(op.bl[j], w[j]);
  } else {
#pragma unroll
    for (int i = 0; i < K; ++i) acc[i].fma(op.urow[i], a_lo);
    acc[0].add(b_lo);
  }
  // high end of cell 1
  if (hi_bnd) {
#pragma unroll
    for (int i = 0; i < K; ++i) acc[K + i].fma(op.br[i], w[2 * K - 1]);
#pragma unroll
    for (int j = 0; j < K - 1; ++j) acc[2 * K - 1].fma(op.br[j], w[K + j]);
  } else {
#pragma unroll
    for (int i = 0; i < K; ++i) acc[K + i].fma(op.ucol[i], a_hi);
    acc[2 * K - 1].add(b_hi);
  }
}

// Generic cell-local contraction of a B-line with a per-cell K x K matrix table.
template <int K, int MODE>
__device__ __forceinline__ void cell_line(const ME<MODE> (*Mt)[K], const Op<MODE>* w, Acc<MODE>* acc) {
#pragma unroll
  for (int c = 0; c < 2; ++c)
#pragma unroll
    for (int i = 0; i < K; ++i)
#pragma unroll
      for (int j = 0; j < K; ++j) acc[c * K + i].fma(Mt[i][j], w[c * K + j]);
}

// boundary kind of a 2-cell patch along an axis: 2*left_at_domain_boundary + right_at_domain_boundary
__device__ __forceinline__ int patch_kind(const Geom& g, int axis, int c0) {
  int n = axis == 0 ? g.nx : (axis == 1 ? g.ny : g.nz);
  int lb = (c0 == 0 && g.bnd_lo[axis]) ? 1 : 0;
  int rb = (c0 + 2 == n && g.bnd_hi[axis]) ? 1 : 0;
  return 2 * lb + rb;
}

// BL = points per tile line: 2K (2-cell tiles, the generic engine) or 16 (the 16-point line
// tiles of the tensor-core kernels, 16/K cells; only tile_cells / face_src / traces are used then).
template <int K, int MODE, int TPC, int BL = 2 * K>
struct TileEngine {
  static constexpr int B = BL;
  static constexpr int CPL = BL / K;  // cells per tile line
  static constexpr int P = B + 1;          // padded row pitch (conflict-free x lines)
  static constexpr int VOL = B * B * P;    // one padded tile
  static constexpr int PL = B * P;         // one padded face plane
  using C = typename MT<MODE>::C;
  using S = typename MT<MODE>::S;

  static constexpr size_t smem_bytes() { return sizeof(C) * TPC * (2 * VOL + 12 * PL) + 16; }
  static constexpr bool kHalf = MT<MODE>::kHalf;

  C* su;  // [TPC][VOL]
  C* sb;  // [TPC][VOL]
  C* tr;  // [TPC][6][2][PL]
  int* s_exp;  // [0]: max|u| bits, [1]: max|r| bits (binary16 block exponents)
  int eu = 0;  // block exponent of the input tile (binary16 modes), u^ = 2^eu u
  int ntiles_total;
  int tile0;
  mutable int skip[3] = {0, 0, 0};  // line tiles: leading points per axis owned by the previous tile
  long long sy, sz;

  __device__ __forceinline__ TileEngine(char* smem, const Geom& g) {
    su = reinterpret_cast<C*>(smem);
    sb = su + TPC * VOL;
    tr = sb + TPC * VOL;
    s_exp = reinterpret_cast<int*>(tr + TPC * 12 * PL);
    ntiles_total = g.ntx * g.nty * g.ntz;
    tile0 = blockIdx.x * TPC;
    sy = (long long)g.nx * K;
    sz = sy * (long long)g.ny * K;
  }

  __device__ __forceinline__ static int idx(int z, int y, int x) { return (z * B + y) * P + x; }

  // tile -> first cell per axis
  __device__ __forceinline__ bool tile_cells(const Geom& g, int t, int& cx, int& cy, int& cz) const {
    int id = tile0 + t;
    if (id >= ntiles_total) return false;
    int tx, ty, tz;
    tile_coords<BL / 2>(g, id, tx, ty, tz);  // band sized by the tile's bytes
    cx = g.tx0 + CPL * tx;
    cy = g.ty0 + CPL * ty;
    cz = g.tz0 + CPL * tz;
    if constexpr (CPL > 2) {  // shifted colour (odd offset): the last line ends at cell n-2
      const int ux = cx, uy = cy, uz = cz;
      if (g.tx0 & 1) cx = min(cx, g.nx - CPL - g.tx0);
      if (g.ty0 & 1) cy = min(cy, g.ny - CPL - g.ty0);
      if (g.tz0 & 1) cz = min(cz, g.nz - CPL - g.tz0);
      skip[0] = (ux - cx) * K;  // leading points written by the previous line (single writer)
      skip[1] = (uy - cy) * K;
      skip[2] = (uz - cz) * K;
    }
    return true;
  }

  // 0: neighbour inside the local array, 1: ghost (z only), 2: domain boundary
  __device__ __forceinline__ static int face_src(const Geom& g, int axis, int hi, int c0) {
    int n = axis == 0 ? g.nx : (axis == 1 ? g.ny : g.nz);
    int c = hi ? c0 + CPL : c0 - 1;
    if (c >= 0 && c < n) return 0;
    if (hi ? g.bnd_hi[axis] : g.bnd_lo[axis]) return 2;
    return 1;
  }

  // ---------------------------------------------------------------- stage 0
  __device__ __forceinline__ void load(const Geom& g, const S* __restrict__ u) {
    for (int i = threadIdx.x; i < TPC * B * B * B; i += blockDim.x) {
      int x = i % B;
      int r = i / B;
      int t = r % TPC;
      r /= TPC;
      int y = r % B;
      int z = r / B;
      int cx, cy, cz;
      C val = C(0);
      if (tile_cells(g, t, cx, cy, cz))
        val = (C)u[(long long)(cz * K + z) * sz + (long long)(cy * K + y) * sy + (cx * K + x)];
      su[t * VOL + idx(z, y, x)] = val;
      if constexpr (kHalf) smax(&s_exp[0], (float)val);
    }
  }

  __device__ __forceinline__ void init_exp() {
    if (threadIdx.x == 0) s_exp[0] = s_exp[1] = 0;
  }
  // input scale 2^eu (binary16 modes: max |u^| in [2, 4))
  __device__ __forceinline__ C uscale() const {
    if constexpr (kHalf) return pow2f(eu);
    return C(1);
  }

  // ---------------------------------------------------------------- stage 1
  // Face traces of the neighbour cell layers, one axis at a time with all of a
  // thread's loads for that axis in flight before any use (high MLP).
  template <int NTH = 256, int FIRST_AXIS = 0>
  __device__ __forceinline__ void traces(const Geom& g, const LevelOp<K, MODE>& op, const S* __restrict__ u) {
    constexpr int ITEMS = TPC * 2 * B * B;  // per axis: 2 faces x B^2 positions per tile
    constexpr int IPT = (ITEMS + NTH - 1) / NTH;
    const C us = uscale();
#pragma unroll
    for (int axis = FIRST_AXIS; axis < 3; ++axis) {
      C w[IPT][K];
      bool act[IPT];
#pragma unroll
      for (int jj = 0; jj < IPT; ++jj) {
        const int i = threadIdx.x + NTH * jj;
        act[jj] = false;
        if (i >= ITEMS) continue;
        const int q = i % B, p = (i / B) % B, hi = (i / (B * B)) & 1, t = i / (2 * B * B);
        int cx, cy, cz;
        if (!tile_cells(g, t, cx, cy, cz)) continue;
        const int c0 = axis == 0 ? cx : (axis == 1 ? cy : cz);
        const int src = face_src(g, axis, hi, c0);
        if (src == 2) continue;
        act[jj] = true;
        int X = cx * K, Y = cy * K, Z = cz * K;
        long long step;
        if (axis == 0) { Z += p; Y += q; X += hi ? B : -K; step = 1; }
        else if (axis == 1) { Z += p; X += q; Y += hi ? B : -K; step = sy; }
        else { Y += p; X += q; Z += hi ? B : -K; step = sz; }
        const S* base;
        if (src == 0) {
          base = u + (long long)Z * sz + (long long)Y * sy + X;
        } else if (hi) {
          base = reinterpret_cast<const S*>(g.ghost_hi) + (long long)(Z - g.nz * K) * sz + (long long)Y * sy + X;
        } else {
          base = reinterpret_cast<const S*>(g.ghost_lo) + (long long)(Z + K) * sz + (long long)Y * sy + X;
        }
        constexpr int V = 16 / sizeof(S);  // elements per 16-byte vector
        if (axis == 0 && K % V == 0) {
          // x faces: the neighbour's K nodes are contiguous -- 16-byte loads (4x / 2x fewer
          // L1 wavefronts than scalar loads that each touch a different row)
#pragma unroll
          for (int c = 0; c < K / V; ++c) {
            if constexpr (V == 4) {
              const float4 q4 = __ldg(reinterpret_cast<const float4*>(base) + c);
              w[jj][4 * c] = (C)q4.x; w[jj][4 * c + 1] = (C)q4.y; w[jj][4 * c + 2] = (C)q4.z; w[jj][4 * c + 3] = (C)q4.w;
            } else {
              const double2 d2 = __ldg(reinterpret_cast<const double2*>(base) + c);
              w[jj][2 * c] = (C)d2.x; w[jj][2 * c + 1] = (C)d2.y;
            }
          }
        } else {
#pragma unroll
          for (int j = 0; j < K; ++j) w[jj][j] = (C)__ldg(base + j * step);
        }
      }
#pragma unroll
      for (int jj = 0; jj < IPT; ++jj) {
        if (!act[jj]) continue;
        const int i = threadIdx.x + NTH * jj;
        const int q = i % B, p = (i / B) % B, hi = (i / (B * B)) & 1, t = i / (2 * B * B);
        C alpha, bsum;
        if constexpr (MODE == MODE_FP16_EC) {
          // EC: the halo partial sums in plain fp32 (operands main + residual/2048
          // reconstruct the fp32 values to 2^-22, so this is the EC product or better)
          float bs = 0.f;
          if (hi) {
            alpha = w[jj][0] * us;
#pragma unroll
            for (int j = 1; j < K; ++j) bs = fmaf(op.urow[j].h + op.urow[j].d / kEcScale, w[jj][j] * us, bs);
          } else {
            alpha = w[jj][K - 1] * us;
#pragma unroll
            for (int j = 0; j < K - 1; ++j) bs = fmaf(op.ucol[j].h + op.ucol[j].d / kEcScale, w[jj][j] * us, bs);
          }
          bsum = bs;
        } else {
          Acc<MODE> beta;
          if (hi) {  // neighbour above: alpha = w[0], beta = sum_{j>=1} urow[j] w[j]
            alpha = w[jj][0] * us;
#pragma unroll
            for (int j = 1; j < K; ++j) beta.fma(op.urow[j], prep<MODE>(w[jj][j] * us));
          } else {   // neighbour below: alpha = w[K-1], beta = sum_{j<=K-2} ucol[j] w[j]
            alpha = w[jj][K - 1] * us;
#pragma unroll
            for (int j = 0; j < K - 1; ++j) beta.fma(op.ucol[j], prep<MODE>(w[jj][j] * us));
          }
          bsum = beta.result();
        }
        C* pl = tr + ((t * 6 + 2 * axis + hi) * 2) * PL;
        pl[p * P + q] = alpha;
        pl[PL + p * P + q] = bsum;
      }
    }
  }

  // tangential masses: y faces (2,3): Mx along q; z faces (4,5): Mx along q then My along p
  __device__ __forceinline__ void trace_masses(const Geom& g, const LevelOp<K, MODE>& op) {
    for (int i = threadIdx.x; i < TPC * 4 * 2 * B; i += blockDim.x) {
      int row = i % B;
      int pl_id = (i / B) % 2;
      int f = 2 + (i / (2 * B)) % 4;
      int t = i / (8 * B);
      int cx, cy, cz;
      if (!tile_cells(g, t, cx, cy, cz)) continue;
      int axis = f >> 1, hi = f & 1;
      if (face_src(g, axis, hi, axis == 1 ? cy : cz) == 2) continue;
      C* r = tr + ((t * 6 + f) * 2 + pl_id) * PL + row * P;
      Op<MODE> w[B];
#pragma unroll
      for (int j = 0; j < B; ++j) w[j] = prep<MODE>(r[j]);
      Acc<MODE> acc[B];
      mass_line<K, MODE>(op, w, acc);
#pragma unroll
      for (int j = 0; j < B; ++j) r[j] = acc[j].result();
    }
    __syncthreads();
    for (int i = threadIdx.x; i < TPC * 2 * 2 * B; i += blockDim.x) {
      int col = i % B;
      int pl_id = (i / B) % 2;
      int f = 4 + (i / (2 * B)) % 2;
      int t = i / (4 * B);
      int cx, cy, cz;
      if (!tile_cells(g, t, cx, cy, cz)) continue;
      if (face_src(g, 2, f & 1, cz) == 2) continue;
      C* r = tr + ((t * 6 + f) * 2 + pl_id) * PL + col;
      Op<MODE> w[B];
#pragma unroll
      for (int j = 0; j < B; ++j) w[j] = prep<MODE>(r[j * P]);
      Acc<MODE> acc[B];
      mass_line<K, MODE>(op, w, acc);
#pragma unroll
      for (int j = 0; j < B; ++j) r[j * P] = acc[j].result();
    }
  }

  __device__ __forceinline__ void face_in(const Geom& g, int t, int f, int c0, int pq, bool& bnd, Op<MODE>& a,
                                          C& b) const {
    bnd = face_src(g, f >> 1, f & 1, c0) == 2;
    if (!bnd) {
      const C* pl = tr + ((t * 6 + f) * 2) * PL;
      a = prep<MODE>(pl[pq]);
      b = pl[PL + pq];
    } else {
      a = prep<MODE>(C(0));
      b = C(0);
    }
  }

  // ---------------------------------------------------------------- stage 2
  __device__ __forceinline__ void xlines(const Geom& g, const LevelOp<K, MODE>& op) {
    for (int i = threadIdx.x; i < TPC * B * B; i += blockDim.x) {
      int y = i % B;
      int z = (i / B) % B;
      int t = i / (B * B);
      int cx, cy, cz;
      if (!tile_cells(g, t, cx, cy, cz)) continue;
      C* row = su + t * VOL + idx(z, y, 0);
      Op<MODE> w[B];
      const C us = uscale();
#pragma unroll
      for (int x = 0; x < B; ++x) w[x] = prep<MODE>(row[x] * us);
      bool lb, hb;
      Op<MODE> al, ah;
      C bl_, bh_;
      face_in(g, t, 0, cx, z * P + y, lb, al, bl_);
      face_in(g, t, 1, cx, z * P + y, hb, ah, bh_);
      Acc<MODE> a[B], b[B];
      mass_line<K, MODE>(op, w, a);
      stiff_line<K, MODE>(op, w, b, lb, al, bl_, hb, ah, bh_);
      C* rowb = sb + t * VOL + idx(z, y, 0);
#pragma unroll
      for (int x = 0; x < B; ++x) {
        row[x] = a[x].result();
        rowb[x] = b[x].result();
      }
    }
  }

  // ---------------------------------------------------------------- stage 3
  __device__ __forceinline__ void ylines(const Geom& g, const LevelOp<K, MODE>& op) {
    for (int i = threadIdx.x; i < TPC * B * B; i += blockDim.x) {
      int x = i % B;
      int z = (i / B) % B;
      int t = i / (B * B);
      int cx, cy, cz;
      if (!tile_cells(g, t, cx, cy, cz)) continue;
      C* ca = su + t * VOL + idx(z, 0, x);
      C* cb = sb + t * VOL + idx(z, 0, x);
      Op<MODE> wa[B], wb[B];
#pragma unroll
      for (int y = 0; y < B; ++y) {
        wa[y] = prep<MODE>(ca[y * P]);
        wb[y] = prep<MODE>(cb[y * P]);
      }
      bool lb, hb;
      Op<MODE> al, ah;
      C bl_, bh_;
      face_in(g, t, 2, cy, z * P + x, lb, al, bl_);
      face_in(g, t, 3, cy, z * P + x, hb, ah, bh_);
      Acc<MODE> c[B], d[B], e[B];
      mass_line<K, MODE>(op, wa, c);
      stiff_line<K, MODE>(op, wa, d, lb, al, bl_, hb, ah, bh_);
      mass_line<K, MODE>(op, wb, e);
#pragma unroll
      for (int y = 0; y < B; ++y) {
        ca[y * P] = c[y].result();
        cb[y * P] = d[y].result() + e[y].result();
      }
    }
  }

  // ---------------------------------------------------------------- stage 4
  // z line (t, y, x) -> v[0..B) in registers.  Returns false for idle threads.
  __device__ __forceinline__ void zline(const Geom& g, const LevelOp<K, MODE>& op, int t, int y, int x, int cz,
                                        C* v) const {
    const C* cc = su + t * VOL + idx(0, y, x);
    const C* cd = sb + t * VOL + idx(0, y, x);
    Op<MODE> wc[B], wd[B];
#pragma unroll
    for (int z = 0; z < B; ++z) {
      wc[z] = prep<MODE>(cc[z * B * P]);
      wd[z] = prep<MODE>(cd[z * B * P]);
    }
    bool lb, hb;
    Op<MODE> al, ah;
    C bl_, bh_;
    face_in(g, t, 4, cz, y * P + x, lb, al, bl_);
    face_in(g, t, 5, cz, y * P + x, hb, ah, bh_);
    Acc<MODE> s[B], m[B];
    stiff_line<K, MODE>(op, wc, s, lb, al, bl_, hb, ah, bh_);
    mass_line<K, MODE>(op, wd, m);
#pragma unroll
    for (int z = 0; z < B; ++z) v[z] = s[z].result() + m[z].result();
  }

  // factor turning zline() output (scaled units) into A u
  __device__ __forceinline__ C out_scale(const LevelOp<K, MODE>& op) const {
    if constexpr (kHalf) return pow2f(-(op.sc.aA + eu));
    return C(1);
  }

  // full A u on the tile up to (and excluding) stage 4; caller runs zline per thread
  __device__ __forceinline__ void apply_to_zstage(const Geom& g, const LevelOp<K, MODE>& op, const S* __restrict__ u) {
    init_exp();
    __syncthreads();
    load(g, u);
    if constexpr (kHalf) {
      __syncthreads();
      eu = block_exp(__int_as_float(s_exp[0]));
    }
    traces(g, op, u);
    __syncthreads();
    trace_masses(g, op);
    __syncthreads();
    xlines(g, op);
    __syncthreads();
    ylines(g, op);
    __syncthreads();
  }
};

}  // namespace sf
