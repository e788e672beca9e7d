// Operator kernels (vmult, smoother colour pass, residual+restriction,
// prolongation+add) and their C-ABI entry points.  See include/sumfact_b200.h
// for the contract and the reference interface each entry point replaces.
#include <cstdint>
#include <cuda_runtime.h>
#include <cuda_fp16.h>

#include <cstdio>
#include <cstring>
#include <type_traits>

#include "sf_common.cuh"
#include "sf_tile.cuh"
#include "../../include/sumfact_b200.h"
#include "sf_internal.h"
#include <cstdlib>

namespace sf {

// tiles per CTA so that a CTA runs ~256 lines per stage
template <int K>
struct Tpc {
  static constexpr int B2 = 4 * K * K;
  static constexpr int value = B2 >= 256 ? 1 : (256 / B2);
};
// K=2: 16, K=3: 7, K=4: 4, K=5: 2, K=6..8: 1

constexpr int kThreads = 256;

// ------------------------------------------------------------------ vmult
template <int K, int MODE>
__global__ void __launch_bounds__(kThreads) k_vmult(const typename MT<MODE>::S* __restrict__ u,
                                                    typename MT<MODE>::S* __restrict__ v, Geom g,
                                                    LevelOp<K, MODE> op) {
  constexpr int TPC = Tpc<K>::value;
  using E = TileEngine<K, MODE, TPC>;
  using C = typename E::C;
  extern __shared__ __align__(16) char smem[];
  u += (long long)blockIdx.y * g.batch_stride;
  v += (long long)blockIdx.y * g.batch_stride;
  E e(smem, g);
  e.apply_to_zstage(g, op, u);
  const C os = e.out_scale(op);
  for (int i = threadIdx.x; i < TPC * E::B * E::B; i += blockDim.x) {
    int x = i % E::B;
    int y = (i / E::B) % E::B;
    int t = i / (E::B * E::B);
    int cx, cy, cz;
    if (!e.tile_cells(g, t, cx, cy, cz)) continue;
    C vv[E::B];
    e.zline(g, op, t, y, x, cz, vv);
    typename E::S* out = v + (long long)(cz * K) * e.sz + (long long)(cy * K + y) * e.sy + (cx * K + x);
#pragma unroll
    for (int z = 0; z < E::B; ++z) out[z * e.sz] = (typename E::S)(vv[z] * os);
  }
}

// full-matrix contraction of a B-line: acc[i] += A[i][j] w[j] (trans: A[j][i])
template <int B, int MODE, bool TRANS>
__device__ __forceinline__ void full_line(const ME<MODE>* A, const Op<MODE>* w, Acc<MODE>* acc) {
#pragma unroll
  for (int i = 0; i < B; ++i)
#pragma unroll
    for (int j = 0; j < B; ++j) acc[i].fma(TRANS ? A[j * B + i] : A[i * B + j], w[j]);
}

// divisor of the fast-diagonalisation step: (lambda sum) [* 2^-aD in binary16 modes]
template <int MODE>
__device__ __forceinline__ typename MT<MODE>::C lam_div(double lsum, const Scales& sc) {
  if constexpr (MT<MODE>::kHalf) return (typename MT<MODE>::C)(lsum * pow2d(-sc.aD));
  return (typename MT<MODE>::C)lsum;
}
// factor turning the scaled patch correction back into S^-1 r (binary16 modes)
template <int MODE>
__device__ __forceinline__ typename MT<MODE>::C corr_scale(const Scales& sc, int er) {
  if constexpr (MT<MODE>::kHalf) return pow2f(-(sc.aD + 6 * sc.aV + er));
  return typename MT<MODE>::C(1);
}
template <int MODE>
__device__ __forceinline__ int read_exp(const int* word) {
  if constexpr (MT<MODE>::kHalf) return block_exp(__int_as_float(*word));
  return 0;
}

// --------------------------------------------------- smoother colour pass
// One colour (tiling shift) of the multiplicative vertex-patch smoother,
// multigrid.py:186-203: r = b - A x on each patch, x_new = x + P^-1 r with the
// fast-diagonalisation inverse.  Reads x_old, writes x_new (ping-pong) so the
// residual of every patch sees only pre-colour values, exactly as the
// reference's full-vector residual does.  (TPC * B^2 <= blockDim: one line per
// thread and stage.)
template <int K, int MODE>
__global__ void __launch_bounds__(kThreads) k_colour(const typename MT<MODE>::S* __restrict__ xo,
                                                     const typename MT<MODE>::S* __restrict__ b,
                                                     typename MT<MODE>::S* __restrict__ xn, Geom g,
                                                     LevelOp<K, MODE> op, PatchEig<K, MODE> eig) {
  constexpr int TPC = Tpc<K>::value;
  using E = TileEngine<K, MODE, TPC>;
  using C = typename E::C;
  using S = typename E::S;
  constexpr int B = E::B, P = E::P, NL = TPC * B * B;
  extern __shared__ __align__(16) char smem[];
  E e(smem, g);
  ME<MODE>* sV = reinterpret_cast<ME<MODE>*>(smem + E::smem_bytes());
  double* sLam = reinterpret_cast<double*>(sV + 4 * B * B);
  for (int i = threadIdx.x; i < 4 * B * B; i += blockDim.x) sV[i] = (&eig.V[0][0][0])[i];
  for (int i = threadIdx.x; i < 4 * B; i += blockDim.x) sLam[i] = (&eig.lam[0][0])[i];
  e.apply_to_zstage(g, op, xo);
  const int i = threadIdx.x;
  int cx = 0, cy = 0, cz = 0;
  const bool act = i < NL && e.tile_cells(g, i / (B * B), cx, cy, cz);
  const int t = i / (B * B);
  {  // z lines: residual (true units), block exponent, forward V_z^T
    const int x = i % B, y = (i / B) % B;
    C r[B];
    if (act) {
      C vv[B];
      e.zline(g, op, t, y, x, cz, vv);
      const C os = e.out_scale(op);
      const S* bp = b + (long long)(cz * K) * e.sz + (long long)(cy * K + y) * e.sy + (cx * K + x);
#pragma unroll
      for (int z = 0; z < B; ++z) {
        r[z] = (C)bp[z * e.sz] - vv[z] * os;
        if constexpr (E::kHalf) smax(&e.s_exp[1], (float)r[z]);
      }
    }
    __syncthreads();
    const C rs = E::kHalf ? (C)pow2f(read_exp<MODE>(&e.s_exp[1])) : C(1);
    if (act) {
      Op<MODE> w[B];
#pragma unroll
      for (int z = 0; z < B; ++z) w[z] = prep<MODE>(r[z] * rs);
      Acc<MODE> acc[B];
      full_line<B, MODE, true>(sV + patch_kind(g, 2, cz) * B * B, w, acc);
      C* col = e.su + t * E::VOL + E::idx(0, y, x);
#pragma unroll
      for (int z = 0; z < B; ++z) col[z * B * P] = acc[z].result();
    }
  }
  __syncthreads();
  const int er = read_exp<MODE>(&e.s_exp[1]);
  if (act) {  // y lines: forward V_y^T
    const int x = i % B, z = (i / B) % B;
    C* col = e.su + t * E::VOL + E::idx(z, 0, x);
    Op<MODE> w[B];
#pragma unroll
    for (int y = 0; y < B; ++y) w[y] = prep<MODE>(col[y * P]);
    Acc<MODE> acc[B];
    full_line<B, MODE, true>(sV + patch_kind(g, 1, cy) * B * B, w, acc);
#pragma unroll
    for (int y = 0; y < B; ++y) col[y * P] = acc[y].result();
  }
  __syncthreads();
  if (act) {  // x lines: forward V_x^T, divide by eigenvalue sums, backward V_x
    const int y = i % B, z = (i / B) % B;
    const int kx = patch_kind(g, 0, cx), ky = patch_kind(g, 1, cy), kz = patch_kind(g, 2, cz);
    C* row = e.su + t * E::VOL + E::idx(z, y, 0);
    Op<MODE> w[B];
#pragma unroll
    for (int x = 0; x < B; ++x) w[x] = prep<MODE>(row[x]);
    Acc<MODE> acc[B];
    full_line<B, MODE, true>(sV + kx * B * B, w, acc);
    const double lzy = (0.0 + sLam[kz * B + z]) + sLam[ky * B + y];
#pragma unroll
    for (int x = 0; x < B; ++x) w[x] = prep<MODE>(acc[x].result() / lam_div<MODE>(lzy + sLam[kx * B + x], op.sc));
    Acc<MODE> acc2[B];
    full_line<B, MODE, false>(sV + kx * B * B, w, acc2);
#pragma unroll
    for (int x = 0; x < B; ++x) row[x] = acc2[x].result();
  }
  __syncthreads();
  if (act) {  // y lines: backward V_y
    const int x = i % B, z = (i / B) % B;
    C* col = e.su + t * E::VOL + E::idx(z, 0, x);
    Op<MODE> w[B];
#pragma unroll
    for (int y = 0; y < B; ++y) w[y] = prep<MODE>(col[y * P]);
    Acc<MODE> acc[B];
    full_line<B, MODE, false>(sV + patch_kind(g, 1, cy) * B * B, w, acc);
#pragma unroll
    for (int y = 0; y < B; ++y) col[y * P] = acc[y].result();
  }
  __syncthreads();
  if (act) {  // z lines: backward V_z, x_new = x_old + correction
    const int x = i % B, y = (i / B) % B;
    const C* col = e.su + t * E::VOL + E::idx(0, y, x);
    Op<MODE> w[B];
#pragma unroll
    for (int z = 0; z < B; ++z) w[z] = prep<MODE>(col[z * B * P]);
    Acc<MODE> acc[B];
    full_line<B, MODE, false>(sV + patch_kind(g, 2, cz) * B * B, w, acc);
    const C cs = corr_scale<MODE>(op.sc, er);
    long long off = (long long)(cz * K) * e.sz + (long long)(cy * K + y) * e.sy + (cx * K + x);
#pragma unroll
    for (int z = 0; z < B; ++z) xn[off + z * e.sz] = (S)((C)xo[off + z * e.sz] + acc[z].result() * cs);
  }
}

// cells not covered by a shifted colour keep their value in the ping-pong copy: the K-point boundary slabs of
// every shifted axis, as contiguous runs (z: two ranges of whole planes, y: two row blocks per plane, x: two
// K-point pieces per row) copied in 16-byte vectors V when K points are a whole number of them
template <typename V>
__global__ void k_copy_slabs(const V* __restrict__ xo, V* __restrict__ xn, int Kv, int K, int Axv, int Ay, int Az,
                             int sx, int sy_, int sz_) {
  const long long plane = (long long)Ay * Axv;
  const long long cz = sz_ ? 2LL * K * plane : 0;
  const long long cy = sy_ ? 2LL * Az * K * Axv : 0;
  const long long cx = sx ? 2LL * Az * Ay * Kv : 0;
  const long long total = cz + cy + cx;
  const int runy = K * Axv;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    long long o;
    if (i < cz) {
      const long long zr = K * plane;
      o = i < zr ? i : (Az - 2LL * K) * plane + i;
    } else if (i < cz + cy) {
      const long long j = i - cz;
      const long long Z = j / (2 * runy);
      const int r = (int)(j - Z * 2 * runy);
      o = Z * plane + (r < runy ? r : (long long)(Ay - 2 * K) * Axv + r);
    } else {
      const long long j = i - cz - cy;
      const long long row = j / (2 * Kv);
      const int r = (int)(j - row * 2 * Kv);
      o = row * Axv + (r < Kv ? r : Axv - 2 * Kv + r);
    }
    xn[o] = xo[o];
  }
}

template <typename S>
static void copy_slabs(const S* xo, S* xn, int K, const sf_grid* gr, const int* shift, cudaStream_t st) {
  const int Ax = gr->nx * K, Ay = gr->ny * K, Az = gr->nz * K;
  if ((K * sizeof(S)) % 16 == 0) {
    constexpr int w = 16 / sizeof(S);
    k_copy_slabs<uint4><<<148 * 4, 256, 0, st>>>((const uint4*)xo, (uint4*)xn, K / w, K, Ax / w, Ay, Az, shift[0],
                                                 shift[1], shift[2]);
  } else {
    k_copy_slabs<S><<<148 * 4, 256, 0, st>>>(xo, xn, K, K, Ax, Ay, Az, shift[0], shift[1], shift[2]);
  }
}

// --------------------------------------------- residual + restriction (fused)
// r = b - A x on each aligned 2x2x2 tile, then P^T along the three axes
// (multigrid.py:249-250 followed by restrict, multigrid.py:112-125).  With
// with_op == 0 the residual is b itself (plain restriction).
template <int K, int MODE>
__global__ void __launch_bounds__(kThreads) k_resid_restrict(const typename MT<MODE>::S* __restrict__ x,
                                                             const typename MT<MODE>::S* __restrict__ b,
                                                             typename MT<MODE>::S* __restrict__ coarse, Geom g,
                                                             LevelOp<K, MODE> op, Embed<K, MODE> emb, int with_op) {
  constexpr int TPC = Tpc<K>::value;
  using E = TileEngine<K, MODE, TPC>;
  using C = typename E::C;
  using S = typename E::S;
  constexpr int B = E::B, P = E::P, NL = TPC * B * B;
  extern __shared__ __align__(16) char smem[];
  E e(smem, g);
  if (with_op) {
    e.apply_to_zstage(g, op, x);
  } else {
    e.init_exp();
    __syncthreads();
  }
  long long syc = (long long)(g.nx / 2) * K, szc = syc * (long long)(g.ny / 2) * K;
  const int i = threadIdx.x;
  int cx = 0, cy = 0, cz = 0;
  const bool act = i < NL && e.tile_cells(g, i / (B * B), cx, cy, cz);
  const int t = i / (B * B);
  {  // z lines: residual, block exponent, restrict along z (B -> K)
    const int xx = i % B, y = (i / B) % B;
    C r[B];
    if (act) {
      C vv[B];
      if (with_op) e.zline(g, op, t, y, xx, cz, vv);
      const C os = e.out_scale(op);
      const S* bp = b + (long long)(cz * K) * e.sz + (long long)(cy * K + y) * e.sy + (cx * K + xx);
#pragma unroll
      for (int z = 0; z < B; ++z) {
        r[z] = with_op ? (C)bp[z * e.sz] - vv[z] * os : (C)bp[z * e.sz];
        if constexpr (E::kHalf) smax(&e.s_exp[1], (float)r[z]);
      }
    }
    __syncthreads();
    const C rs = E::kHalf ? (C)pow2f(read_exp<MODE>(&e.s_exp[1])) : C(1);
    if (act) {
      Op<MODE> w[B];
#pragma unroll
      for (int z = 0; z < B; ++z) w[z] = prep<MODE>(r[z] * rs);
      C* col = e.sb + t * E::VOL + E::idx(0, y, xx);
#pragma unroll
      for (int kc = 0; kc < K; ++kc) {
        Acc<MODE> a;
#pragma unroll
        for (int j = 0; j < B; ++j) a.fma(emb.P[j][kc], w[j]);
        col[kc * B * P] = a.result();
      }
    }
  }
  __syncthreads();
  const C back = E::kHalf ? (C)pow2f(-read_exp<MODE>(&e.s_exp[1])) : C(1);
  // y lines: (zc < K, x < B)
  for (int j2 = threadIdx.x; j2 < TPC * K * B; j2 += blockDim.x) {
    int xx = j2 % B, zc = (j2 / B) % K, tt = j2 / (K * B);
    int ax, ay, az;
    if (!e.tile_cells(g, tt, ax, ay, az)) continue;
    C* col = e.sb + tt * E::VOL + E::idx(zc, 0, xx);
    Op<MODE> w[B];
#pragma unroll
    for (int y = 0; y < B; ++y) w[y] = prep<MODE>(col[y * P]);
    C out[K];
#pragma unroll
    for (int kc = 0; kc < K; ++kc) {
      Acc<MODE> a;
#pragma unroll
      for (int j = 0; j < B; ++j) a.fma(emb.P[j][kc], w[j]);
      out[kc] = a.result();
    }
#pragma unroll
    for (int kc = 0; kc < K; ++kc) col[kc * P] = out[kc];
  }
  __syncthreads();
  // x lines: (zc, yc) -> K coarse values
  for (int j2 = threadIdx.x; j2 < TPC * K * K; j2 += blockDim.x) {
    int yc = j2 % K, zc = (j2 / K) % K, tt = j2 / (K * K);
    int ax, ay, az;
    if (!e.tile_cells(g, tt, ax, ay, az)) continue;
    const C* row = e.sb + tt * E::VOL + E::idx(zc, yc, 0);
    Op<MODE> w[B];
#pragma unroll
    for (int xx = 0; xx < B; ++xx) w[xx] = prep<MODE>(row[xx]);
    S* out = coarse + (long long)((az / 2) * K + zc) * szc + (long long)((ay / 2) * K + yc) * syc + (ax / 2) * K;
#pragma unroll
    for (int kc = 0; kc < K; ++kc) {
      Acc<MODE> a;
#pragma unroll
      for (int j = 0; j < B; ++j) a.fma(emb.P[j][kc], w[j]);
      out[kc] = (S)(a.result() * back);
    }
  }
}

// -------------------------------------------------- prolongation (+ add)
// fine += P (x) P (x) P e on every coarse cell, x first (multigrid.py:128-143, 252)
template <int K, int MODE>
__global__ void __launch_bounds__(kThreads) k_prolong_add(const typename MT<MODE>::S* __restrict__ ec,
                                                          typename MT<MODE>::S* __restrict__ fine, int ncx, int ncy,
                                                          int ncz, Embed<K, MODE> emb) {
  constexpr int TPC = Tpc<K>::value;
  constexpr int B = 2 * K, P = B + 1, VOL = B * B * P;
  constexpr bool kHalf = MT<MODE>::kHalf;
  using C = typename MT<MODE>::C;
  using S = typename MT<MODE>::S;
  extern __shared__ __align__(16) char smem[];
  C* s = reinterpret_cast<C*>(smem);
  int* s_exp = reinterpret_cast<int*>(s + TPC * VOL);
  long long syc = (long long)ncx * K, szc = syc * (long long)ncy * K;
  long long syf = 2 * syc, szf = syf * 2LL * ncy * K;
  int ncell = ncx * ncy * ncz;
  auto cell = [&](int t, int& x, int& y, int& z) {
    int id = blockIdx.x * TPC + t;
    if (id >= ncell) return false;
    x = id % ncx; y = (id / ncx) % ncy; z = id / (ncx * ncy);
    return true;
  };
  if (threadIdx.x == 0) s_exp[0] = 0;
  __syncthreads();
  // x lines straight from global: (t, zc, yc) -> B values along fine x (one line per thread)
  const int i = threadIdx.x;
  const int yc = i % K, zc = (i / K) % K, t0 = i / (K * K);
  int cx = 0, cy = 0, cz = 0;
  const bool act = i < TPC * K * K && cell(t0, cx, cy, cz);
  C in[K];
  if (act) {
    const S* src = ec + (long long)(cz * K + zc) * szc + (long long)(cy * K + yc) * syc + cx * K;
#pragma unroll
    for (int j = 0; j < K; ++j) {
      in[j] = (C)src[j];
      if constexpr (kHalf) smax(&s_exp[0], (float)in[j]);
    }
  }
  __syncthreads();
  const int ee = kHalf ? block_exp(__int_as_float(s_exp[0])) : 0;
  if (act) {
    const C sc = kHalf ? (C)pow2f(ee) : C(1);
    Op<MODE> w[K];
#pragma unroll
    for (int j = 0; j < K; ++j) w[j] = prep<MODE>(in[j] * sc);
    C* row = s + t0 * VOL + (zc * B + yc) * P;
#pragma unroll
    for (int o = 0; o < B; ++o) {
      Acc<MODE> a;
#pragma unroll
      for (int j = 0; j < K; ++j) a.fma(emb.P[o][j], w[j]);
      row[o] = a.result();
    }
  }
  __syncthreads();
  // y lines: (t, zc, x) K -> B
  for (int j2 = threadIdx.x; j2 < TPC * K * B; j2 += blockDim.x) {
    int xf = j2 % B, zz = (j2 / B) % K, t = j2 / (K * B);
    int ax, ay, az;
    if (!cell(t, ax, ay, az)) continue;
    C* col = s + t * VOL + (zz * B) * P + xf;
    Op<MODE> w[K];
#pragma unroll
    for (int j = 0; j < K; ++j) w[j] = prep<MODE>(col[j * P]);
#pragma unroll
    for (int o = 0; o < B; ++o) {
      Acc<MODE> a;
#pragma unroll
      for (int j = 0; j < K; ++j) a.fma(emb.P[o][j], w[j]);
      col[o * P] = a.result();
    }
  }
  __syncthreads();
  const C back = kHalf ? (C)pow2f(-ee) : C(1);
  // z lines: (t, y, x) K -> B, added into the fine vector; one work item per (column, group of HB outputs).
  // An item's HB fine values are all in flight before its first store (a read-modify-write loop would serialise
  // into dependent DRAM round trips: the compiler cannot hoist a load above a store to the same array).  fp64
  // takes all B per item (measured fastest); the fp32-storage modes split the column in two (register budget).
  constexpr int HB = MODE == MODE_FP64 ? B : K, NH = B / HB;
  for (int j2 = threadIdx.x; j2 < NH * TPC * B * B; j2 += blockDim.x) {
    const int h = j2 / (TPC * B * B);
    const int jj = j2 - h * (TPC * B * B);
    int xf = jj % B, yf = (jj / B) % B, t = jj / (B * B);
    int ax, ay, az;
    if (!cell(t, ax, ay, az)) continue;
    const C* col = s + t * VOL + yf * P + xf;
    Op<MODE> w[K];
#pragma unroll
    for (int j = 0; j < K; ++j) w[j] = prep<MODE>(col[j * B * P]);
    S* out = fine + (long long)(2 * az * K + h * HB) * szf + (long long)(2 * ay * K + yf) * syf + (2 * ax * K + xf);
    auto group = [&](auto O0) {  // compile-time output offset: constant indices into the embedding
      constexpr int oc = decltype(O0)::value;
      C old[HB];
#pragma unroll
      for (int o = 0; o < HB; ++o) old[o] = (C)out[o * szf];
#pragma unroll
      for (int o = 0; o < HB; ++o) {
        Acc<MODE> a;
#pragma unroll
        for (int j = 0; j < K; ++j) a.fma(emb.P[oc + o][j], w[j]);
        out[o * szf] = (S)(old[o] + a.result() * back);
      }
    };
    if constexpr (NH == 1) group(std::integral_constant<int, 0>{});
    else if (h == 0) group(std::integral_constant<int, 0>{});
    else group(std::integral_constant<int, B - HB>{});
  }
}

// ------------------------------------------- standalone patch inverse (batch)
// out = (V_z (x) V_y (x) V_x) diag(1/(lam_z+lam_y+lam_x)) (V_z^T (x) V_y^T (x) V_x^T) in
// on `count` contiguous (2K)^3 patches sharing one kind per axis, x first in
// both sweeps -- PatchSolver.apply_batch (multigrid.py:71-83).
template <int K, int MODE>
__global__ void __launch_bounds__(kThreads) k_patch_apply(const typename MT<MODE>::S* __restrict__ in,
                                                          typename MT<MODE>::S* __restrict__ out, int count, int kx,
                                                          int ky, int kz, PatchEig<K, MODE> eig, Scales sc) {
  constexpr int TPC = Tpc<K>::value;
  constexpr int B = 2 * K, P = B + 1, VOL = B * B * P;
  constexpr bool kHalf = MT<MODE>::kHalf;
  using C = typename MT<MODE>::C;
  using S = typename MT<MODE>::S;
  extern __shared__ __align__(16) char smem[];
  C* s = reinterpret_cast<C*>(smem);
  int* s_exp = reinterpret_cast<int*>(s + TPC * VOL);
  const long long pvol = (long long)B * B * B;
  if (threadIdx.x == 0) s_exp[0] = 0;
  __syncthreads();
  for (int i = threadIdx.x; i < TPC * B * B * B; i += blockDim.x) {
    int t = i / (B * B * B), r = i % (B * B * B);
    int id = blockIdx.x * TPC + t;
    const C v = id < count ? (C)in[id * pvol + r] : C(0);
    s[t * VOL + (r / B) * P + r % B] = v;
    if constexpr (kHalf) smax(&s_exp[0], (float)v);
  }
  __syncthreads();
  const int ee = kHalf ? block_exp(__int_as_float(s_exp[0])) : 0;
  const C s_in = kHalf ? (C)pow2f(ee) : C(1);
  const ME<MODE>* Vx = &eig.V[kx][0][0];
  const ME<MODE>* Vy = &eig.V[ky][0][0];
  const ME<MODE>* Vz = &eig.V[kz][0][0];
  for (int pass = 0; pass < 2; ++pass) {
    // x lines
    for (int i = threadIdx.x; i < TPC * B * B; i += blockDim.x) {
      int y = i % B, z = (i / B) % B, t = i / (B * B);
      C* row = s + t * VOL + (z * B + y) * P;
      Op<MODE> w[B];
#pragma unroll
      for (int x = 0; x < B; ++x) w[x] = prep<MODE>(pass == 0 ? row[x] * s_in : row[x]);
      Acc<MODE> acc[B];
      if (pass == 0) full_line<B, MODE, true>(Vx, w, acc); else full_line<B, MODE, false>(Vx, w, acc);
#pragma unroll
      for (int x = 0; x < B; ++x) row[x] = acc[x].result();
    }
    __syncthreads();
    for (int i = threadIdx.x; i < TPC * B * B; i += blockDim.x) {
      int x = i % B, z = (i / B) % B, t = i / (B * B);
      C* col = s + t * VOL + (z * B) * P + x;
      Op<MODE> w[B];
#pragma unroll
      for (int y = 0; y < B; ++y) w[y] = prep<MODE>(col[y * P]);
      Acc<MODE> acc[B];
      if (pass == 0) full_line<B, MODE, true>(Vy, w, acc); else full_line<B, MODE, false>(Vy, w, acc);
#pragma unroll
      for (int y = 0; y < B; ++y) col[y * P] = acc[y].result();
    }
    __syncthreads();
    for (int i = threadIdx.x; i < TPC * B * B; i += blockDim.x) {
      int x = i % B, y = (i / B) % B, t = i / (B * B);
      C* col = s + t * VOL + y * P + x;
      Op<MODE> w[B];
#pragma unroll
      for (int z = 0; z < B; ++z) w[z] = prep<MODE>(col[z * B * P]);
      Acc<MODE> acc[B];
      if (pass == 0) full_line<B, MODE, true>(Vz, w, acc); else full_line<B, MODE, false>(Vz, w, acc);
      if (pass == 0) {
        // lambda_sum over block axes (z, y, x) in fp64, cast, then divide (multigrid.py:60-69, 79-80)
#pragma unroll
        for (int z = 0; z < B; ++z)
          col[z * B * P] =
              acc[z].result() / lam_div<MODE>(((0.0 + eig.lam[kz][z]) + eig.lam[ky][y]) + eig.lam[kx][x], sc);
      } else {
#pragma unroll
        for (int z = 0; z < B; ++z) col[z * B * P] = acc[z].result();
      }
    }
    __syncthreads();
  }
  const C cs = corr_scale<MODE>(sc, ee);
  for (int i = threadIdx.x; i < TPC * B * B * B; i += blockDim.x) {
    int t = i / (B * B * B), r = i % (B * B * B);
    int id = blockIdx.x * TPC + t;
    if (id < count) out[id * pvol + r] = (S)(s[t * VOL + (r / B) * P + r % B] * cs);
  }
}

// ===================================================================== host

static thread_local char g_err[512] = "";

static int fail(int code, const char* fmt, const char* detail = "") {
  snprintf(g_err, sizeof(g_err), fmt, detail);
  return code;
}

static int check_launch(const char* what) {
  cudaError_t err = cudaGetLastError();
  if (err != cudaSuccess) {
    snprintf(g_err, sizeof(g_err), "%s: %s", what, cudaGetErrorString(err));
    return SF_ECUDA;
  }
  return SF_OK;
}

template <int MODE>
static ME<MODE> pack(double x) {
  ME<MODE> m;
  if constexpr (MODE == MODE_FP64) {
    m.h = x;
  } else if constexpr (MODE == MODE_FP32) {
    m.h = (float)x;
  } else if constexpr (MODE == MODE_FP16) {
    m.h = __half2float(__float2half_rn((float)x));
  } else {
    float x32 = (float)x;
    float h = __half2float(__float2half_rn(x32));
    m.h = h;
    m.d = __half2float(__float2half_rn((x32 - h) * kEcScale));
  }
  return m;
}

// level operator layout (host doubles): M[K*K], D[K*K], ucol[K], urow[K], bl[K], br[K]
template <int K, int MODE>
static LevelOp<K, MODE> pack_op(const double* src) {
  LevelOp<K, MODE> op;
  for (int i = 0; i < K; ++i)
    for (int j = 0; j < K; ++j) {
      op.M[i][j] = pack<MODE>(src[i * K + j]);
      op.D[i][j] = pack<MODE>(src[K * K + i * K + j]);
    }
  const double* v = src + 2 * K * K;
  for (int i = 0; i < K; ++i) {
    op.ucol[i] = pack<MODE>(v[i]);
    op.urow[i] = pack<MODE>(v[K + i]);
    op.bl[i] = pack<MODE>(v[2 * K + i]);
    op.br[i] = pack<MODE>(v[3 * K + i]);
  }
  return op;
}

// eigen layout: V[4][2K][2K] then lam[4][2K]
template <int K, int MODE>
static PatchEig<K, MODE> pack_eig(const double* src) {
  PatchEig<K, MODE> e;
  constexpr int B = 2 * K;
  for (int q = 0; q < 4; ++q)
    for (int i = 0; i < B; ++i)
      for (int j = 0; j < B; ++j) e.V[q][i][j] = pack<MODE>(src[(q * B + i) * B + j]);
  for (int q = 0; q < 4; ++q)
    for (int i = 0; i < B; ++i) e.lam[q][i] = src[4 * B * B + q * B + i];
  return e;
}

template <int K, int MODE>
static Embed<K, MODE> pack_emb(const double* src) {
  Embed<K, MODE> e;
  for (int i = 0; i < 2 * K; ++i)
    for (int j = 0; j < K; ++j) e.P[i][j] = pack<MODE>(src[i * K + j]);
  return e;
}

static int make_geom(const sf_grid* gr, int k, int shift_x, int shift_y, int shift_z, Geom& g) {
  if (!gr) return fail(SF_EINVAL, "null grid");
  if (gr->nx < 2 || gr->ny < 2 || gr->nz < 2 || (gr->nx & 1) || (gr->ny & 1) || (gr->nz & 1))
    return fail(SF_EINVAL, "cell counts must be even and >= 2");
  g.nx = gr->nx; g.ny = gr->ny; g.nz = gr->nz;
  g.tx0 = shift_x; g.ty0 = shift_y; g.tz0 = shift_z;
  g.ntx = gr->nx / 2 - shift_x; g.nty = gr->ny / 2 - shift_y; g.ntz = gr->nz / 2 - shift_z;
  g.bnd_lo[0] = g.bnd_hi[0] = 1;
  g.bnd_lo[1] = g.bnd_hi[1] = 1;
  g.bnd_lo[2] = gr->ghost_lo ? 0 : 1;
  g.bnd_hi[2] = gr->ghost_hi ? 0 : 1;
  g.ghost_lo = gr->ghost_lo;
  g.ghost_hi = gr->ghost_hi;
  g.batch_stride = (long long)gr->nx * gr->ny * gr->nz * (long long)k * k * k;
  (void)k;
  return SF_OK;
}

template <typename F>
static int set_smem(F* kern, size_t bytes) {
  static_assert(std::is_function<F>::value, "kernel");
  cudaError_t err = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
  if (err != cudaSuccess) {
    snprintf(g_err, sizeof(g_err), "cudaFuncSetAttribute: %s", cudaGetErrorString(err));
    return SF_ECUDA;
  }
  return SF_OK;
}

// SUMFACT_B200_GENERIC=1 forces the CUDA-core tile engine (A/B testing of the tensor-core paths)
static bool use_generic() {
  static int v = [] {
    const char* e = getenv("SUMFACT_B200_GENERIC");
    return (e && *e && *e != '0') ? 1 : 0;
  }();
  return v != 0;
}

template <int K, int MODE>
static int launch_vmult(const sf_grid* gr, const double* opd, const void* u, void* v, int batch, cudaStream_t st,
                        int z0 = 0, int z1 = -1) {
  Geom g;
  int rc = make_geom(gr, K, 0, 0, 0, g);
  if (rc) return rc;
  if (z1 >= 0) {  // tiles of the z-cell range [z0, z1) only (interior / boundary split of a slab)
    g.tz0 = z0;
    g.ntz = (z1 - z0) / 2;
  }
  if constexpr (K == 8 && (MODE == MODE_FP64 || MODE == MODE_FP32)) {
    if (!use_generic()) {
      const int r = launch_vmult_dmma8(g, opd, u, v, batch, st, MODE == MODE_FP32);
      if (r != kUseGeneric) {  // (declined: local array too large for 32-bit tile offsets)
        if (r) return check_launch("sf_vmult (dmma)");
        return SF_OK;
      }
    }
  }
  if constexpr (K == 8 && (MODE == MODE_FP16 || MODE == MODE_FP16_EC)) {
    if (!use_generic()) {
      if (launch_vmult_hmma8(MODE, g, opd, u, v, batch, st)) return check_launch("sf_vmult (hmma)");
      return SF_OK;
    }
  }
  if constexpr ((K == 4 || K == 2) && (MODE == MODE_FP64 || MODE == MODE_FP32)) {
    if (!use_generic()) {
      const int r = launch_vmult_dmma_line(K, g, opd, u, v, batch, st, MODE == MODE_FP32);
      if (r != kUseGeneric) {
        if (r) return check_launch("sf_vmult (dmma line)");
        return SF_OK;
      }
    }
  }
  if constexpr ((K == 4 || K == 2) && (MODE == MODE_FP16 || MODE == MODE_FP16_EC)) {
    if (!use_generic()) {
      const int r = launch_vmult_hmma_line(MODE, K, g, opd, u, v, batch, st);
      if (r != kUseGeneric) {
        if (r) return check_launch("sf_vmult (hmma line)");
        return SF_OK;
      }
    }
  }
  constexpr int TPC = Tpc<K>::value;
  using E = TileEngine<K, MODE, TPC>;
  Prepared<K, MODE> pr(opd, nullptr);
  auto op = pack_op<K, MODE>(pr.opd);
  op.sc = pr.sc;
  size_t smem = E::smem_bytes();
  if ((rc = set_smem(k_vmult<K, MODE>, smem))) return rc;
  int tiles = g.ntx * g.nty * g.ntz;
  dim3 grid((tiles + TPC - 1) / TPC, batch);
  using S = typename MT<MODE>::S;
  k_vmult<K, MODE><<<grid, kThreads, smem, st>>>((const S*)u, (S*)v, g, op);
  return check_launch("sf_vmult");
}

template <int K, int MODE>
static int launch_colour(const sf_grid* gr, const int* shift, const double* opd, const double* eigd, const void* xo,
                         const void* b, void* xn, cudaStream_t st, int z0 = -1, int z1 = -1, bool copy = true) {
  Geom g;
  // shift[i] is tensor axis i (x = 0), multigrid.py:189-192
  int rc = make_geom(gr, K, shift[0], shift[1], shift[2], g);
  if (rc) return rc;
  constexpr int TPC = Tpc<K>::value;
  using E = TileEngine<K, MODE, TPC>;
  using S = typename MT<MODE>::S;
  if (z0 >= 0) {  // tiles whose first cell lies in [z0, z1) only (z-slab interior / boundary split)
    if (K != 8) return fail(SF_EUNSUPPORTED, "z-range colour passes are Q7 (2-cell tiles) only");
    if (z1 == z0) return SF_OK;
    g.tz0 = z0;
    g.ntz = (z1 - z0) / 2;
  }
  if (g.ntx < 1 || g.nty < 1 || g.ntz < 1) {
    if (!copy) return SF_OK;
    if (!xo) return fail(SF_EUNSUPPORTED, "zero-iterate colour pass on a grid without patches");
    // colour without patches: x_new = x_old
    size_t bytes = (size_t)gr->nx * gr->ny * gr->nz * K * K * K * sizeof(S);
    if (cudaMemcpyAsync(xn, xo, bytes, cudaMemcpyDeviceToDevice, st) != cudaSuccess)
      return check_launch("sf_smooth_colour copy");
    return SF_OK;
  }
  bool done = false;
  // the Q7 DMMA kernels copy the uncovered cells themselves (whole-grid launches only; fusing it into the binary16
  // kernel measured 5 % slower there, so those keep the separate copy)
  const bool fuse_copy = copy && z0 < 0 && (shift[0] || shift[1] || shift[2]);
  bool copied = false;
  if constexpr (K == 8 && (MODE == MODE_FP64 || MODE == MODE_FP32)) {
    if (!use_generic()) {
      const int r = launch_colour_dmma8(g, opd, eigd, xo, b, xn, st, MODE == MODE_FP32, fuse_copy);
      if (r != kUseGeneric) {
        if (r) return check_launch("sf_smooth_colour (dmma)");
        done = true;
        copied = fuse_copy;
      }
    }
  }
  if constexpr ((K == 4 || K == 2) && (MODE == MODE_FP64 || MODE == MODE_FP32)) {
    if (!use_generic()) {
      const int r = launch_colour_dmma_line(K, g, opd, eigd, xo, b, xn, st, MODE == MODE_FP32);
      if (r != kUseGeneric) {
        if (r) return check_launch("sf_smooth_colour (dmma line)");
        done = true;
      }
    }
  }
  if constexpr ((K == 4 || K == 2) && (MODE == MODE_FP16 || MODE == MODE_FP16_EC)) {
    if (!use_generic()) {
      const int r = launch_colour_hmma_line(MODE, K, g, opd, eigd, xo, b, xn, st);
      if (r != kUseGeneric) {
        if (r) return check_launch("sf_smooth_colour (hmma line)");
        done = true;
      }
    }
  }
  if constexpr (K == 8 && (MODE == MODE_FP16 || MODE == MODE_FP16_EC)) {
    if (!use_generic()) {
      if (launch_colour_hmma8(MODE, g, opd, eigd, xo, b, xn, st)) return check_launch("sf_smooth_colour (hmma)");
      done = true;
    }
  }
  if (!done) {
    if (!xo) return fail(SF_EUNSUPPORTED, "zero-iterate colour pass: this grid takes the generic kernel");
    Prepared<K, MODE> pr(opd, eigd);
    auto op = pack_op<K, MODE>(pr.opd);
    op.sc = pr.sc;
    auto eig = pack_eig<K, MODE>(pr.eigd);
    size_t smem = E::smem_bytes() + sizeof(ME<MODE>) * 4 * 4 * K * K + sizeof(double) * 8 * K;
    if ((rc = set_smem(k_colour<K, MODE>, smem))) return rc;
    int tiles = g.ntx * g.nty * g.ntz;
    k_colour<K, MODE><<<(tiles + TPC - 1) / TPC, kThreads, smem, st>>>((const S*)xo, (const S*)b, (S*)xn, g, op,
                                                                        eig);
    if ((rc = check_launch("sf_smooth_colour"))) return rc;
  }
  if (copy && !copied && (shift[0] || shift[1] || shift[2])) {
    copy_slabs<S>((const S*)xo, (S*)xn, K, gr, shift, st);
    return check_launch("sf_smooth_colour slabs");
  }
  return SF_OK;
}

template <int K, int MODE>
static int launch_copy_uncovered(const sf_grid* gr, const int* shift, const void* xo, void* xn, cudaStream_t st) {
  using S = typename MT<MODE>::S;
  if (!(shift[0] || shift[1] || shift[2])) return SF_OK;
  copy_slabs<S>((const S*)xo, (S*)xn, K, gr, shift, st);
  return check_launch("sf_copy_uncovered");
}

template <int K, int MODE>
static int launch_resid_restrict(const sf_grid* gr, const double* opd, const double* embd, const void* x,
                                 const void* b, void* coarse, int with_op, cudaStream_t st) {
  Geom g;
  int rc = make_geom(gr, K, 0, 0, 0, g);
  if (rc) return rc;
  if (gr->ghost_lo || gr->ghost_hi) {
    // restriction is slab-local (aligned tiles); ghosts only feed the operator
  }
  if constexpr ((K == 4 || K == 2) && (MODE == MODE_FP64 || MODE == MODE_FP32)) {
    if (with_op && !use_generic()) {
      const int r = launch_resid_restrict_dmma_line(K, g, opd, embd, x, b, coarse, st, MODE == MODE_FP32);
      if (r != kUseGeneric) {
        if (r) return check_launch("sf_residual_restrict (dmma line)");
        return SF_OK;
      }
    }
  }
  if constexpr ((K == 4 || K == 2) && (MODE == MODE_FP16 || MODE == MODE_FP16_EC)) {
    if (with_op && !use_generic()) {
      const int r = launch_resid_restrict_hmma_line(MODE, K, g, opd, embd, x, b, coarse, st);
      if (r != kUseGeneric) {
        if (r) return check_launch("sf_residual_restrict (hmma line)");
        return SF_OK;
      }
    }
  }
  if constexpr (K == 8 && (MODE == MODE_FP64 || MODE == MODE_FP32)) {
    if (with_op && !use_generic()) {
      const int r = launch_resid_restrict_dmma8(g, opd, embd, x, b, coarse, st, MODE == MODE_FP32);
      if (r != kUseGeneric) {
        if (r) return check_launch("sf_residual_restrict (dmma)");
        return SF_OK;
      }
    }
  }
  if constexpr (K == 8 && (MODE == MODE_FP16 || MODE == MODE_FP16_EC)) {
    if (with_op && !use_generic()) {
      if (launch_resid_restrict_hmma8(MODE, g, opd, embd, x, b, coarse, st))
        return check_launch("sf_residual_restrict (hmma)");
      return SF_OK;
    }
  }
  constexpr int TPC = Tpc<K>::value;
  using E = TileEngine<K, MODE, TPC>;
  using S = typename MT<MODE>::S;
  Prepared<K, MODE> pr(opd, nullptr);
  auto op = pack_op<K, MODE>(pr.opd);
  op.sc = pr.sc;
  auto emb = pack_emb<K, MODE>(embd);
  size_t smem = E::smem_bytes();
  if ((rc = set_smem(k_resid_restrict<K, MODE>, smem))) return rc;
  int tiles = g.ntx * g.nty * g.ntz;
  k_resid_restrict<K, MODE><<<(tiles + TPC - 1) / TPC, kThreads, smem, st>>>((const S*)x, (const S*)b, (S*)coarse,
                                                                              g, op, emb, with_op);
  return check_launch("sf_residual_restrict");
}

template <int K, int MODE>
static int launch_prolong_add(const sf_grid* coarse, const double* embd, const void* e, void* fine, cudaStream_t st) {
  if (!coarse || coarse->nx < 1 || coarse->ny < 1 || coarse->nz < 1) return fail(SF_EINVAL, "bad coarse grid");
  if constexpr ((K == 8 || K == 4 || K == 2) && (MODE == MODE_FP16 || MODE == MODE_FP16_EC)) {
    if (!use_generic()) {
      const int r = launch_prolong_hmma(MODE, K, coarse->nx, coarse->ny, coarse->nz, embd, e, fine, st);
      if (r != kUseGeneric) return r ? check_launch("sf_prolongate_add (hmma)") : SF_OK;
    }
  }
  if constexpr ((K == 8 || K == 4 || K == 2) && (MODE == MODE_FP64 || MODE == MODE_FP32)) {
    if (!use_generic()) {
      const int r = launch_prolong_dmma(K, coarse->nx, coarse->ny, coarse->nz, embd, e, fine, st, MODE == MODE_FP32);
      if (r != kUseGeneric) return r ? check_launch("sf_prolongate_add (dmma)") : SF_OK;
    }
  }
  constexpr int TPC = Tpc<K>::value;
  constexpr int B = 2 * K;
  using S = typename MT<MODE>::S;
  using C = typename MT<MODE>::C;
  auto emb = pack_emb<K, MODE>(embd);
  size_t smem = sizeof(C) * TPC * B * B * (B + 1) + 16;
  int rc;
  if ((rc = set_smem(k_prolong_add<K, MODE>, smem))) return rc;
  int cells = coarse->nx * coarse->ny * coarse->nz;
  k_prolong_add<K, MODE><<<(cells + TPC - 1) / TPC, kThreads, smem, st>>>((const S*)e, (S*)fine, coarse->nx,
                                                                           coarse->ny, coarse->nz, emb);
  return check_launch("sf_prolongate_add");
}

template <int K, int MODE>
static int launch_patch_apply(int count, const int* kinds, const double* eigd, const void* in, void* out,
                              cudaStream_t st) {
  constexpr int TPC = Tpc<K>::value;
  constexpr int B = 2 * K;
  using S = typename MT<MODE>::S;
  using C = typename MT<MODE>::C;
  Prepared<K, MODE> pr(nullptr, eigd);
  auto eig = pack_eig<K, MODE>(pr.eigd);
  size_t smem = sizeof(C) * TPC * B * B * (B + 1) + 16;
  int rc;
  if ((rc = set_smem(k_patch_apply<K, MODE>, smem))) return rc;
  k_patch_apply<K, MODE><<<(count + TPC - 1) / TPC, kThreads, smem, st>>>((const S*)in, (S*)out, count, kinds[0],
                                                                            kinds[1], kinds[2], eig, pr.sc);
  return check_launch("sf_patch_apply");
}

}  // namespace sf

// ----------------------------------------------------------------- C-ABI

using namespace sf;

#define SF_DISPATCH(k, mode, CALL)                                                   \
  do {                                                                               \
    switch ((k) * 4 + (mode)) {                                                      \
      case 1 * 4 + 0: return CALL(2, 0); case 1 * 4 + 1: return CALL(2, 1);          \
      case 1 * 4 + 2: return CALL(2, 2); case 1 * 4 + 3: return CALL(2, 3);          \
      case 2 * 4 + 0: return CALL(3, 0); case 2 * 4 + 1: return CALL(3, 1);          \
      case 2 * 4 + 2: return CALL(3, 2); case 2 * 4 + 3: return CALL(3, 3);          \
      case 3 * 4 + 0: return CALL(4, 0); case 3 * 4 + 1: return CALL(4, 1);          \
      case 3 * 4 + 2: return CALL(4, 2); case 3 * 4 + 3: return CALL(4, 3);          \
      case 4 * 4 + 0: return CALL(5, 0); case 4 * 4 + 1: return CALL(5, 1);          \
      case 4 * 4 + 2: return CALL(5, 2); case 4 * 4 + 3: return CALL(5, 3);          \
      case 5 * 4 + 0: return CALL(6, 0); case 5 * 4 + 1: return CALL(6, 1);          \
      case 5 * 4 + 2: return CALL(6, 2); case 5 * 4 + 3: return CALL(6, 3);          \
      case 6 * 4 + 0: return CALL(7, 0); case 6 * 4 + 1: return CALL(7, 1);          \
      case 6 * 4 + 2: return CALL(7, 2); case 6 * 4 + 3: return CALL(7, 3);          \
      case 7 * 4 + 0: return CALL(8, 0); case 7 * 4 + 1: return CALL(8, 1);          \
      case 7 * 4 + 2: return CALL(8, 2); case 7 * 4 + 3: return CALL(8, 3);          \
      default: return fail(SF_EUNSUPPORTED, "unsupported degree/mode%s", "");        \
    }                                                                                \
  } while (0)

static int check_common(int mode, int k) {
  g_err[0] = 0;  // every entry point starts here: no stale message survives a later failure
  if (mode < 0 || mode > 3) return fail(SF_EINVAL, "mode must be 0..3 (fp64, fp32, fp16, fp16_ec)");
  if (k < 1 || k > SF_MAX_DEGREE) return fail(SF_EUNSUPPORTED, "degree k must be in 1..7");
  return SF_OK;
}

// vectors are read with 16-byte vector loads / cp.async chunks: every vector pointer (and ghost plane) must be
// 16-byte aligned (cudaMalloc and torch allocations are 256-byte aligned)
static bool misaligned(const void* p) { return ((uintptr_t)p & 15) != 0; }
static bool misaligned_grid(const sf_grid* g) { return g && (misaligned(g->ghost_lo) || misaligned(g->ghost_hi)); }
#define SF_ALIGNED(...)                                                                      \
  do {                                                                                       \
    const void* ps_[] = {__VA_ARGS__};                                                       \
    for (const void* p_ : ps_)                                                               \
      if (misaligned(p_)) return fail(SF_EINVAL, "vectors must be 16-byte aligned");         \
  } while (0)

extern "C" {

int sf_abi_version(void) { return SF_ABI_VERSION; }

const char* sf_last_error(void) { return g_err; }

int sf_vmult(int mode, int k, const sf_grid* grid, const double* level_op, const void* u, void* v, int batch,
             void* stream) {
  int rc = check_common(mode, k);
  if (rc) return rc;
  if (!u || !v || !level_op) return fail(SF_EINVAL, "null pointer");
  SF_ALIGNED(u, v);
  if (misaligned_grid(grid)) return fail(SF_EINVAL, "ghost planes must be 16-byte aligned");
  if (batch < 1) return fail(SF_EINVAL, "batch must be >= 1");
  cudaStream_t st = (cudaStream_t)stream;
#define CALL(K, M) launch_vmult<K, M>(grid, level_op, u, v, batch, st)
  SF_DISPATCH(k, mode, CALL);
#undef CALL
}

int sf_vmult_zrange(int mode, int k, const sf_grid* grid, int z0, int z1, const double* level_op, const void* u,
                    void* v, void* stream) {
  int rc = check_common(mode, k);
  if (rc) return rc;
  if (!u || !v || !level_op || !grid) return fail(SF_EINVAL, "null pointer");
  SF_ALIGNED(u, v);
  if (misaligned_grid(grid)) return fail(SF_EINVAL, "ghost planes must be 16-byte aligned");
  if (z0 < 0 || z1 > grid->nz || z0 >= z1 || (z0 & 1) || (z1 & 1))
    return fail(SF_EINVAL, "z range must be an even, non-empty subrange of [0, nz)");
  cudaStream_t st = (cudaStream_t)stream;
#define CALL(K, M) launch_vmult<K, M>(grid, level_op, u, v, 1, st, z0, z1)
  SF_DISPATCH(k, mode, CALL);
#undef CALL
}

int sf_smooth_colour(int mode, int k, const sf_grid* grid, const int* shift, const double* level_op,
                     const double* patch_eig, const void* x_old, const void* b, void* x_new, void* stream) {
  int rc = check_common(mode, k);
  if (rc) return rc;
  if (!shift || !b || !x_new || !level_op || !patch_eig) return fail(SF_EINVAL, "null pointer");
  SF_ALIGNED(x_old, b, x_new);
  if (misaligned_grid(grid)) return fail(SF_EINVAL, "ghost planes must be 16-byte aligned");
  for (int i = 0; i < 3; ++i)
    if (shift[i] != 0 && shift[i] != 1) return fail(SF_EINVAL, "shift entries must be 0 or 1");
  if (x_old == x_new) return fail(SF_EINVAL, "x_old and x_new must be distinct buffers");
  if (!x_old) {  // zero current iterate: only the unshifted colour (every cell covered), only the tensor-core paths
    if (shift[0] || shift[1] || shift[2]) return fail(SF_EINVAL, "x_old may be NULL only for the unshifted colour");
    if (!(k == 7 || k == 3 || k == 1) || use_generic())
      return fail(SF_EUNSUPPORTED, "zero-iterate colour pass: Q7 / Q3 / Q1 tensor-core kernels only");
  }
  cudaStream_t st = (cudaStream_t)stream;
#define CALL(K, M) launch_colour<K, M>(grid, shift, level_op, patch_eig, x_old, b, x_new, st)
  SF_DISPATCH(k, mode, CALL);
#undef CALL
}

int sf_smooth_colour_zrange(int mode, int k, const sf_grid* grid, const int* shift, int z0, int z1,
                            const double* level_op, const double* patch_eig, const void* x_old, const void* b,
                            void* x_new, void* stream) {
  int rc = check_common(mode, k);
  if (rc) return rc;
  if (!grid || !shift || !x_old || !b || !x_new || !level_op || !patch_eig) return fail(SF_EINVAL, "null pointer");
  SF_ALIGNED(x_old, b, x_new);
  if (misaligned_grid(grid)) return fail(SF_EINVAL, "ghost planes must be 16-byte aligned");
  for (int i = 0; i < 3; ++i)
    if (shift[i] != 0 && shift[i] != 1) return fail(SF_EINVAL, "shift entries must be 0 or 1");
  if (x_old == x_new) return fail(SF_EINVAL, "x_old and x_new must be distinct buffers");
  if (z0 < shift[2] || z1 < z0 || z1 > grid->nz || ((z0 - shift[2]) & 1) || ((z1 - z0) & 1) ||
      z1 > grid->nz - (shift[2] ? 1 : 0))
    return fail(SF_EINVAL, "z range must start on a tile of the colour and hold whole 2-cell tiles");
  cudaStream_t st = (cudaStream_t)stream;
#define CALL(K, M) launch_colour<K, M>(grid, shift, level_op, patch_eig, x_old, b, x_new, st, z0, z1, false)
  SF_DISPATCH(k, mode, CALL);
#undef CALL
}

int sf_copy_uncovered(int mode, int k, const sf_grid* grid, const int* shift, const void* x_old, void* x_new,
                      void* stream) {
  int rc = check_common(mode, k);
  if (rc) return rc;
  if (!grid || !shift || !x_old || !x_new) return fail(SF_EINVAL, "null pointer");
  for (int i = 0; i < 3; ++i)
    if (shift[i] != 0 && shift[i] != 1) return fail(SF_EINVAL, "shift entries must be 0 or 1");
  cudaStream_t st = (cudaStream_t)stream;
#define CALL(K, M) launch_copy_uncovered<K, M>(grid, shift, x_old, x_new, st)
  SF_DISPATCH(k, mode, CALL);
#undef CALL
}

int sf_residual_restrict(int mode, int k, const sf_grid* fine_grid, const double* level_op, const double* embedding,
                         const void* x, const void* b, void* coarse, void* stream) {
  int rc = check_common(mode, k);
  if (rc) return rc;
  if (!b || !coarse || !embedding) return fail(SF_EINVAL, "null pointer");
  SF_ALIGNED(x, b, coarse);
  if (misaligned_grid(fine_grid)) return fail(SF_EINVAL, "ghost planes must be 16-byte aligned");
  int with_op = x != nullptr;
  if (with_op && !level_op) return fail(SF_EINVAL, "level_op required with x");
  cudaStream_t st = (cudaStream_t)stream;
  static const double zeros[4 * 8 * 8] = {0};
  const double* opd = with_op ? level_op : zeros;
#define CALL(K, M) launch_resid_restrict<K, M>(fine_grid, opd, embedding, x, b, coarse, with_op, st)
  SF_DISPATCH(k, mode, CALL);
#undef CALL
}

int sf_prolongate_add(int mode, int k, const sf_grid* coarse_grid, const double* embedding, const void* e,
                      void* fine, void* stream) {
  int rc = check_common(mode, k);
  if (rc) return rc;
  if (!e || !fine || !embedding) return fail(SF_EINVAL, "null pointer");
  SF_ALIGNED(e, fine);
  cudaStream_t st = (cudaStream_t)stream;
#define CALL(K, M) launch_prolong_add<K, M>(coarse_grid, embedding, e, fine, st)
  SF_DISPATCH(k, mode, CALL);
#undef CALL
}

int sf_patch_apply(int mode, int k, long long count, const int* kinds, const double* patch_eig, const void* in,
                   void* out, void* stream) {
  int rc = check_common(mode, k);
  if (rc) return rc;
  if (!kinds || !patch_eig || (count > 0 && (!in || !out))) return fail(SF_EINVAL, "null pointer");
  if (count < 0 || count > (1LL << 30)) return fail(SF_EINVAL, "bad patch count");
  for (int i = 0; i < 3; ++i)
    if (kinds[i] < 0 || kinds[i] > 3) return fail(SF_EINVAL, "kind must be 0..3");
  if (count == 0) return SF_OK;
  cudaStream_t st = (cudaStream_t)stream;
#define CALL(K, M) launch_patch_apply<K, M>((int)count, kinds, patch_eig, in, out, st)
  SF_DISPATCH(k, mode, CALL);
#undef CALL
}

}  // extern "C"
