// FP64 Q7 kernels on the tensor cores (DMMA).  See sf_dmma.cuh for the
// schedule and the shared-memory layouts.
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>
#include <mutex>
#include <type_traits>
#include <vector>

#include "sf_dmma.cuh"
#include "sf_internal.h"

namespace sf {
namespace dm {
// prologue_fast addresses with 32-bit element offsets: 24 planes of the local array must fit
static bool offsets32(const Geom& g) {
  return 24LL * g.nx * g.ny * K * K < 2147483647LL;
}

// FP32 mode on the DMMA kernels: the operator data is demoted to fp32 values (as the reference's
// contract_mode casts its matrices, precision.py:206-230) and stays fp64-typed in the tables.
static const double* demote32(std::vector<double>& buf, const double* p, size_t n) {
  buf.assign(p, p + n);
  for (double& x : buf) x = (double)(float)x;
  return buf.data();
}
static size_t op_len(int K) { return 2 * K * K + 4 * K; }
static size_t eig_len(int K) { return 16 * K * K + 8 * K; }
static bool aligned16(const void* p) { return ((uintptr_t)p & 15) == 0; }

struct PatchL {
  double L[4][B][B];  // L_smooth[kind], kind = 2*left_bnd + right_bnd
};

// L_smooth[(lb,rb)] = [[D + lb*Bl, U], [U^T, D + rb*Br]] rebuilt from the cell-wise blocks
static PatchL build_patch_l(const double* opd) {
  const double* D = opd + K * K;
  const double* ucol = opd + 2 * K * K;
  const double* urow = ucol + K;
  const double* bl = urow + K;
  const double* br = bl + K;
  PatchL p;
  for (int q = 0; q < 4; ++q) {
    const int lb = q >> 1, rb = q & 1;
    for (int i = 0; i < B; ++i)
      for (int j = 0; j < B; ++j) p.L[q][i][j] = 0.0;
    for (int c = 0; c < 2; ++c)
      for (int i = 0; i < K; ++i)
        for (int j = 0; j < K; ++j) p.L[q][c * K + i][c * K + j] = D[i * K + j];
    for (int i = 0; i < K; ++i) {
      p.L[q][i][K] = ucol[i];          // U column 0
      p.L[q][K - 1][K + i] = urow[i];  // U row K-1
      p.L[q][K][i] = ucol[i];          // U^T row 0
      p.L[q][K + i][K - 1] = urow[i];  // U^T column K-1
    }
    if (lb)
      for (int i = 0; i < K; ++i) {
        p.L[q][i][0] += bl[i];
        if (i > 0) p.L[q][0][i] += bl[i];
      }
    if (rb)
      for (int i = 0; i < K; ++i) {
        p.L[q][K + i][B - 1] += br[i];
        if (i < K - 1) p.L[q][B - 1][K + i] += br[i];
      }
  }
  return p;
}

template <int K = 8>
static LevelOp<K, MODE_FP64> pack_op64(const double* opd) {
  LevelOp<K, MODE_FP64> op;
  for (int i = 0; i < K; ++i)
    for (int j = 0; j < K; ++j) {
      op.M[i][j].h = opd[i * K + j];
      op.D[i][j].h = opd[K * K + i * K + j];
    }
  const double* vv = opd + 2 * K * K;
  for (int i = 0; i < K; ++i) {
    op.ucol[i].h = vv[i];
    op.urow[i].h = vv[K + i];
    op.bl[i].h = vv[2 * K + i];
    op.br[i].h = vv[3 * K + i];
  }
  return op;
}

// ---------------------------------------------------------------------------
// Device-resident operator fragment tables of one level (fp64, K = 8).
// Fragment slot fr = 4*nb + kc of lane ln holds B[k][n] = Op[8nb + (ln>>2)][k-index]:
//   std : k-index = 4kc + (ln&3)             (A fragment loaded from shared memory)
//   perm: k-index = 8(kc>>1) + 2(ln&3) + (kc&1)  (A fragment = the previous C fragment,
//         so two contractions along the same axis chain in registers)
struct Tables8 {
  double L[4][8][32];    // L_smooth[kind], std
  double Vf[4][8][32];   // Op = V^T (forward transform), std
  double Vfp[4][8][32];  // Op = V^T, perm
  double Vb[4][8][32];   // Op = V (backward transform), std
  double Vbp[4][8][32];  // Op = V, perm
  double lam[4][16];     // generalised eigenvalues per kind
};

template <class S>
__global__ void __launch_bounds__(kThreads, 2) k_vmult_dmma8(const S* __restrict__ u, S* __restrict__ v,
                                                            Geom g, LevelOp<K, MODE_FP64> op,
                                                            const Tables8* __restrict__ tab, Band bd, int prefetch) {
  extern __shared__ __align__(128) double smem[];
  Tile T;
  int batch;
  if (!tile_setup_band(T, smem, g, bd, batch)) return;
  u += (long long)batch * g.batch_stride;
  v += (long long)batch * g.batch_stride;
  if (prefetch) prefetch_ahead_l2(g, bd, T, u);
  Frags f;
  Halo h;
  init_frags(T, op, f, h);
  prologue_fast(T, g, op, u, f, &tab->L[0][0][0]);  // L fragments staged into smem (T.sLf)
  xy_stages<S>(T, f, h);
  __syncthreads();
  load_l(T, f, T.kind[2]);
  S* vb = v + (long long)(T.cz * K) * T.sz + (long long)(T.cy * K) * T.sy + T.cx * K;
  for (int yy = 0; yy < 2; ++yy) {
    const int y = 2 * T.warp + yy;
#pragma unroll
    for (int g8 = 0; g8 < 2; ++g8) {
      double acc[2][2];
      z_group(T, f, h, y, 8 * g8, acc);
      const int x = 8 * g8 + T.r;
#pragma unroll
      for (int nb = 0; nb < 2; ++nb)
#pragma unroll
        for (int i = 0; i < 2; ++i) vb[(long long)(8 * nb + T.c2 + i) * T.sz + (long long)y * T.sy + x] = (S)acc[nb][i];
    }
  }
}





__device__ __forceinline__ void load_frag(const double* tab /* [8][32] */, double (*l)[4], int lane) {
#pragma unroll
  for (int nb = 0; nb < 2; ++nb)
#pragma unroll
    for (int kc = 0; kc < 4; ++kc) l[nb][kc] = __ldg(tab + (nb * 4 + kc) * 32 + lane);
}

// acc += A . Op^T with 16 inputs (4 k-chunks) and 16 outputs (2 n-blocks)
__device__ __forceinline__ void full_group(const double (*l)[4], const double* a, double (*acc)[2]) {
#pragma unroll
  for (int kc = 0; kc < 4; ++kc)
#pragma unroll
    for (int nb = 0; nb < 2; ++nb) dmma(acc[nb][0], acc[nb][1], a[kc], l[nb][kc]);
}

// One colour of the vertex-patch smoother on DMMA (multigrid.py:186-203): per
// patch tile r = b - A x_old, x_new = x_old + (V_z V_y V_x) Lambda^-1 (V_x^T V_y^T V_z^T) r.
// Stage order: residual z-lines -> V_z^T (registers) | V_y^T | V_x^T, 1/lambda,
// V_x (registers) | V_y | V_z -> +x_old -> HBM; '|' = shared-memory transpose.
// KK = 8: one patch per tile line; KK = 4 / 2: a 16-point line holds 2 / 4 patches and the
// transforms are blockdiag(V_patch) (line tables built per line boundary kind).
// XZ: zero current iterate (x_old = NULL: the first, unshifted colour of a V-cycle's pre-smoothing): r = b, the
// operator stages and the x_old reads are skipped; bitwise the full pass on a zero vector.
template <int KK = 8, class S = double, bool XZ = false>
__global__ void __launch_bounds__(kThreads, 2) k_colour_dmma(const S* __restrict__ xo,
                                                            const S* __restrict__ b, S* __restrict__ xn,
                                                            Geom g, LevelOp<KK, MODE_FP64> op,
                                                            const Tables8* __restrict__ tab, Band bd,
                                                            int copy_unc = 0) {
  extern __shared__ __align__(128) double smem[];
  Tile T;
  int batch;
  if (!tile_setup_band<KK>(T, smem, g, bd, batch)) return;
  if constexpr (KK == 8 && !XZ) {
    if (copy_unc) copy_uncovered_ext<S, kThreads>(g, T.cx, T.cy, T.cz, xo, xn);
  }
  Frags f;
  Halo h;
  if constexpr (!XZ) {
    prefetch_tile_rows_l2<KK>(T, b);
    prefetch_ahead_l2<KK>(g, bd, T, xo);
    init_frags<KK>(T, op, f, h);
    prologue_fast<KK>(T, g, op, xo, f, &tab->L[0][0][0]);  // L fragments staged into smem (T.sLf)
    xy_stages<S, KK>(T, f, h);
    __syncthreads();
  }
  const int lane = T.lane, r = T.r, c2 = T.c2, w = T.warp;
  const int kx = T.kind[0], ky = T.kind[1], kz = T.kind[2];
  const long long off0 = (long long)(T.cz * KK) * T.sz + (long long)(T.cy * KK) * T.sy + T.cx * KK;
  double V[2][4];
  // ---- z lines: residual and forward V_z^T (chained in registers), out in T layout
  if constexpr (!XZ) load_l(T, f, kz);
  load_frag(&tab->Vfp[kz][0][0], V, lane);
  {
    double t[2][2][2][2];
#pragma unroll
    for (int yy = 0; yy < 2; ++yy) {
      const int y = 2 * w + yy;
#pragma unroll
      for (int g8 = 0; g8 < 2; ++g8) {
        double acc[2][2] = {{0.0, 0.0}, {0.0, 0.0}};
        if constexpr (!XZ) z_group(T, f, h, y, 8 * g8, acc);
        const int x = 8 * g8 + r;
        double a[4];
#pragma unroll
        for (int kc = 0; kc < 4; ++kc) {
          const int z = 8 * (kc >> 1) + c2 + (kc & 1);
          a[kc] = rd<S>((double)__ldg(b + off0 + (long long)z * T.sz + (long long)y * T.sy + x) - acc[kc >> 1][kc & 1]);
        }
        double (*o)[2] = t[yy][g8];
        o[0][0] = o[0][1] = o[1][0] = o[1][1] = 0.0;
        full_group(V, a, o);
      }
    }
    __syncwarp();
#pragma unroll
    for (int yy = 0; yy < 2; ++yy)
#pragma unroll
      for (int g8 = 0; g8 < 2; ++g8)
#pragma unroll
        for (int nb = 0; nb < 2; ++nb)
#pragma unroll
          for (int i = 0; i < 2; ++i) T.sU[idxT(8 * nb + c2 + i, 2 * w + yy, 8 * g8 + r)] = rd<S>(t[yy][g8][nb][i]);
  }
  __syncthreads();
  // ---- warp-private z' planes: V_y^T | V_x^T, 1/lambda, V_x | V_y
  const double* lamx = tab->lam[kx];
  const double* lamy = tab->lam[ky];
  const double* lamz = tab->lam[kz];
  for (int zz = 0; zz < 2; ++zz) {
    const int z = 2 * w + zz;
    double o[2][2][2];
    load_frag(&tab->Vf[ky][0][0], V, lane);
#pragma unroll
    for (int g8 = 0; g8 < 2; ++g8) {
      const int x = 8 * g8 + r;
      double a[4];
#pragma unroll
      for (int kc = 0; kc < 4; ++kc) a[kc] = T.sU[idxT(z, 4 * kc + T.k4, x)];
      o[g8][0][0] = o[g8][0][1] = o[g8][1][0] = o[g8][1][1] = 0.0;
      full_group(V, a, o[g8]);
    }
    __syncwarp();
#pragma unroll
    for (int g8 = 0; g8 < 2; ++g8)
#pragma unroll
      for (int nb = 0; nb < 2; ++nb)
#pragma unroll
        for (int i = 0; i < 2; ++i) T.sU[idxG(z, 8 * nb + c2 + i, 8 * g8 + r)] = rd<S>(o[g8][nb][i]);
    __syncwarp();
    load_frag(&tab->Vf[kx][0][0], V, lane);
    double Vb[2][4];
    load_frag(&tab->Vbp[kx][0][0], Vb, lane);
    const double lz = 0.0 + __ldg(lamz + z);
#pragma unroll
    for (int g8 = 0; g8 < 2; ++g8) {
      const int y = 8 * g8 + r;
      double a[4];
#pragma unroll
      for (int kc = 0; kc < 4; ++kc) a[kc] = T.sU[idxG(z, y, 4 * kc + T.k4)];
      double acc[2][2] = {{0.0, 0.0}, {0.0, 0.0}};
      full_group(V, a, acc);
      const double lzy = lz + __ldg(lamy + y);
#pragma unroll
      for (int kc = 0; kc < 4; ++kc) {
        const int x = 8 * (kc >> 1) + c2 + (kc & 1);
        a[kc] = rd<S>(acc[kc >> 1][kc & 1] / (lzy + __ldg(lamx + x)));
      }
      o[g8][0][0] = o[g8][0][1] = o[g8][1][0] = o[g8][1][1] = 0.0;
      full_group(Vb, a, o[g8]);
    }
    __syncwarp();
#pragma unroll
    for (int g8 = 0; g8 < 2; ++g8)
#pragma unroll
      for (int nb = 0; nb < 2; ++nb)
        *reinterpret_cast<double2*>(&T.sU[idxA(z, 8 * g8 + r, 8 * nb + c2)]) =
            make_double2(rd<S>(o[g8][nb][0]), rd<S>(o[g8][nb][1]));
    __syncwarp();
    load_frag(&tab->Vb[ky][0][0], V, lane);
#pragma unroll
    for (int g8 = 0; g8 < 2; ++g8) {
      const int x = 8 * g8 + r;
      double a[4];
#pragma unroll
      for (int kc = 0; kc < 4; ++kc) a[kc] = T.sU[idxA(z, 4 * kc + T.k4, x)];
      o[g8][0][0] = o[g8][0][1] = o[g8][1][0] = o[g8][1][1] = 0.0;
      full_group(V, a, o[g8]);
    }
    __syncwarp();
#pragma unroll
    for (int g8 = 0; g8 < 2; ++g8)
#pragma unroll
      for (int nb = 0; nb < 2; ++nb)
#pragma unroll
        for (int i = 0; i < 2; ++i) T.sU[idxC(z, 8 * nb + c2 + i, 8 * g8 + r)] = rd<S>(o[g8][nb][i]);
    __syncwarp();
  }
  __syncthreads();
  // ---- z lines: backward V_z, x_new = x_old + correction
  load_frag(&tab->Vb[kz][0][0], V, lane);
  for (int yy = 0; yy < 2; ++yy) {
    const int y = 2 * w + yy;
#pragma unroll
    for (int g8 = 0; g8 < 2; ++g8) {
      const int x = 8 * g8 + r;
      double a[4];
#pragma unroll
      for (int kc = 0; kc < 4; ++kc) a[kc] = T.sU[idxC(4 * kc + T.k4, y, x)];
      double acc[2][2] = {{0.0, 0.0}, {0.0, 0.0}};
      full_group(V, a, acc);
#pragma unroll
      for (int nb = 0; nb < 2; ++nb)
#pragma unroll
        for (int i = 0; i < 2; ++i) {
          const int z = 8 * nb + c2 + i;
          if (KK < 8 && (x < T.skip[0] || y < T.skip[1] || z < T.skip[2])) continue;
          const long long o = off0 + (long long)z * T.sz + (long long)y * T.sy + x;
          xn[o] = (S)((XZ ? 0.0 : (double)__ldg(xo + o)) + rd<S>(acc[nb][i]));
        }
    }
  }
}

static Tables8 build_tables8(const double* opd, const double* eigd) {
  PatchL pl = build_patch_l(opd);
  Tables8 t;
  auto perm = [](int kc, int c) { return 8 * (kc >> 1) + 2 * c + (kc & 1); };
  for (int q = 0; q < 4; ++q) {
    const double* V = eigd + q * 256;  // V[i][j], row-major
    for (int fr = 0; fr < 8; ++fr)
      for (int ln = 0; ln < 32; ++ln) {
        const int nb = fr >> 2, kc = fr & 3, n = 8 * nb + (ln >> 2), c = ln & 3;
        const int ks = 4 * kc + c, kp = perm(kc, c);
        t.L[q][fr][ln] = pl.L[q][n][ks];
        t.Vf[q][fr][ln] = V[ks * 16 + n];   // (V^T)[n][k] = V[k][n]
        t.Vfp[q][fr][ln] = V[kp * 16 + n];
        t.Vb[q][fr][ln] = V[n * 16 + ks];
        t.Vbp[q][fr][ln] = V[n * 16 + kp];
      }
    for (int i = 0; i < 16; ++i) t.lam[q][i] = eigd[4 * 256 + q * 16 + i];
  }
  return t;
}

// content-addressed cache of uploaded tables (setup-time cudaMalloc/cudaMemcpy)
static std::mutex g_tab_mu;
struct TabEntry {
  int dev;
  std::vector<double> key;
  void* ptr;
};
static std::vector<TabEntry> g_tabs;

static const Tables8* tables8(const double* opd, const double* eigd) {
  int dev = 0;
  cudaGetDevice(&dev);
  std::vector<double> key(opd, opd + 2 * K * K + 4 * K);
  key.insert(key.end(), eigd, eigd + 4 * 256 + 4 * 16);
  std::lock_guard<std::mutex> lk(g_tab_mu);
  for (auto& e : g_tabs)
    if (e.dev == dev && e.key == key) return reinterpret_cast<const Tables8*>(e.ptr);
  Tables8 host = build_tables8(opd, eigd);
  void* d = nullptr;
  if (cudaMalloc(&d, sizeof(Tables8)) != cudaSuccess) return nullptr;
  if (cudaMemcpy(d, &host, sizeof(Tables8), cudaMemcpyHostToDevice) != cudaSuccess) return nullptr;
  g_tabs.push_back({dev, std::move(key), d});
  return reinterpret_cast<const Tables8*>(d);
}

// ---------------------------------------------------------------------------
// Residual + restriction (multigrid.py:249-250 + restrict :112-125) on DMMA:
// r = b - A x on the aligned tile, P^T along z chained in registers with the
// residual, then P^T along y and x on the CUDA cores (1/8 of the data).
struct PTab8 {
  double PTp[4][32];  // Op = P^T (8 x 16), perm k order, one n block
  double P[16][8];    // embedding P[fine][coarse]
};

template <int KK = 8, class S = double>
__global__ void __launch_bounds__(kThreads, 2) k_resid_restrict_dmma(const S* __restrict__ x,
                                                                    const S* __restrict__ b,
                                                                    S* __restrict__ coarse, Geom g,
                                                                    LevelOp<KK, MODE_FP64> op,
                                                                    const Tables8* __restrict__ tab,
                                                                    const PTab8* __restrict__ pt, Band bd) {
  extern __shared__ __align__(128) double smem[];
  Tile T;
  int batch;
  if (!tile_setup_band<KK>(T, smem, g, bd, batch)) return;
  prefetch_tile_rows_l2<KK>(T, b);
  prefetch_ahead_l2<KK>(g, bd, T, x);
  Frags f;
  Halo h;
  init_frags<KK>(T, op, f, h);
  prologue_fast<KK>(T, g, op, x, f, &tab->L[0][0][0]);  // L fragments staged into smem (T.sLf)
  xy_stages<S, KK>(T, f, h);
  __syncthreads();
  const int lane = T.lane, r = T.r, c2 = T.c2, w = T.warp;
  const long long off0 = (long long)(T.cz * KK) * T.sz + (long long)(T.cy * KK) * T.sy + T.cx * KK;
  load_l(T, f, T.kind[2]);
  double pfr[4];
#pragma unroll
  for (int kc = 0; kc < 4; ++kc) pfr[kc] = __ldg(&pt->PTp[kc][lane]);
  double keep[2][2][2];
#pragma unroll
  for (int yy = 0; yy < 2; ++yy) {
    const int y = 2 * w + yy;
#pragma unroll
    for (int g8 = 0; g8 < 2; ++g8) {
      double acc[2][2];
      z_group(T, f, h, y, 8 * g8, acc);
      const int xx = 8 * g8 + r;
      double a[4];
#pragma unroll
      for (int kc = 0; kc < 4; ++kc) {
        const int z = 8 * (kc >> 1) + c2 + (kc & 1);
        a[kc] = rd<S>((double)__ldg(b + off0 + (long long)z * T.sz + (long long)y * T.sy + xx) - acc[kc >> 1][kc & 1]);
      }
      keep[yy][g8][0] = keep[yy][g8][1] = 0.0;
#pragma unroll
      for (int kc = 0; kc < 4; ++kc) dmma(keep[yy][g8][0], keep[yy][g8][1], a[kc], pfr[kc]);
    }
  }
  __syncthreads();  // sB (dd) fully consumed
  // y and x restriction stages on DMMA as well (8-line groups, the z stage's permuted-k P^T fragments pfr):
  // S1 [zc][y][x] (y pitch 18, zc pitch 290) -> S2 [zc][yc][x] (yc pitch 18, zc pitch 146) -> coarse
  constexpr int R1Y = 18, R1Z = 290, R2Y = 18, R2Z = 146;
  double* S1 = T.sB;
#pragma unroll
  for (int yy = 0; yy < 2; ++yy)
#pragma unroll
    for (int g8 = 0; g8 < 2; ++g8)
#pragma unroll
      for (int i = 0; i < 2; ++i) S1[(c2 + i) * R1Z + (2 * w + yy) * R1Y + 8 * g8 + r] = rd<S>(keep[yy][g8][i]);
  __syncthreads();
  double* S2 = T.sU;
#pragma unroll
  for (int j = 0; j < 2; ++j) {  // y stage: group (zc, x half) = 2 w + j, lines x = xb + r; k = y
    const int gi = 2 * w + j, zc = gi >> 1, xb = 8 * (gi & 1);
    double acc[2] = {0.0, 0.0};
#pragma unroll
    for (int kc = 0; kc < 4; ++kc) {
      const int kp = 8 * (kc >> 1) + c2 + (kc & 1);
      dmma(acc[0], acc[1], S1[zc * R1Z + kp * R1Y + xb + r], pfr[kc]);
    }
#pragma unroll
    for (int i = 0; i < 2; ++i) S2[zc * R2Z + (c2 + i) * R2Y + xb + r] = rd<S>(acc[i]);
  }
  __syncthreads();
  {  // x stage: group zc = w, lines yc = r; k = x -> coarse (xc = c2, c2 + 1)
    double acc[2] = {0.0, 0.0};
#pragma unroll
    for (int kc = 0; kc < 4; ++kc) {
      const int kp = 8 * (kc >> 1) + c2 + (kc & 1);
      dmma(acc[0], acc[1], S2[w * R2Z + r * R2Y + kp], pfr[kc]);
    }
    const long long syc = (long long)(g.nx / 2) * KK, szc = syc * (long long)(g.ny / 2) * KK;
    S* out = coarse + (long long)((T.cz / 2) * KK + w) * szc + (long long)((T.cy / 2) * KK + r) * syc +
             (T.cx / 2) * KK + c2;
    out[0] = (S)acc[0];
    out[1] = (S)acc[1];
  }
}

static std::vector<std::pair<std::vector<double>, void*>> g_ptabs;

// Embedding along a 16-point tile line: blockdiag of the cell-pair embedding P (2KK x KK) over
// the line's 16 / (2KK) coarse cells -> a 16 x 8 matrix (KK = 8: P itself).
static const PTab8* ptables8(const double* embd_raw, int KK = 8) {
  int dev = 0;
  cudaGetDevice(&dev);
  std::vector<double> key(embd_raw, embd_raw + 2 * KK * KK);
  key.push_back((double)dev);
  key.push_back((double)KK);
  std::lock_guard<std::mutex> lk(g_tab_mu);
  for (auto& e : g_ptabs)
    if (e.first == key) return reinterpret_cast<const PTab8*>(e.second);
  double embd[16 * 8] = {};
  for (int c = 0; c < 16 / (2 * KK); ++c)
    for (int i = 0; i < 2 * KK; ++i)
      for (int j = 0; j < KK; ++j) embd[(c * 2 * KK + i) * 8 + c * KK + j] = embd_raw[i * KK + j];
  PTab8 host;
  for (int kc = 0; kc < 4; ++kc)
    for (int ln = 0; ln < 32; ++ln) {
      const int n = ln >> 2, kp = 8 * (kc >> 1) + 2 * (ln & 3) + (kc & 1);
      host.PTp[kc][ln] = embd[kp * 8 + n];  // (P^T)[n][k] = P[k][n]
    }
  for (int i = 0; i < 16; ++i)
    for (int j = 0; j < 8; ++j) host.P[i][j] = embd[i * 8 + j];
  void* d = nullptr;
  if (cudaMalloc(&d, sizeof(PTab8)) != cudaSuccess) return nullptr;
  if (cudaMemcpy(d, &host, sizeof(PTab8), cudaMemcpyHostToDevice) != cudaSuccess) return nullptr;
  g_ptabs.push_back({std::move(key), d});
  return reinterpret_cast<const PTab8*>(d);
}

// Prolongation + add on DMMA (multigrid.py:128-143, then x + e): one CTA (8 warps) per 16^3 fine tile = one 8^3
// block of coarse points; z -> y -> x stages, each an 8 -> 16 contraction with the line embedding E
// (blockdiag of the cell-pair embedding; m8n8k4, 2 k-chunks x 2 n-blocks per 8-line group); stage outputs are
// rounded to the storage type S as the reference stores them; the fine tile is staged by cp.async at the start
// and updated in the x stage.  Shared pitches: conflict-free C-fragment stores and (mostly) A gathers.
struct ETab8 {
  double B[2][2][32];  // [nb][kc][lane]: E[8 nb + (lane >> 2)][4 kc + (lane & 3)]
};
constexpr int EQ1Y = 12, EQ1Z = 98, EQ2Y = 10, EQ2Z = 162, EXY = 24, EXZ = 384;

template <int KK, class S>
__global__ void __launch_bounds__(kThreads, 2) k_prolong_dmma(const S* __restrict__ ec, S* __restrict__ fine,
                                                             int ncx, int ncy, int ncz,
                                                             const ETab8* __restrict__ et) {
  extern __shared__ __align__(128) double smem[];
  double* Q1 = smem;                                  // z stage out [z][yc][xc]
  double* Q2 = Q1 + 16 * EQ1Z;                        // y stage out [z][y][xc]
  S* X = reinterpret_cast<S*>(Q2 + 16 * EQ2Z);        // fine tile [z][y][x]
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5, r = lane >> 2, k4 = lane & 3;
  const long long csy = (long long)ncx * KK, csz = csy * (long long)ncy * KK;
  const long long fsy = 2 * csy, fsz = 2 * fsy * (long long)ncy * KK;
  const S* eb = ec + (long long)(8 * blockIdx.z) * csz + (long long)(8 * blockIdx.y) * csy + 8 * blockIdx.x;
  S* fb = fine + (long long)(16 * blockIdx.z) * fsz + (long long)(16 * blockIdx.y) * fsy + 16 * blockIdx.x;
  constexpr int CPR = 16 * (int)sizeof(S) / 16, NCH = 256 * CPR / kThreads;  // 16-byte chunks per fine row
#pragma unroll
  for (int k2 = 0; k2 < NCH; ++k2) {
    const int c = tid + kThreads * k2, ch = c % CPR, row = c / CPR, y = row & 15, z = row >> 4;
    const int e = ch * (16 / (int)sizeof(S));
    cp_async16(X + z * EXZ + y * EXY + e, fb + z * fsz + y * fsy + e);
  }
  double bf[2][2];
#pragma unroll
  for (int nb = 0; nb < 2; ++nb)
#pragma unroll
    for (int kc = 0; kc < 2; ++kc) bf[nb][kc] = __ldg(&et->B[nb][kc][lane]);
  auto group = [&](const double (&a)[2], double (&acc)[2][2]) {
#pragma unroll
    for (int nb = 0; nb < 2; ++nb) {
      acc[nb][0] = acc[nb][1] = 0.0;
#pragma unroll
      for (int kc = 0; kc < 2; ++kc) dmma(acc[nb][0], acc[nb][1], a[kc], bf[nb][kc]);
    }
  };
  {  // z stage: warp w = coarse row yc, lines xc = r; k = zc
    double a[2], acc[2][2];
#pragma unroll
    for (int kc = 0; kc < 2; ++kc) a[kc] = (double)__ldg(eb + (4 * kc + k4) * csz + w * csy + r);
    group(a, acc);
#pragma unroll
    for (int nb = 0; nb < 2; ++nb)
#pragma unroll
      for (int i = 0; i < 2; ++i) Q1[(8 * nb + 2 * k4 + i) * EQ1Z + w * EQ1Y + r] = rd<S>(acc[nb][i]);
  }
  __syncthreads();
#pragma unroll
  for (int j = 0; j < 2; ++j) {  // y stage: plane z = 2 w + j, lines xc = r; k = yc
    const int z = 2 * w + j;
    double a[2], acc[2][2];
#pragma unroll
    for (int kc = 0; kc < 2; ++kc) a[kc] = Q1[z * EQ1Z + (4 * kc + k4) * EQ1Y + r];
    group(a, acc);
#pragma unroll
    for (int nb = 0; nb < 2; ++nb)
#pragma unroll
      for (int i = 0; i < 2; ++i) Q2[z * EQ2Z + (8 * nb + 2 * k4 + i) * EQ2Y + r] = rd<S>(acc[nb][i]);
  }
  cp_async_wait_all();
  __syncthreads();
#pragma unroll
  for (int j = 0; j < 4; ++j) {  // x stage: group (z, half h) = 4 w + j, lines y = 8 h + r; k = xc; += fine
    const int z = (4 * w + j) >> 1, y = 8 * ((4 * w + j) & 1) + r;
    double a[2], acc[2][2];
#pragma unroll
    for (int kc = 0; kc < 2; ++kc) a[kc] = Q2[z * EQ2Z + y * EQ2Y + 4 * kc + k4];
    group(a, acc);
#pragma unroll
    for (int nb = 0; nb < 2; ++nb) {
      const int x = 8 * nb + 2 * k4;
      const S x0 = X[z * EXZ + y * EXY + x], x1 = X[z * EXZ + y * EXY + x + 1];
      S* p = fb + z * fsz + y * fsy + x;
      p[0] = (S)((double)x0 + rd<S>(acc[nb][0]));
      p[1] = (S)((double)x1 + rd<S>(acc[nb][1]));
    }
  }
}

static std::vector<std::pair<std::vector<double>, void*>> g_etabs;

static const ETab8* etables8(const double* embd_raw, int KK) {
  int dev = 0;
  cudaGetDevice(&dev);
  std::vector<double> key(embd_raw, embd_raw + 2 * KK * KK);
  key.push_back((double)dev);
  key.push_back((double)KK);
  std::lock_guard<std::mutex> lk(g_tab_mu);
  for (auto& e : g_etabs)
    if (e.first == key) return reinterpret_cast<const ETab8*>(e.second);
  double E[16 * 8] = {};
  for (int c = 0; c < 16 / (2 * KK); ++c)
    for (int i = 0; i < 2 * KK; ++i)
      for (int j = 0; j < KK; ++j) E[(c * 2 * KK + i) * 8 + c * KK + j] = embd_raw[i * KK + j];
  ETab8 host;
  for (int nb = 0; nb < 2; ++nb)
    for (int kc = 0; kc < 2; ++kc)
      for (int ln = 0; ln < 32; ++ln) host.B[nb][kc][ln] = E[(8 * nb + (ln >> 2)) * 8 + 4 * kc + (ln & 3)];
  void* d = nullptr;
  if (cudaMalloc(&d, sizeof(ETab8)) != cudaSuccess) return nullptr;
  if (cudaMemcpy(d, &host, sizeof(ETab8), cudaMemcpyHostToDevice) != cudaSuccess) return nullptr;
  g_etabs.push_back({std::move(key), d});
  return reinterpret_cast<const ETab8*>(d);
}

template <int KK, class S>
static int launch_prolong_t(int ncx, int ncy, int ncz, const double* embd, const void* e, void* fine,
                            cudaStream_t st) {
  if ((ncx * KK) % 8 || (ncy * KK) % 8 || (ncz * KK) % 8 || ncz * KK / 8 > 65535 || ncy * KK / 8 > 65535)
    return kUseGeneric;
  if (!aligned16(e) || !aligned16(fine)) return kUseGeneric;
  const ETab8* et = etables8(embd, KK);
  if (!et) return -3;
  const int smem = (int)(sizeof(double) * 16 * (EQ1Z + EQ2Z) + sizeof(S) * 16 * EXZ);
  if (cudaFuncSetAttribute(k_prolong_dmma<KK, S>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem) != cudaSuccess)
    return -3;
  const dim3 grid(ncx * KK / 8, ncy * KK / 8, ncz * KK / 8);
  k_prolong_dmma<KK, S><<<grid, kThreads, smem, st>>>((const S*)e, (S*)fine, ncx, ncy, ncz, et);
  return cudaGetLastError() == cudaSuccess ? 0 : -3;
}

// ---------------------------------------------------------------------------
// Q1 / Q3 (K = 2, 4) on DMMA: the same 16^3-point tile, now (16/K)^3 cells.  A tile line is
// 16 / K cells; its 1-D operators are the 16 x 16 line matrices -- blockdiag(M_cell) for the
// mass (per-lane B fragments from init_frags<K>) and, for the stiffness, the block-tridiagonal
// line operator (D on the diagonal, the rank-2 face couplings U / U^T between consecutive cells,
// Nitsche rows at domain-boundary ends) built here per boundary kind.  Faces to cells outside
// the tile line use the same (alpha, beta) halo as K = 8.
template <int KK>
static PatchL build_line_l(const double* opd) {
  constexpr int CPL = 16 / KK;
  const double* D = opd + KK * KK;
  const double* ucol = opd + 2 * KK * KK;
  const double* urow = ucol + KK;
  const double* bl = urow + KK;
  const double* br = bl + KK;
  PatchL p;
  for (int q = 0; q < 4; ++q) {
    const int lb = q >> 1, rb = q & 1;
    for (int i = 0; i < B; ++i)
      for (int j = 0; j < B; ++j) p.L[q][i][j] = 0.0;
    for (int c = 0; c < CPL; ++c)
      for (int i = 0; i < KK; ++i)
        for (int j = 0; j < KK; ++j) p.L[q][c * KK + i][c * KK + j] = D[i * KK + j];
    for (int c = 0; c + 1 < CPL; ++c) {
      const int o = c * KK, o2 = (c + 1) * KK;
      for (int i = 0; i < KK; ++i) {
        p.L[q][o + i][o2] = ucol[i];           // U column 0
        p.L[q][o + KK - 1][o2 + i] = urow[i];  // U row K-1
        p.L[q][o2][o + i] = ucol[i];           // U^T row 0
        p.L[q][o2 + i][o + KK - 1] = urow[i];  // U^T column K-1
      }
    }
    if (lb)
      for (int i = 0; i < KK; ++i) {
        p.L[q][i][0] += bl[i];
        if (i > 0) p.L[q][0][i] += bl[i];
      }
    if (rb) {
      const int e = B - KK;
      for (int i = 0; i < KK; ++i) {
        p.L[q][e + i][B - 1] += br[i];
        if (i < KK - 1) p.L[q][B - 1][e + i] += br[i];
      }
    }
  }
  return p;
}

template <int KK>
static const Tables8* line_tables(const double* opd) {
  int dev = 0;
  cudaGetDevice(&dev);
  std::vector<double> key(opd, opd + 2 * KK * KK + 4 * KK);
  key.push_back(-1000.0 - KK);  // tag: line tables of cell size KK
  std::lock_guard<std::mutex> lk(g_tab_mu);
  for (auto& e : g_tabs)
    if (e.dev == dev && e.key == key) return reinterpret_cast<const Tables8*>(e.ptr);
  PatchL pl = build_line_l<KK>(opd);
  Tables8 host{};
  for (int q = 0; q < 4; ++q)
    for (int fr = 0; fr < 8; ++fr)
      for (int ln = 0; ln < 32; ++ln) {
        const int nb = fr >> 2, kc = fr & 3;
        host.L[q][fr][ln] = pl.L[q][8 * nb + (ln >> 2)][4 * kc + (ln & 3)];
      }
  void* d = nullptr;
  if (cudaMalloc(&d, sizeof(Tables8)) != cudaSuccess) return nullptr;
  if (cudaMemcpy(d, &host, sizeof(Tables8), cudaMemcpyHostToDevice) != cudaSuccess) return nullptr;
  g_tabs.push_back({dev, std::move(key), d});
  return reinterpret_cast<const Tables8*>(d);
}

// Fragment tables of the line operators for the colour pass: L_line[kind] and the transforms
// blockdiag(V_patch) over the 16 / (2 KK) patches of a tile line (patch j's kind: left domain
// boundary only for j = 0, right only for the last), eigenvalues concatenated.
template <int KK>
static Tables8 build_line_tables(const double* opd, const double* eigd) {
  constexpr int PB = 2 * KK, PPL = 16 / PB;  // patch size, patches per line
  PatchL pl = build_line_l<KK>(opd);
  Tables8 t{};
  auto perm = [](int kc, int c) { return 8 * (kc >> 1) + 2 * c + (kc & 1); };
  for (int q = 0; q < 4; ++q) {
    const int lb = q >> 1, rb = q & 1;
    double V[16][16] = {};
    double lam[16];
    for (int j = 0; j < PPL; ++j) {
      const int kind = (j == 0 ? 2 * lb : 0) + (j == PPL - 1 ? rb : 0);
      const double* Vp = eigd + kind * PB * PB;
      for (int a = 0; a < PB; ++a) {
        for (int c = 0; c < PB; ++c) V[j * PB + a][j * PB + c] = Vp[a * PB + c];
        lam[j * PB + a] = eigd[4 * PB * PB + kind * PB + a];
      }
    }
    for (int fr = 0; fr < 8; ++fr)
      for (int ln = 0; ln < 32; ++ln) {
        const int nb = fr >> 2, kc = fr & 3, n = 8 * nb + (ln >> 2), c = ln & 3;
        const int ks = 4 * kc + c, kp = perm(kc, c);
        t.L[q][fr][ln] = pl.L[q][n][ks];
        t.Vf[q][fr][ln] = V[ks][n];
        t.Vfp[q][fr][ln] = V[kp][n];
        t.Vb[q][fr][ln] = V[n][ks];
        t.Vbp[q][fr][ln] = V[n][kp];
      }
    for (int i = 0; i < 16; ++i) t.lam[q][i] = lam[i];
  }
  return t;
}

template <int KK>
static const Tables8* line_colour_tables(const double* opd, const double* eigd) {
  int dev = 0;
  cudaGetDevice(&dev);
  std::vector<double> key(opd, opd + 2 * KK * KK + 4 * KK);
  key.insert(key.end(), eigd, eigd + 4 * 4 * KK * KK + 4 * 2 * KK);
  key.push_back(-2000.0 - KK);  // tag: colour line tables of cell size KK
  std::lock_guard<std::mutex> lk(g_tab_mu);
  for (auto& e : g_tabs)
    if (e.dev == dev && e.key == key) return reinterpret_cast<const Tables8*>(e.ptr);
  Tables8 host = build_line_tables<KK>(opd, eigd);
  void* d = nullptr;
  if (cudaMalloc(&d, sizeof(Tables8)) != cudaSuccess) return nullptr;
  if (cudaMemcpy(d, &host, sizeof(Tables8), cudaMemcpyHostToDevice) != cudaSuccess) return nullptr;
  g_tabs.push_back({dev, std::move(key), d});
  return reinterpret_cast<const Tables8*>(d);
}

template <int KK>
static int launch_colour_line(const Geom& g0, const double* opd, const double* eigd, const void* xo, const void* b,
                              void* xn, cudaStream_t st, bool f32) {
  constexpr int CPL = 16 / KK;
  if (g0.nx % CPL || g0.ny % CPL || g0.nz % CPL || !offsets32(g0)) return kUseGeneric;
  const int n3[3] = {g0.nx, g0.ny, g0.nz}, s3[3] = {g0.tx0, g0.ty0, g0.tz0};
  for (int a = 0; a < 3; ++a)
    if (s3[a] && n3[a] < CPL + 2) return kUseGeneric;  // shifted line must fit inside [1, n-1)
  Geom g = g0;
  g.ntx = g.nx / CPL;  // shifted colours: the last line is clamped to end at cell n-2 (tile_fields)
  g.nty = g.ny / CPL;
  g.ntz = g.nz / CPL;
  std::vector<double> o32, e32;
  if (f32) {
    if (!aligned16(xo)) return kUseGeneric;
    opd = demote32(o32, opd, op_len(KK));
    eigd = demote32(e32, eigd, eig_len(KK));
  }
  const Tables8* tab = line_colour_tables<KK>(opd, eigd);
  if (!tab) return -3;
  auto op = pack_op64<KK>(opd);
  auto go = [&](auto kern, auto* ut) {
    using S = std::remove_const_t<std::remove_pointer_t<decltype(ut)>>;
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmemTile) != cudaSuccess)
      return -3;
    const Band bd = make_band(g);
    kern<<<dim3(g.ntx, bd.by, bd.zb), kThreads, kSmemTile, st>>>((const S*)xo, (const S*)b, (S*)xn, g, op, tab, bd,
                                                                 0);
    return cudaGetLastError() == cudaSuccess ? 0 : -3;
  };
  if (!xo)  // zero iterate (unshifted colour only; checked by the caller)
    return f32 ? go(k_colour_dmma<KK, float, true>, (const float*)nullptr)
               : go(k_colour_dmma<KK, double, true>, (const double*)nullptr);
  return f32 ? go(k_colour_dmma<KK, float>, (const float*)nullptr)
             : go(k_colour_dmma<KK, double>, (const double*)nullptr);
}

template <int KK, class S>
__global__ void __launch_bounds__(kThreads, 2) k_vmult_dmma_line(const S* __restrict__ u, S* __restrict__ v,
                                                                Geom g, LevelOp<KK, MODE_FP64> op,
                                                                const Tables8* __restrict__ tab, Band bd, int prefetch) {
  extern __shared__ __align__(128) double smem[];
  Tile T;
  int batch;
  if (!tile_setup_band<KK>(T, smem, g, bd, batch)) return;
  u += (long long)batch * g.batch_stride;
  v += (long long)batch * g.batch_stride;
  if (prefetch) prefetch_ahead_l2<KK>(g, bd, T, u);
  Frags f;
  Halo h;
  init_frags<KK>(T, op, f, h);
  prologue_fast<KK>(T, g, op, u, f, &tab->L[0][0][0]);
  xy_stages<S, KK>(T, f, h);
  __syncthreads();
  load_l(T, f, T.kind[2]);
  S* vb = v + (long long)(T.cz * KK) * T.sz + (long long)(T.cy * KK) * T.sy + T.cx * KK;
  for (int yy = 0; yy < 2; ++yy) {
    const int y = 2 * T.warp + yy;
#pragma unroll
    for (int g8 = 0; g8 < 2; ++g8) {
      double acc[2][2];
      z_group(T, f, h, y, 8 * g8, acc);
      const int x = 8 * g8 + T.r;
#pragma unroll
      for (int nb = 0; nb < 2; ++nb)
#pragma unroll
        for (int i = 0; i < 2; ++i) vb[(long long)(8 * nb + T.c2 + i) * T.sz + (long long)y * T.sy + x] = (S)acc[nb][i];
    }
  }
}

template <int KK>
static int launch_line(const Geom& g0, const double* opd, const void* u, void* v, int batch, cudaStream_t st,
                       bool f32) {
  constexpr int CPL = 16 / KK;
  // z extent: the caller's tile range [tz0, tz0 + 2 ntz) cells (whole array or a slab sub-range)
  const int zc = 2 * g0.ntz;
  if (g0.nx % CPL || g0.ny % CPL || zc % CPL || !offsets32(g0)) return kUseGeneric;
  Geom g = g0;
  g.ntx = g.nx / CPL;
  g.nty = g.ny / CPL;
  g.ntz = zc / CPL;
  std::vector<double> o32;
  if (f32) {
    if (!aligned16(u)) return kUseGeneric;
    opd = demote32(o32, opd, op_len(KK));
  }
  const Tables8* tab = line_tables<KK>(opd);
  if (!tab) return -3;
  auto op = pack_op64<KK>(opd);
  auto go = [&](auto kern, auto* ut) {
    using S = std::remove_const_t<std::remove_pointer_t<decltype(ut)>>;
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmemTile) != cudaSuccess)
      return -3;
    const Band bd = make_band(g);
    const int per = bd.zb > 65535 ? 1 : 65535 / bd.zb;
    for (int b0 = 0; b0 < batch; b0 += per) {
      const int nb = batch - b0 < per ? batch - b0 : per;
      kern<<<dim3(g.ntx, bd.by, bd.zb * nb), kThreads, kSmemTile, st>>>(
          (const S*)u + (long long)b0 * g.batch_stride, (S*)v + (long long)b0 * g.batch_stride, g, op, tab, bd, 148);
    }
    return cudaGetLastError() == cudaSuccess ? 0 : -3;
  };
  return f32 ? go(k_vmult_dmma_line<KK, float>, (const float*)nullptr)
             : go(k_vmult_dmma_line<KK, double>, (const double*)nullptr);
}

}  // namespace dm

// FP64 vmult for K = 2 and 4 on DMMA (16-point tile lines of 16/K cells); kUseGeneric when the
// local grid is not a multiple of 16/K cells per axis.
int launch_vmult_dmma_line(int k_nodes, const Geom& g, const double* opd, const void* u, void* v, int batch,
                           cudaStream_t st, bool f32) {
  if (k_nodes == 4) return dm::launch_line<4>(g, opd, u, v, batch, st, f32);
  if (k_nodes == 2) return dm::launch_line<2>(g, opd, u, v, batch, st, f32);
  return kUseGeneric;
}

int launch_vmult_dmma8(const Geom& g, const double* opd, const void* u, void* v, int batch, cudaStream_t st,
                       bool f32) {
  if (!dm::offsets32(g)) return kUseGeneric;
  static_assert(dm::kSmemTile <= 113 * 1024, "two CTAs per SM");
  std::vector<double> o32;
  if (f32) {
    if (!dm::aligned16(u)) return kUseGeneric;
    opd = dm::demote32(o32, opd, dm::op_len(8));
  }
  auto op = dm::pack_op64(opd);
  static const double zero_eig[4 * 256 + 4 * 16] = {0};
  const dm::Tables8* tab = dm::tables8(opd, zero_eig);
  if (!tab) return -3;
  static const int pf = [] {
    const char* e = getenv("SUMFACT_B200_PREFETCH");
    return e ? atoi(e) : 148;  // one CTA per SM ahead: +2.5% (profiles/r01_vmult_fp64.md)
  }();

  auto go = [&](auto kern, auto* ut) {
    using S = std::remove_const_t<std::remove_pointer_t<decltype(ut)>>;
    cudaError_t err = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dm::kSmemTile);
    if (err != cudaSuccess) return -3;
    const dm::Band bd = dm::make_band(g);
    // grid z = (z, band) x batch; split very large batches across launches (gridDim.z <= 65535)
    const int per = bd.zb > 65535 ? 1 : 65535 / bd.zb;
    for (int b0 = 0; b0 < batch; b0 += per) {
      const int nb = batch - b0 < per ? batch - b0 : per;
      const S* ub = (const S*)u + (long long)b0 * g.batch_stride;
      S* vb = (S*)v + (long long)b0 * g.batch_stride;
      kern<<<dim3(g.ntx, bd.by, bd.zb * nb), dm::kThreads, dm::kSmemTile, st>>>(ub, vb, g, op, tab, bd, pf);
    }
    return cudaGetLastError() == cudaSuccess ? 0 : -3;
  };
  return f32 ? go(dm::k_vmult_dmma8<float>, (const float*)nullptr)
             : go(dm::k_vmult_dmma8<double>, (const double*)nullptr);
}

}  // namespace sf

namespace sf {
// FP64 colour pass for K = 2 and 4 on DMMA (kUseGeneric when the grid does not tile)
int launch_colour_dmma_line(int k_nodes, const Geom& g, const double* opd, const double* eigd, const void* xo,
                            const void* b, void* xn, cudaStream_t st, bool f32) {
  if (k_nodes == 4) return dm::launch_colour_line<4>(g, opd, eigd, xo, b, xn, st, f32);
  if (k_nodes == 2) return dm::launch_colour_line<2>(g, opd, eigd, xo, b, xn, st, f32);
  return kUseGeneric;
}

int launch_colour_dmma8(const Geom& g, const double* opd, const double* eigd, const void* xo, const void* b, void* xn,
                        cudaStream_t st, bool f32, bool copy_unc) {
  if (!dm::offsets32(g)) return kUseGeneric;
  std::vector<double> o32, e32;
  if (f32) {
    if (!dm::aligned16(xo)) return kUseGeneric;
    opd = dm::demote32(o32, opd, dm::op_len(8));
    eigd = dm::demote32(e32, eigd, dm::eig_len(8));
  }
  const dm::Tables8* tab = dm::tables8(opd, eigd);
  if (!tab) return -3;
  auto op = dm::pack_op64(opd);
  auto go = [&](auto kern, auto* ut) {
    using S = std::remove_const_t<std::remove_pointer_t<decltype(ut)>>;
    cudaError_t err = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dm::kSmemTile);
    if (err != cudaSuccess) return -3;
    const dm::Band bd = dm::make_band(g);
    kern<<<dim3(g.ntx, bd.by, bd.zb), dm::kThreads, dm::kSmemTile, st>>>((const S*)xo, (const S*)b, (S*)xn, g, op,
                                                                         tab, bd, copy_unc ? 1 : 0);
    return cudaGetLastError() == cudaSuccess ? 0 : -3;
  };
  if (!xo)  // zero iterate (unshifted colour only; checked by the caller)
    return f32 ? go(dm::k_colour_dmma<8, float, true>, (const float*)nullptr)
               : go(dm::k_colour_dmma<8, double, true>, (const double*)nullptr);
  return f32 ? go(dm::k_colour_dmma<8, float>, (const float*)nullptr)
             : go(dm::k_colour_dmma<8, double>, (const double*)nullptr);
}
}  // namespace sf

namespace sf {
namespace dm {
template <int KK>
static int launch_restrict_line(const Geom& g0, const double* opd, const double* embd, const void* x, const void* b,
                                void* coarse, cudaStream_t st, bool f32) {
  constexpr int CPL = 16 / KK;
  if (g0.nx % CPL || g0.ny % CPL || g0.nz % CPL || !offsets32(g0)) return kUseGeneric;
  Geom g = g0;
  g.ntx = g.nx / CPL;
  g.nty = g.ny / CPL;
  g.ntz = g.nz / CPL;
  std::vector<double> o32, m32;
  if (f32) {
    if (!aligned16(x)) return kUseGeneric;
    opd = demote32(o32, opd, op_len(KK));
    embd = demote32(m32, embd, 2 * KK * KK);
  }
  const Tables8* tab = line_tables<KK>(opd);
  const PTab8* pt = ptables8(embd, KK);
  if (!tab || !pt) return -3;
  auto op = pack_op64<KK>(opd);
  auto go = [&](auto kern, auto* ut) {
    using S = std::remove_const_t<std::remove_pointer_t<decltype(ut)>>;
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmemTile) != cudaSuccess)
      return -3;
    const Band bd = make_band(g);
    kern<<<dim3(g.ntx, bd.by, bd.zb), kThreads, kSmemTile, st>>>((const S*)x, (const S*)b, (S*)coarse, g, op, tab,
                                                                 pt, bd);
    return cudaGetLastError() == cudaSuccess ? 0 : -3;
  };
  return f32 ? go(k_resid_restrict_dmma<KK, float>, (const float*)nullptr)
             : go(k_resid_restrict_dmma<KK, double>, (const double*)nullptr);
}
}  // namespace dm

// FP64 residual + restriction for K = 2 and 4 on DMMA line tiles (kUseGeneric when the grid does not tile)
int launch_resid_restrict_dmma_line(int k_nodes, const Geom& g, const double* opd, const double* embd, const void* x,
                                    const void* b, void* coarse, cudaStream_t st, bool f32) {
  if (k_nodes == 4) return dm::launch_restrict_line<4>(g, opd, embd, x, b, coarse, st, f32);
  if (k_nodes == 2) return dm::launch_restrict_line<2>(g, opd, embd, x, b, coarse, st, f32);
  return kUseGeneric;
}

int launch_resid_restrict_dmma8(const Geom& g, const double* opd, const double* embd, const void* x, const void* b,
                                void* coarse, cudaStream_t st, bool f32) {
  if (!dm::offsets32(g)) return kUseGeneric;
  std::vector<double> o32, m32;
  if (f32) {
    if (!dm::aligned16(x)) return kUseGeneric;
    opd = dm::demote32(o32, opd, dm::op_len(8));
    embd = dm::demote32(m32, embd, 2 * 8 * 8);
  }
  // L fragments come from the level tables (built without eigenvectors here)
  static const double zero_eig[4 * 256 + 4 * 16] = {0};
  const dm::Tables8* tab = dm::tables8(opd, zero_eig);
  const dm::PTab8* pt = dm::ptables8(embd);
  if (!tab || !pt) return -3;
  auto op = dm::pack_op64(opd);
  auto go = [&](auto kern, auto* ut) {
    using S = std::remove_const_t<std::remove_pointer_t<decltype(ut)>>;
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dm::kSmemTile) != cudaSuccess)
      return -3;
    const dm::Band bd = dm::make_band(g);
    kern<<<dim3(g.ntx, bd.by, bd.zb), dm::kThreads, dm::kSmemTile, st>>>((const S*)x, (const S*)b, (S*)coarse, g, op,
                                                                         tab, pt, bd);
    return cudaGetLastError() == cudaSuccess ? 0 : -3;
  };
  return f32 ? go(dm::k_resid_restrict_dmma<8, float>, (const float*)nullptr)
             : go(dm::k_resid_restrict_dmma<8, double>, (const double*)nullptr);
}
}  // namespace sf

namespace sf {
int launch_prolong_dmma(int k_nodes, int ncx, int ncy, int ncz, const double* embd, const void* e, void* fine,
                        cudaStream_t st, bool f32) {
  switch (k_nodes) {
    case 8: return f32 ? dm::launch_prolong_t<8, float>(ncx, ncy, ncz, embd, e, fine, st)
                       : dm::launch_prolong_t<8, double>(ncx, ncy, ncz, embd, e, fine, st);
    case 4: return f32 ? dm::launch_prolong_t<4, float>(ncx, ncy, ncz, embd, e, fine, st)
                       : dm::launch_prolong_t<4, double>(ncx, ncy, ncz, embd, e, fine, st);
    case 2: return f32 ? dm::launch_prolong_t<2, float>(ncx, ncy, ncz, embd, e, fine, st)
                       : dm::launch_prolong_t<2, double>(ncx, ncy, ncz, embd, e, fine, st);
    default: return kUseGeneric;
  }
}
}  // namespace sf
