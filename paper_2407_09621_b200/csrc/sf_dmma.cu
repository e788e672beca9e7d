// FP64 Q7 kernels on the tensor cores (DMMA).  See sf_dmma.cuh for the
// schedule and the shared-memory layouts.
#include <cuda_runtime.h>

#include <cstdlib>

#include "sf_dmma.cuh"
#include "sf_internal.h"

namespace sf {
namespace dm {

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

__global__ void __launch_bounds__(kThreads, 2) k_vmult_dmma8(const double* __restrict__ u, double* __restrict__ v,
                                                            Geom g, LevelOp<K, MODE_FP64> op, PatchL pl) {
  extern __shared__ __align__(128) double smem[];
  u += (long long)blockIdx.y * g.batch_stride;
  v += (long long)blockIdx.y * g.batch_stride;
  Tile T;
  if (!tile_setup(T, smem, g, blockIdx.x)) return;
  Frags f;
  Halo h;
  init_frags(T, op, f, h);
  stage_l_frags(T, &pl.L[0][0][0]);
  prologue(T, g, op, u, f);
  xy_stages(T, f, h);
  __syncthreads();
  load_l(T, f, T.kind[2]);
  double* vb = v + (long long)(T.cz * K) * T.sz + (long long)(T.cy * K) * T.sy + T.cx * K;
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
        for (int i = 0; i < 2; ++i) vb[(long long)(8 * nb + T.c2 + i) * T.sz + (long long)y * T.sy + x] = acc[nb][i];
    }
  }
}


// Persistent warp-specialised variant: 8 consumer warps run the x/y/z stages of
// tile i while 4 producer warps stage tile i+1 (cp.async tile, L2 trace loads,
// trace-plane masses) into the other half of a double buffer.  Named barriers:
// FULL[b] (producers arrive, consumers sync), EMPTY[b] (consumers arrive,
// producers sync), CONS (consumers only), PROD (producers only).
constexpr int kCons = 256, kProd = 128, kWsThreads = kCons + kProd;
constexpr size_t kSmemWs = sizeof(double) * (2 * (VOL + 12 * TRP) + VOL + 4 * 8 * 32);
enum { BAR_FULL0 = 1, BAR_EMPTY0 = 3, BAR_CONS = 5, BAR_PROD = 6 };

__global__ void __launch_bounds__(kWsThreads, 1) k_vmult_dmma8_ws(const double* __restrict__ u,
                                                                 double* __restrict__ v, Geom g,
                                                                 LevelOp<K, MODE_FP64> op, PatchL pl) {
  extern __shared__ __align__(128) double smem[];
  double* sUbuf[2] = {smem, smem + VOL};
  double* trbuf[2] = {smem + 2 * VOL, smem + 2 * VOL + 12 * TRP};
  double* sB = smem + 2 * VOL + 24 * TRP;
  double* sLf = sB + VOL;
  const int ntiles = g.ntx * g.nty * g.ntz;
  const int tid = threadIdx.x;
  Tile T;
  T.sB = sB;
  T.sLf = sLf;
  tile_geom(T, g, 0);  // lane/warp fields
  for (int i = tid; i < 4 * 8 * 32; i += kWsThreads) {
    const int kind = i >> 8, fr = (i >> 5) & 7, ln = i & 31;
    sLf[i] = pl.L[kind][8 * (fr >> 2) + (ln >> 2)][4 * (fr & 3) + (ln & 3)];
  }
  Frags f;
  Halo h;
  init_frags(T, op, f, h);
  __syncthreads();
  int n = 0;
  for (int t = blockIdx.x; t < ntiles; t += gridDim.x) ++n;

  if (tid >= kCons) {  // ---------------- producers
    const int ptid = tid - kCons;
    int it = 0;
    for (int t = blockIdx.x; t < ntiles; t += gridDim.x, ++it) {
      const int b = it & 1;
      if (it >= 2) bar_sync(BAR_EMPTY0 + b, kWsThreads);
      T.sU = sUbuf[b];
      T.tr = trbuf[b];
      tile_geom(T, g, t);
      T.warp = ptid >> 5;
      produce<kProd>(T, g, op, u, f, ptid, [] { bar_sync(BAR_PROD, kProd); });
      bar_arrive(BAR_FULL0 + b, kWsThreads);
    }
    for (int j = n - 2 < 0 ? 0 : n - 2; j < n; ++j) bar_sync(BAR_EMPTY0 + (j & 1), kWsThreads);
    return;
  }
  // ---------------- consumers
  int it = 0;
  for (int t = blockIdx.x; t < ntiles; t += gridDim.x, ++it) {
    const int b = it & 1;
    T.sU = sUbuf[b];
    T.tr = trbuf[b];
    tile_geom(T, g, t);
    bar_sync(BAR_FULL0 + b, kWsThreads);
    xy_stages(T, f, h);
    bar_sync(BAR_CONS, kCons);
    load_l(T, f, T.kind[2]);
    double* vb = v + (long long)(T.cz * K) * T.sz + (long long)(T.cy * K) * T.sy + T.cx * K;
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
          for (int i = 0; i < 2; ++i)
            vb[(long long)(8 * nb + T.c2 + i) * T.sz + (long long)y * T.sy + x] = acc[nb][i];
      }
    }
    bar_sync(BAR_CONS, kCons);  // sB / sU[b] free before the next tile reuses them
    bar_arrive(BAR_EMPTY0 + b, kWsThreads);
  }
}

}  // namespace dm

int launch_vmult_dmma8(const Geom& g, const double* opd, const void* u, void* v, int batch, cudaStream_t st) {
  static_assert(dm::kSmemTile <= 113 * 1024, "two CTAs per SM");
  auto op = dm::pack_op64(opd);
  dm::PatchL pl = dm::build_patch_l(opd);
  static const int ws = [] {
    const char* e = getenv("SUMFACT_B200_DMMA_WS");
    return (e && *e == '0') ? 0 : 1;
  }();
  if (ws && batch == 1) {
    cudaError_t err =
        cudaFuncSetAttribute(dm::k_vmult_dmma8_ws, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dm::kSmemWs);
    if (err != cudaSuccess) return -3;
    int sms = 148;
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int tiles = g.ntx * g.nty * g.ntz;
    const int grid = tiles < sms ? tiles : sms;
    dm::k_vmult_dmma8_ws<<<grid, dm::kWsThreads, dm::kSmemWs, st>>>((const double*)u, (double*)v, g, op, pl);
    return cudaGetLastError() == cudaSuccess ? 0 : -3;
  }
  cudaError_t err =
      cudaFuncSetAttribute(dm::k_vmult_dmma8, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dm::kSmemTile);
  if (err != cudaSuccess) return -3;
  const int tiles = g.ntx * g.nty * g.ntz;
  dm::k_vmult_dmma8<<<dim3(tiles, batch), dm::kThreads, dm::kSmemTile, st>>>((const double*)u, (double*)v, g, op,
                                                                              pl);
  return cudaGetLastError() == cudaSuccess ? 0 : -3;
}

}  // namespace sf
