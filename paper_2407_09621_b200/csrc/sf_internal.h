// Internal (non-ABI) launchers shared between translation units.
#pragma once
#include <cuda_runtime.h>

#include <cuda_fp16.h>

#include <cmath>

#include "sf_common.cuh"

namespace sf {

// host: one matrix entry prepared under a mode (fp16: demoted; EC: (main, 2^11-scaled residual))
template <int MODE>
inline ME<MODE> pack_me(double x) {
  ME<MODE> m;
  if constexpr (MODE == MODE_FP64) {
    m.h = x;
  } else if constexpr (MODE == MODE_FP32) {
    m.h = (float)x;
  } else if constexpr (MODE == MODE_FP16) {
    m.h = __half2float(__float2half_rn((float)x));
  } else {
    const float x32 = (float)x;
    const float h = __half2float(__float2half_rn(x32));
    m.h = h;
    m.d = __half2float(__float2half_rn((x32 - h) * kEcScale));
  }
  return m;
}

// host: static power-of-two range scales of one level for the binary16 modes
// (sf_common.cuh).  Writes scaled copies of level_op (M by 2^aM,
// the stiffness blocks by 2^aL) and of the eigenvector table (V by 2^aV).
inline int ceil_log2(double x) {
  int e;
  const double m = std::frexp(x, &e);  // x = m 2^e, m in [0.5, 1)
  return m == 0.5 ? e - 1 : e;
}
inline Scales level_scales(int K, const double* opd, const double* eigd, double* op_out, double* eig_out) {
  Scales sc{0, 0, 0};
  if (opd) {
    double mM = 0, mL = 0;
    for (int i = 0; i < K * K; ++i) mM = std::fmax(mM, std::fabs(opd[i]));
    for (int i = K * K; i < 2 * K * K + 4 * K; ++i) mL = std::fmax(mL, std::fabs(opd[i]));
    const int aM = mM > 0 ? -ceil_log2(mM) : 0;     // max|M^| in (1/2, 1]
    const int aL = mL > 0 ? 7 - ceil_log2(mL) : 0;  // max|L^| in (64, 128]
    sc.aA = aL + 2 * aM;
    for (int i = 0; i < K * K; ++i) op_out[i] = std::ldexp(opd[i], aM);
    for (int i = K * K; i < 2 * K * K + 4 * K; ++i) op_out[i] = std::ldexp(opd[i], aL);
  }
  if (eigd) {
    const int B = 2 * K;
    double mV = 0, lmin = 1e300;
    for (int i = 0; i < 4 * B * B; ++i) mV = std::fmax(mV, std::fabs(eigd[i]));
    for (int i = 0; i < 4 * B; ++i) lmin = std::fmin(lmin, eigd[4 * B * B + i]);
    sc.aV = 1 - ceil_log2(mV);          // max|V^| in (1, 2]
    sc.aD = ceil_log2(3.0 * lmin) - 8;  // divided values <= 2^-7 of the forward transform
    for (int i = 0; i < 4 * B * B; ++i) eig_out[i] = std::ldexp(eigd[i], sc.aV);
    for (int i = 0; i < 4 * B; ++i) eig_out[4 * B * B + i] = eigd[4 * B * B + i];
  }
  return sc;
}

// host: the (possibly range-scaled) operator blocks a launch packs into kernel parameters
template <int K, int MODE>
struct Prepared {
  double op[2 * K * K + 4 * K];
  double eig[4 * 4 * K * K + 8 * K];
  const double* opd;
  const double* eigd;
  Scales sc{0, 0, 0};
  Prepared(const double* o, const double* e) : opd(o), eigd(e) {
    if constexpr (MT<MODE>::kHalf) {
      sc = level_scales(K, o, e, op, eig);
      if (o) opd = op;
      if (e) eigd = eig;
    }
  }
};

// host: L_smooth[(lb,rb)] (16x16, Q7) = [[D + lb*Bl, U], [U^T, D + rb*Br]] from the cell-wise blocks
inline void build_patch_l_host(const double* opd, double* L /* [4][16][16] */) {
  constexpr int K = 8, B = 16;
  const double* D = opd + K * K;
  const double* ucol = opd + 2 * K * K;
  const double* urow = ucol + K;
  const double* bl = urow + K;
  const double* br = bl + K;
  for (int q = 0; q < 4; ++q) {
    double* P = L + q * B * B;
    const int lb = q >> 1, rb = q & 1;
    for (int i = 0; i < B * B; ++i) P[i] = 0.0;
    for (int c = 0; c < 2; ++c)
      for (int i = 0; i < K; ++i)
        for (int j = 0; j < K; ++j) P[(c * K + i) * B + c * K + j] = D[i * K + j];
    for (int i = 0; i < K; ++i) {
      P[i * B + K] = ucol[i];            // U column 0
      P[(K - 1) * B + K + i] = urow[i];  // U row K-1
      P[K * B + i] = ucol[i];            // U^T row 0
      P[(K + i) * B + K - 1] = urow[i];  // U^T column K-1
    }
    if (lb)
      for (int i = 0; i < K; ++i) {
        P[i * B] += bl[i];
        if (i > 0) P[i] += bl[i];
      }
    if (rb)
      for (int i = 0; i < K; ++i) {
        P[(K + i) * B + B - 1] += br[i];
        if (i < K - 1) P[(B - 1) * B + K + i] += br[i];
      }
  }
}
// host: the 16-point tile-line operators for cell size KK in {2, 4, 8} (16/KK cells per line):
// L_line[(lb,rb)] = block-tridiagonal (D, rank-2 U / U^T between consecutive cells, Nitsche at the
// line ends), M_line = blockdiag(M_cell), and the patch transforms / eigenvalues of the line's
// 16/(2KK) vertex patches (patch j's kind: left boundary only for j = 0, right only for the last).
inline void build_line_ops_host(int KK, const double* opd, const double* eigd, double* M /*[256]*/,
                                double* L /*[4][256]*/, double* V /*[4][256] or null*/, double* lam /*[4][16]*/) {
  const int CPL = 16 / KK, PB = 2 * KK, PPL = 16 / PB;
  const double* D = opd + KK * KK;
  const double* ucol = opd + 2 * KK * KK;
  const double* urow = ucol + KK;
  const double* bl = urow + KK;
  const double* br = bl + KK;
  for (int i = 0; i < 256; ++i) M[i] = 0.0;
  for (int c = 0; c < CPL; ++c)
    for (int i = 0; i < KK; ++i)
      for (int j = 0; j < KK; ++j) M[(c * KK + i) * 16 + c * KK + j] = opd[i * KK + j];
  for (int q = 0; q < 4; ++q) {
    double* P = L + q * 256;
    const int lb = q >> 1, rb = q & 1;
    for (int i = 0; i < 256; ++i) P[i] = 0.0;
    for (int c = 0; c < CPL; ++c)
      for (int i = 0; i < KK; ++i)
        for (int j = 0; j < KK; ++j) P[(c * KK + i) * 16 + c * KK + j] = D[i * KK + j];
    for (int c = 0; c + 1 < CPL; ++c) {
      const int o = c * KK, o2 = (c + 1) * KK;
      for (int i = 0; i < KK; ++i) {
        P[(o + i) * 16 + o2] = ucol[i];
        P[(o + KK - 1) * 16 + o2 + i] = urow[i];
        P[o2 * 16 + o + i] = ucol[i];
        P[(o2 + i) * 16 + o + KK - 1] = urow[i];
      }
    }
    if (lb)
      for (int i = 0; i < KK; ++i) {
        P[i * 16] += bl[i];
        if (i > 0) P[i] += bl[i];
      }
    if (rb) {
      const int e = 16 - KK;
      for (int i = 0; i < KK; ++i) {
        P[(e + i) * 16 + 15] += br[i];
        if (i < KK - 1) P[15 * 16 + e + i] += br[i];
      }
    }
    if (V) {
      double* W = V + q * 256;
      for (int i = 0; i < 256; ++i) W[i] = 0.0;
      for (int j = 0; j < PPL; ++j) {
        const int kind = (j == 0 ? 2 * lb : 0) + (j == PPL - 1 ? rb : 0);
        const double* Vp = eigd + kind * PB * PB;
        for (int a = 0; a < PB; ++a) {
          for (int c = 0; c < PB; ++c) W[(j * PB + a) * 16 + j * PB + c] = Vp[a * PB + c];
          lam[q * 16 + j * PB + a] = eigd[4 * PB * PB + kind * PB + a];
        }
      }
    }
  }
}

// FP64 Q7 vmult on DMMA tensor cores (sf_dmma.cu); returns 0 or SF_ECUDA
constexpr int kUseGeneric = -4;  // tensor-core launcher declines (falls back to the tile engine)
// f32: fp32 storage on the same FP64 tensor-core kernels (operator data demoted to fp32 values,
// stage outputs rounded to fp32); kUseGeneric if a vector is not 16-byte aligned
int launch_vmult_dmma_line(int k_nodes, const Geom& g, const double* level_op, const void* u, void* v, int batch,
                           cudaStream_t st, bool f32 = false);
int launch_vmult_dmma8(const Geom& g, const double* level_op, const void* u, void* v, int batch, cudaStream_t st,
                       bool f32 = false);
// FP64 Q7 smoother colour pass on DMMA (sf_dmma.cu)
int launch_colour_dmma_line(int k_nodes, const Geom& g, const double* level_op, const double* patch_eig,
                            const void* x_old, const void* b, void* x_new, cudaStream_t st, bool f32 = false);
// copy_unc: the kernel also copies the shifted colour's uncovered cells (then the caller does not)
int launch_colour_dmma8(const Geom& g, const double* level_op, const double* patch_eig, const void* x_old,
                        const void* b, void* x_new, cudaStream_t st, bool f32 = false, bool copy_unc = false);
// FP64 Q7 residual + restriction on DMMA (sf_dmma.cu)
int launch_resid_restrict_dmma_line(int k_nodes, const Geom& g, const double* level_op, const double* embedding,
                                    const void* x, const void* b, void* coarse, cudaStream_t st, bool f32 = false);
int launch_resid_restrict_dmma8(const Geom& g, const double* level_op, const double* embedding, const void* x,
                                const void* b, void* coarse, cudaStream_t st, bool f32 = false);
// FP16 / FP16-EC Q7 kernels on HMMA (sf_hmma.cu)
// fp64 / fp32-storage prolongation + add on DMMA (sf_dmma.cu); kUseGeneric when the coarse grid does not tile
int launch_prolong_dmma(int k_nodes, int ncx, int ncy, int ncz, const double* embedding, const void* e, void* fine,
                        cudaStream_t st, bool f32);
// binary16 prolongation + add on HMMA (sf_hmma.cu); kUseGeneric when the coarse grid does not tile
int launch_prolong_hmma(int mode, int k_nodes, int ncx, int ncy, int ncz, const double* embedding, const void* e,
                        void* fine, cudaStream_t st);
int launch_resid_restrict_hmma_line(int mode, int k_nodes, const Geom& g, const double* level_op,
                                    const double* embedding, const void* x, const void* b, void* coarse,
                                    cudaStream_t st);
int launch_resid_restrict_hmma8(int mode, const Geom& g, const double* level_op, const double* embedding,
                                const void* x, const void* b, void* coarse, cudaStream_t st);
int launch_vmult_hmma_line(int mode, int k_nodes, const Geom& g, const double* level_op, const void* u, void* v,
                           int batch, cudaStream_t st);
int launch_colour_hmma_line(int mode, int k_nodes, const Geom& g, const double* level_op, const double* patch_eig,
                            const void* x_old, const void* b, void* x_new, cudaStream_t st);
int launch_vmult_hmma8(int mode, const Geom& g, const double* level_op, const void* u, void* v, int batch,
                       cudaStream_t st);
int launch_colour_hmma8(int mode, const Geom& g, const double* level_op, const double* patch_eig, const void* x_old,
                        const void* b, void* x_new, cudaStream_t st);
}  // namespace sf
