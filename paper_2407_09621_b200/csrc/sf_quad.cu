// Pre/post-processing of the solve on the device: the load vector with boundary data
// and the L2 / broken-H1 error norms for general data, as sum-factorised Gauss-point contractions
// (src/discretization.py:317-459).  The data (f, g, the exact solution / gradient) are tabulated at
// the Gauss points by the caller -- on the device when the callables accept CUDA tensors -- one
// z-chunk of cells at a time, so a 1e9-DoF solve never leaves the device.
//
//   k_quad_load   : b_cell = (S^T (x) S^T (x) S^T) (w f)          assemble_rhs :317-348 (x, then y, then z)
//   k_face_load   : b_face_layer += coef_normal (x) (S^T (x) S^T) (w g)   _rhs_boundary :351-394
//   k_quad_error  : sum_q w (I u_h - f)^2 with I = Sz (x) Sy (x) Sx (values or one derivative axis)
//                   l2_error / h1_seminorm_error :405-459 (_quadrature_values :405-419, x, then y, then z)
// FP64 throughout (the reference's pre/post-processing is fp64).  One CTA per cell; the three
// contractions run through shared memory; reductions are fixed-order (per-CTA partials, then one
// fixed tree), so repeated runs are bitwise identical.
#include <cuda_runtime.h>

#include <cstdio>

#include "../../include/sumfact_b200.h"

namespace {

constexpr int kThreads = 128;
thread_local char g_err[256] = "";

int invalid(const char* what, const char* why) {
  snprintf(g_err, sizeof(g_err), "%s: %s", what, why);
  return SF_EINVAL;
}
int launched(const char* what) {
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    snprintf(g_err, sizeof(g_err), "%s: %s", what, cudaGetErrorString(e));
    return SF_ECUDA;
  }
  return SF_OK;
}

// out[o][i][r] = sum_k M[i][k] in[o][k][r] on shared-memory tensors (M is rows x cols, row-major)
template <int O, int I, int KD, int R>
__device__ __forceinline__ void contract_smem(const double* __restrict__ M, const double* in, double* out) {
  for (int e = threadIdx.x; e < O * I * R; e += kThreads) {
    const int r = e % R, i = (e / R) % I, o = e / (R * I);
    double s = 0.0;
#pragma unroll
    for (int k = 0; k < KD; ++k) s = fma(M[i * KD + k], in[(o * KD + k) * R + r], s);
    out[e] = s;
  }
}

// one cell's K^3 DoFs -> its Q^3 Gauss-point values (x, then y, then z), A = u's row length
template <int K, int Q>
__global__ void __launch_bounds__(kThreads) k_quad_error(int n, int nzc, const double* __restrict__ u,
                                                         const double* __restrict__ mats /* 3 x Q x K: x, y, z */,
                                                         const double* __restrict__ fq, const double* __restrict__ w,
                                                         int z0, double* __restrict__ part) {
  __shared__ double sm[3 * Q * K];
  __shared__ double a[K * K * K > Q * Q * Q ? K * K * K : Q * Q * Q];
  __shared__ double b[K * K * Q > Q * Q * Q ? K * K * Q : Q * Q * Q];
  __shared__ double red[kThreads];
  const int cx = blockIdx.x, cy = blockIdx.y, cz = blockIdx.z;
  const long long A = (long long)n * K;
  for (int i = threadIdx.x; i < 3 * Q * K; i += kThreads) sm[i] = mats[i];
  for (int e = threadIdx.x; e < K * K * K; e += kThreads) {
    const int x = e % K, y = (e / K) % K, z = e / (K * K);
    a[e] = u[((long long)(cz * K + z) * A + (cy * K + y)) * A + cx * K + x];
  }
  __syncthreads();
  contract_smem<K * K, Q, K, 1>(sm, a, b);              // x: [z][y][qx]
  __syncthreads();
  contract_smem<K, Q, K, Q>(sm + Q * K, b, a);          // y: [z][qy][qx]
  __syncthreads();
  contract_smem<1, Q, K, Q * Q>(sm + 2 * Q * K, a, b);  // z: [qz][qy][qx]
  __syncthreads();
  const long long AQ = (long long)n * Q;
  double s = 0.0;
  for (int e = threadIdx.x; e < Q * Q * Q; e += kThreads) {
    const int qx = e % Q, qy = (e / Q) % Q, qz = e / (Q * Q);
    const int gz = cz * Q + qz, gy = cy * Q + qy, gx = cx * Q + qx;
    const double d = b[e] - fq[((long long)gz * AQ + gy) * AQ + gx];
    s = fma(w[(z0 + cz) * Q + qz] * w[gy] * w[gx], d * d, s);
  }
  red[threadIdx.x] = s;
  __syncthreads();
  for (int t = kThreads / 2; t > 0; t >>= 1) {
    if (threadIdx.x < t) red[threadIdx.x] += red[threadIdx.x + t];
    __syncthreads();
  }
  if (threadIdx.x == 0) part[((long long)cz * n + cy) * n + cx] = red[0];
}

// one cell's Q^3 weighted Gauss-point data -> its K^3 load-vector entries (S^T along x, then y, then z)
template <int K, int Q>
__global__ void __launch_bounds__(kThreads) k_quad_load(int n, int nzc, const double* __restrict__ fq,
                                                        const double* __restrict__ st /* K x Q = S^T */,
                                                        const double* __restrict__ w, int z0,
                                                        double* __restrict__ bvec) {
  __shared__ double sm[K * Q];
  __shared__ double a[Q * Q * Q > K * K * K ? Q * Q * Q : K * K * K];
  __shared__ double b[Q * Q * K > Q * K * K ? Q * Q * K : Q * K * K];
  const int cx = blockIdx.x, cy = blockIdx.y, cz = blockIdx.z;
  const long long AQ = (long long)n * Q, A = (long long)n * K;
  for (int i = threadIdx.x; i < K * Q; i += kThreads) sm[i] = st[i];
  for (int e = threadIdx.x; e < Q * Q * Q; e += kThreads) {
    const int qx = e % Q, qy = (e / Q) % Q, qz = e / (Q * Q);
    const int gz = cz * Q + qz, gy = cy * Q + qy, gx = cx * Q + qx;
    // the reference weights the values axis by axis (z, y, x) before contracting
    a[e] = fq[((long long)gz * AQ + gy) * AQ + gx] * w[(z0 + cz) * Q + qz] * w[gy] * w[gx];
  }
  __syncthreads();
  contract_smem<Q * Q, K, Q, 1>(sm, a, b);      // x: [qz][qy][x]
  __syncthreads();
  contract_smem<Q, K, Q, K>(sm, b, a);          // y: [qz][y][x]
  __syncthreads();
  contract_smem<1, K, Q, K * K>(sm, a, b);      // z: [z][y][x]
  __syncthreads();
  for (int e = threadIdx.x; e < K * K * K; e += kThreads) {
    const int x = e % K, y = (e / K) % K, z = e / (K * K);
    bvec[((long long)(cz * K + z) * A + (cy * K + y)) * A + cx * K + x] = b[e];
  }
}

// Nitsche data term of one domain face (normal tensor axis `axis`, side 0/1): for every face cell
// (t1 slow, t0 fast tangential cell), tang = (S^T (x) S^T)(w g) over its Q^2 face points (last
// tangential axis first), then b[cell boundary layer][i_n] += coef[i_n] tang.  g: the face grid
// (n Q)^2 in (slow, fast) tangential order; z-slab range [z0, z0 + nzc) of the local b.
template <int K, int Q>
__global__ void __launch_bounds__(kThreads) k_face_load(int n, int nzc, int z0, int axis, int side,
                                                        const double* __restrict__ g,
                                                        const double* __restrict__ st, const double* __restrict__ w,
                                                        const double* __restrict__ coef, double* __restrict__ bvec) {
  __shared__ double sm[K * Q];
  __shared__ double a[Q * Q];
  __shared__ double bb[Q * K];
  __shared__ double t2[K * K];
  const int c0 = blockIdx.x, c1 = blockIdx.y;  // fast / slow tangential cell (slow = z for x / y faces)
  const long long AQ = (long long)n * Q, A = (long long)n * K;
  for (int i = threadIdx.x; i < K * Q; i += kThreads) sm[i] = st[i];
  // global slow-axis cell (z is local to the slab for x / y faces)
  const int gs = axis == 2 ? c1 : z0 + c1;
  for (int e = threadIdx.x; e < Q * Q; e += kThreads) {
    const int qf = e % Q, qs = e / Q;
    const long long gi = (long long)(gs * Q + qs) * AQ + c0 * Q + qf;
    a[e] = g[gi] * w[gs * Q + qs] * w[c0 * Q + qf];
  }
  __syncthreads();
  contract_smem<Q, K, Q, 1>(sm, a, bb);  // fast axis: [qs][f]
  __syncthreads();
  contract_smem<1, K, Q, K>(sm, bb, t2);  // slow axis: [s][f]
  __syncthreads();
  for (int e = threadIdx.x; e < K * K * K; e += kThreads) {
    const int f = e % K, s = (e / K) % K, i = e / (K * K);  // i: node along the normal
    const int ci = side ? n - 1 : 0;
    long long x, y, z;
    if (axis == 0) { x = ci * K + i; y = c0 * K + f; z = c1 * K + s; }
    else if (axis == 1) { y = ci * K + i; x = c0 * K + f; z = c1 * K + s; }
    else { z = (ci - z0) * K + i; x = c0 * K + f; y = c1 * K + s; }
    if (axis == 2 && (ci < z0 || ci >= z0 + nzc)) continue;  // face outside this slab
    bvec[(z * A + y) * A + x] += coef[i] * t2[s * K + f];
  }
}

__global__ void k_sum_fixed(long long m, const double* __restrict__ part, double* __restrict__ out) {
  __shared__ double s[1024];
  double acc = 0.0;
  for (long long i = threadIdx.x; i < m; i += 1024) acc += part[i];
  s[threadIdx.x] = acc;
  __syncthreads();
  for (int t = 512; t > 0; t >>= 1) {
    if (threadIdx.x < t) s[threadIdx.x] += s[threadIdx.x + t];
    __syncthreads();
  }
  if (threadIdx.x == 0) *out = s[0];
}

#define SF_QUAD_DISPATCH(K, Q, CALL)                                             \
  switch (K * 16 + Q) {                                                          \
    case 2 * 16 + 3: CALL(2, 3); break; case 2 * 16 + 4: CALL(2, 4); break;      \
    case 3 * 16 + 4: CALL(3, 4); break; case 3 * 16 + 5: CALL(3, 5); break;      \
    case 4 * 16 + 5: CALL(4, 5); break; case 4 * 16 + 6: CALL(4, 6); break;      \
    case 5 * 16 + 6: CALL(5, 6); break; case 5 * 16 + 7: CALL(5, 7); break;      \
    case 6 * 16 + 7: CALL(6, 7); break; case 6 * 16 + 8: CALL(6, 8); break;      \
    case 7 * 16 + 8: CALL(7, 8); break; case 7 * 16 + 9: CALL(7, 9); break;      \
    case 8 * 16 + 9: CALL(8, 9); break; case 8 * 16 + 10: CALL(8, 10); break;    \
    default: return invalid(what, "unsupported (degree, quadrature points): q must be k+2 or k+3"); \
  }

}  // namespace

extern "C" {

const char* sf_quad_last_error(void) { return g_err; }

int sf_quad_error(int k, int q, int n, int z0, int nzc, const double* u, const double* mats, const double* fq,
                  const double* w, double* part, double* out_dev, void* stream) {
  const char* what = "sf_quad_error";
  g_err[0] = 0;
  if (n < 1 || nzc < 0 || z0 < 0 || !mats || !w || !part || !out_dev || (nzc && (!u || !fq)))
    return invalid(what, "bad extent or null pointer");
  cudaStream_t st = (cudaStream_t)stream;
  if (nzc == 0) {
    k_sum_fixed<<<1, 1024, 0, st>>>(0, part, out_dev);
    return launched(what);
  }
  const int K = k + 1;
  const dim3 grid(n, n, nzc);
#define CALL(KK, QQ) k_quad_error<KK, QQ><<<grid, kThreads, 0, st>>>(n, nzc, u, mats, fq, w, z0, part)
  SF_QUAD_DISPATCH(K, q, CALL);
#undef CALL
  k_sum_fixed<<<1, 1024, 0, st>>>((long long)n * n * nzc, part, out_dev);
  return launched(what);
}

int sf_quad_load(int k, int q, int n, int z0, int nzc, const double* fq, const double* st_mat, const double* w,
                 double* b, void* stream) {
  const char* what = "sf_quad_load";
  g_err[0] = 0;
  if (n < 1 || nzc < 0 || z0 < 0 || !st_mat || !w || (nzc && (!fq || !b)))
    return invalid(what, "bad extent or null pointer");
  if (nzc == 0) return SF_OK;
  const int K = k + 1;
  const dim3 grid(n, n, nzc);
  cudaStream_t st = (cudaStream_t)stream;
#define CALL(KK, QQ) k_quad_load<KK, QQ><<<grid, kThreads, 0, st>>>(n, nzc, fq, st_mat, w, z0, b)
  SF_QUAD_DISPATCH(K, q, CALL);
#undef CALL
  return launched(what);
}

int sf_face_load(int k, int q, int n, int z0, int nzc, int axis, int side, const double* g, const double* st_mat,
                 const double* w, const double* coef, double* b, void* stream) {
  const char* what = "sf_face_load";
  g_err[0] = 0;
  if (n < 1 || nzc < 1 || z0 < 0 || axis < 0 || axis > 2 || (side != 0 && side != 1) || !g || !st_mat || !w ||
      !coef || !b)
    return invalid(what, "bad extent, face or null pointer");
  const int K = k + 1;
  const dim3 grid(n, axis == 2 ? n : nzc);
  cudaStream_t st = (cudaStream_t)stream;
#define CALL(KK, QQ) \
  k_face_load<KK, QQ><<<grid, kThreads, 0, st>>>(n, nzc, z0, axis, side, g, st_mat, w, coef, b)
  SF_QUAD_DISPATCH(K, q, CALL);
#undef CALL
  return launched(what);
}

}  // extern "C"
