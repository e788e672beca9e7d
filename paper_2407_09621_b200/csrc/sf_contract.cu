// Batched 1-D contraction, the reference's native kernel restated on the GPU:
//   out[o, i, r] = sum_k m[i, k] * u[o, k, r]      (src/_core/_contract.pyx:14-45)
// with the reference's exact arithmetic: ascending k, one rounded multiply and one
// rounded add per term (gcc -O3 without FMA contraction on the reference's x86 build),
// starting from 0 -- so fp64 and fp32 results are bitwise those of contract_f8 /
// contract_f4.  The precision modes of contract_mode (precision.py:206-230) are applied
// in-kernel: fp16 demotes both operands (RNE, subnormals kept), fp16_ec evaluates
// main = c(mh, uh), corr = c(dm, uh) + c(mh, du) and returns main + corr / 2048.
// This is the API-level drop-in for contract_batch; the hot path itself uses the fused
// tile kernels (sf_dmma.cu, sf_hmma.cu, sf_ops.cu).
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <cstdio>

#include "../../include/sumfact_b200.h"

namespace {

thread_local char g_err[256] = "";

__device__ __forceinline__ float d16(float x) { return __half2float(__float2half_rn(x)); }

template <typename T>
__device__ __forceinline__ T mul_rn(T a, T b);
template <>
__device__ __forceinline__ double mul_rn(double a, double b) { return __dmul_rn(a, b); }
template <>
__device__ __forceinline__ float mul_rn(float a, float b) { return __fmul_rn(a, b); }
template <typename T>
__device__ __forceinline__ T add_rn(T a, T b);
template <>
__device__ __forceinline__ double add_rn(double a, double b) { return __dadd_rn(a, b); }
template <>
__device__ __forceinline__ float add_rn(float a, float b) { return __fadd_rn(a, b); }

// one thread per (o, i, r) output; consecutive threads along r (inner, contiguous)
template <typename T, int MODE>
__global__ void k_contract(long long outer, int n, long long inner, int rows, const T* __restrict__ m,
                           const T* __restrict__ u, T* __restrict__ out) {
  const long long total = outer * rows * inner;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total;
       t += (long long)gridDim.x * blockDim.x) {
    const long long r = t % inner;
    const long long oi = t / inner;
    const int i = (int)(oi % rows);
    const long long o = oi / rows;
    const T* up = u + o * n * inner + r;
    const T* mp = m + (long long)i * n;
    if constexpr (MODE <= 1) {  // fp64 / fp32
      T acc = T(0);
      for (int k = 0; k < n; ++k) acc = add_rn(acc, mul_rn(mp[k], up[k * inner]));
      out[t] = acc;
    } else if constexpr (MODE == 2) {  // fp16: demoted operands, exact products, fp32 sums
      float acc = 0.f;
      for (int k = 0; k < n; ++k) acc = __fadd_rn(acc, __fmul_rn(d16(mp[k]), d16(up[k * inner])));
      out[t] = acc;
    } else {  // fp16_ec (precision.py:168-174, 224-229)
      float main = 0.f, c1 = 0.f, c2 = 0.f;
      for (int k = 0; k < n; ++k) {
        const float mv = mp[k], uv = up[k * inner];
        const float mh = d16(mv), uh = d16(uv);
        const float dm = d16(__fmul_rn(__fsub_rn(mv, mh), 2048.f));
        const float du = d16(__fmul_rn(__fsub_rn(uv, uh), 2048.f));
        main = __fadd_rn(main, __fmul_rn(mh, uh));
        c1 = __fadd_rn(c1, __fmul_rn(dm, uh));
        c2 = __fadd_rn(c2, __fmul_rn(mh, du));
      }
      out[t] = __fadd_rn(main, __fdiv_rn(__fadd_rn(c1, c2), 2048.f));
    }
  }
}

}  // namespace

extern "C" {

const char* sf_contract_last_error(void) { return g_err; }

int sf_contract(int mode, long long outer, int n, long long inner, int rows, const void* m, const void* u, void* out,
                void* stream) {
  g_err[0] = 0;
  auto invalid = [](const char* why) {
    snprintf(g_err, sizeof(g_err), "sf_contract: %s", why);
    return SF_EINVAL;
  };
  if (mode < 0 || mode > 3) return invalid("mode must be 0..3");
  if (outer < 0 || inner < 0 || n < 0 || rows < 0) return invalid("negative extent");
  const long long total = outer * rows * inner;
  if (total == 0) return SF_OK;
  if (!m || !u || !out) return invalid("null pointer");
  cudaStream_t st = (cudaStream_t)stream;
  long long blocks = (total + 255) / 256;
  if (blocks > 148 * 32) blocks = 148 * 32;
  switch (mode) {
    case 0: k_contract<double, 0><<<(int)blocks, 256, 0, st>>>(outer, n, inner, rows, (const double*)m,
                                                              (const double*)u, (double*)out); break;
    case 1: k_contract<float, 1><<<(int)blocks, 256, 0, st>>>(outer, n, inner, rows, (const float*)m,
                                                             (const float*)u, (float*)out); break;
    case 2: k_contract<float, 2><<<(int)blocks, 256, 0, st>>>(outer, n, inner, rows, (const float*)m,
                                                             (const float*)u, (float*)out); break;
    default: k_contract<float, 3><<<(int)blocks, 256, 0, st>>>(outer, n, inner, rows, (const float*)m,
                                                              (const float*)u, (float*)out); break;
  }
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    snprintf(g_err, sizeof(g_err), "sf_contract: %s", cudaGetErrorString(e));
    return SF_ECUDA;
  }
  return SF_OK;
}

}  // extern "C"
