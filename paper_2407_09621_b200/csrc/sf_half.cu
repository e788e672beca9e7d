// binary16 demotion primitives of the reference's precision module (precision.py:60-197), on the GPU with the
// same conversion the FP16 / FP16-EC kernels use (demote16 in sf_common.cuh: cvt.rn.f16.f32, round to nearest
// even, subnormals kept, overflow to inf).  NaN handling mirrors each reference function explicitly (the
// hardware conversion returns its own canonical NaN): to_half / from_half canonicalise (precision.py:104,125;
// from_half's NaNs come out positive),
// demote16 keeps the top payload bits like numpy's float16 cast (precision.py:130-137).
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

#include "../../include/sumfact_b200.h"
#include "sf_common.cuh"

namespace {

constexpr int kThreads = 256;
thread_local char g_err[256] = "";

int grid_for(long long n) {
  long long b = (n + kThreads - 1) / kThreads;
  if (b < 1) b = 1;
  if (b > 148 * 16) b = 148 * 16;
  return (int)b;
}

int launched(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    snprintf(g_err, sizeof(g_err), "%s: %s", what, cudaGetErrorString(e));
    return SF_ECUDA;
  }
  return SF_OK;
}

__device__ __forceinline__ unsigned short half_bits(float x) {  // precision.py:60-113
  const unsigned f = __float_as_uint(x);
  const unsigned short sign = (unsigned short)((f >> 16) & 0x8000u);
  if ((f & 0x7FFFFFFFu) > 0x7F800000u) return sign | 0x7E00u;  // canonical quiet NaN, sign kept
  return __half_as_ushort(__float2half_rn(x));
}

__device__ __forceinline__ float half_value(unsigned short h) {  // precision.py:116-127
  // NaN patterns: the reference forms sign * nan, which keeps the (positive) NaN operand -> 0x7FC00000 for both signs
  if ((h & 0x7C00u) == 0x7C00u && (h & 0x3FFu)) return __uint_as_float(0x7FC00000u);
  return __half2float(__ushort_as_half(h));
}

__device__ __forceinline__ float demote_np(float x) {  // numpy float32 -> float16 -> float32 (precision.py:130-137)
  const unsigned f = __float_as_uint(x);
  if ((f & 0x7FFFFFFFu) > 0x7F800000u) {
    unsigned hs = (f & 0x7FFFFFu) >> 13;
    if (hs == 0) hs = 1;  // stays a NaN
    return __uint_as_float((f & 0x80000000u) | 0x7F800000u | (hs << 13));
  }
  return sf::demote16(x);
}

__global__ void k_to_half(long long n, const float* __restrict__ x, unsigned short* __restrict__ h) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    h[i] = half_bits(x[i]);
}

__global__ void k_from_half(long long n, const unsigned short* __restrict__ h, float* __restrict__ x) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    x[i] = half_value(h[i]);
}

__global__ void k_demote16(long long n, const float* __restrict__ x, float* __restrict__ y) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    y[i] = demote_np(x[i]);
}

// precision.py:160-167: main = to_half(x); residual = to_half((x - from_half(main)) * 2^11) in fp32
__global__ void k_ec_split(long long n, const float* __restrict__ x, unsigned short* __restrict__ hm,
                           unsigned short* __restrict__ hr, int* __restrict__ bad) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const float v = x[i];
    if (!isfinite(v) || fabsf(v) > 65504.0f) atomicOr(bad, 1);  // HalfRangeError (checked on the host)
    const unsigned short m = half_bits(v);
    hm[i] = m;
    hr[i] = half_bits((v - half_value(m)) * sf::kEcScale);
  }
}

// precision.py:178-197: P = A_h B_h + (A_d B_h [left] + A_h B_d [right]) / 2^11, fp32 accumulation (ascending k;
// half x half products are exact in fp32).  One thread per output.
__global__ void k_ec_matmul(int m, int k, int n, const unsigned short* __restrict__ am,
                            const unsigned short* __restrict__ ar, const unsigned short* __restrict__ bm,
                            const unsigned short* __restrict__ br, int left, int right, float* __restrict__ out) {
  const long long id = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (id >= (long long)m * n) return;
  const int i = (int)(id / n), j = (int)(id % n);
  float p = 0.f, c1 = 0.f, c2 = 0.f;
  for (int q = 0; q < k; ++q) {
    const float a = half_value(am[(long long)i * k + q]), b = half_value(bm[(long long)q * n + j]);
    p = fmaf(a, b, p);
    if (left) c1 = fmaf(half_value(ar[(long long)i * k + q]), b, c1);
    if (right) c2 = fmaf(a, half_value(br[(long long)q * n + j]), c2);
  }
  const float corr = (0.f + c1) + c2;  // corr = zeros; corr += left; corr += right
  out[id] = p + corr / sf::kEcScale;
}

}  // namespace

extern "C" {

const char* sf_half_last_error(void) { return g_err; }

static int invalid(const char* what) {
  snprintf(g_err, sizeof(g_err), "%s: negative size, bad refine flag or null pointer", what);
  return SF_EINVAL;
}

int sf_to_half(long long n, const float* x, unsigned short* bits, void* stream) {
  g_err[0] = 0;
  if (n < 0 || (n && (!x || !bits))) return invalid("sf_to_half");
  if (n == 0) return SF_OK;
  k_to_half<<<grid_for(n), kThreads, 0, (cudaStream_t)stream>>>(n, x, bits);
  return launched("sf_to_half");
}

int sf_from_half(long long n, const unsigned short* bits, float* x, void* stream) {
  g_err[0] = 0;
  if (n < 0 || (n && (!x || !bits))) return invalid("sf_from_half");
  if (n == 0) return SF_OK;
  k_from_half<<<grid_for(n), kThreads, 0, (cudaStream_t)stream>>>(n, bits, x);
  return launched("sf_from_half");
}

int sf_demote16(long long n, const float* x, float* out, void* stream) {
  g_err[0] = 0;
  if (n < 0 || (n && (!x || !out))) return invalid("sf_demote16");
  if (n == 0) return SF_OK;
  k_demote16<<<grid_for(n), kThreads, 0, (cudaStream_t)stream>>>(n, x, out);
  return launched("sf_demote16");
}

int sf_ec_split(long long n, const float* x, unsigned short* main_bits, unsigned short* resid_bits, int* range_flag_dev,
                void* stream) {
  g_err[0] = 0;
  if (n < 0 || !range_flag_dev || (n && (!x || !main_bits || !resid_bits))) return invalid("sf_ec_split");
  if (n == 0) return SF_OK;
  k_ec_split<<<grid_for(n), kThreads, 0, (cudaStream_t)stream>>>(n, x, main_bits, resid_bits, range_flag_dev);
  return launched("sf_ec_split");
}

int sf_ec_matmul(int m, int k, int n, const unsigned short* a_main, const unsigned short* a_resid,
                 const unsigned short* b_main, const unsigned short* b_resid, int refine, float* out, void* stream) {
  g_err[0] = 0;
  if (m < 0 || k < 0 || n < 0 || refine < 0 || refine > 2) return invalid("sf_ec_matmul");
  if ((long long)m * n == 0) return SF_OK;
  if (!a_main || !a_resid || !b_main || !b_resid || !out) return invalid("sf_ec_matmul");
  const long long total = (long long)m * n;
  const int left = refine != 2, right = refine != 1;  // 0 both, 1 left, 2 right
  k_ec_matmul<<<(int)((total + kThreads - 1) / kThreads), kThreads, 0, (cudaStream_t)stream>>>(
      m, k, n, a_main, a_resid, b_main, b_resid, left, right, out);
  return launched("sf_ec_matmul");
}

}  // extern "C"
