// Bandwidth-bound vector kernels for the FGMRES outer loop and the V-cycle
// precision boundary (krylov.py:49-137, multigrid.py:262-266).  128-bit
// coalesced grid-stride loops; the dot product is a fixed-shape two-pass tree
// (no atomics), so repeated runs are bitwise identical (SPEC determinism).
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <cstdio>

#include "../../include/sumfact_b200.h"

namespace {

constexpr int kDotBlocks = SF_DOT_SCRATCH;
constexpr int kThreads = 256;

int grid_for(long long n, int per_thread) {
  long long blocks = (n / per_thread + kThreads - 1) / kThreads;
  if (blocks < 1) blocks = 1;
  if (blocks > 148 * 16) blocks = 148 * 16;
  return (int)blocks;
}

template <typename A, typename B>
__global__ void k_convert(long long n, const A* __restrict__ in, B* __restrict__ out) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    out[i] = (B)in[i];
}

__global__ void k_dot_partial(long long n, const double* __restrict__ x, const double* __restrict__ y,
                              double* __restrict__ part) {
  __shared__ double s[kThreads];
  double acc = 0.0;
  const long long stride = (long long)kDotBlocks * kThreads;
  // two independent accumulators per thread for ILP; fixed assignment -> deterministic
  double acc2 = 0.0;
  long long i = blockIdx.x * (long long)kThreads + threadIdx.x;
  for (; i + stride < n; i += 2 * stride) {
    acc = fma(x[i], y[i], acc);
    acc2 = fma(x[i + stride], y[i + stride], acc2);
  }
  if (i < n) acc = fma(x[i], y[i], acc);
  s[threadIdx.x] = acc + acc2;
  __syncthreads();
  for (int w = kThreads / 2; w > 0; w >>= 1) {
    if (threadIdx.x < w) s[threadIdx.x] += s[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) part[blockIdx.x] = s[0];
}

// Fused MGS step (krylov.py:73-84): w -= coef * x elementwise exactly as k_axpy_dev, and the partial sums of
// <y, w_new> (y = w when y == nullptr: the closing norm) in exactly k_dot_partial's element -> thread ->
// accumulator assignment, so the reduced value is bitwise the separate dot's.  One pass over w instead of two.
__global__ void k_axpy_dot_partial(long long n, double sign, const double* __restrict__ coef,
                                   const double* __restrict__ x, double* __restrict__ w, const double* __restrict__ y,
                                   double* __restrict__ part) {
  __shared__ double s[kThreads];
  const double a = sign * (*coef);
  double acc = 0.0, acc2 = 0.0;
  const long long stride = (long long)kDotBlocks * kThreads;
  long long i = blockIdx.x * (long long)kThreads + threadIdx.x;
  for (; i + stride < n; i += 2 * stride) {
    const double w0 = fma(a, x[i], w[i]), w1 = fma(a, x[i + stride], w[i + stride]);
    w[i] = w0;
    w[i + stride] = w1;
    acc = fma(y ? y[i] : w0, w0, acc);
    acc2 = fma(y ? y[i + stride] : w1, w1, acc2);
  }
  if (i < n) {
    const double w0 = fma(a, x[i], w[i]);
    w[i] = w0;
    acc = fma(y ? y[i] : w0, w0, acc);
  }
  s[threadIdx.x] = acc + acc2;
  __syncthreads();
  for (int t = kThreads / 2; t > 0; t >>= 1) {
    if (threadIdx.x < t) s[threadIdx.x] += s[threadIdx.x + t];
    __syncthreads();
  }
  if (threadIdx.x == 0) part[blockIdx.x] = s[0];
}

// Two dots sharing the right operand in one pass: <x1, y> and <x2, y>, each with k_dot_partial's order.
__global__ void k_dot2_partial(long long n, const double* __restrict__ x1, const double* __restrict__ x2,
                               const double* __restrict__ y, double* __restrict__ part1, double* __restrict__ part2) {
  __shared__ double s1[kThreads], s2[kThreads];
  double a1 = 0.0, a1b = 0.0, a2 = 0.0, a2b = 0.0;
  const long long stride = (long long)kDotBlocks * kThreads;
  long long i = blockIdx.x * (long long)kThreads + threadIdx.x;
  for (; i + stride < n; i += 2 * stride) {
    const double y0 = y[i], y1 = y[i + stride];
    a1 = fma(x1[i], y0, a1);
    a1b = fma(x1[i + stride], y1, a1b);
    a2 = fma(x2[i], y0, a2);
    a2b = fma(x2[i + stride], y1, a2b);
  }
  if (i < n) {
    a1 = fma(x1[i], y[i], a1);
    a2 = fma(x2[i], y[i], a2);
  }
  s1[threadIdx.x] = a1 + a1b;
  s2[threadIdx.x] = a2 + a2b;
  __syncthreads();
  for (int t = kThreads / 2; t > 0; t >>= 1) {
    if (threadIdx.x < t) {
      s1[threadIdx.x] += s1[threadIdx.x + t];
      s2[threadIdx.x] += s2[threadIdx.x + t];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    part1[blockIdx.x] = s1[0];
    part2[blockIdx.x] = s2[0];
  }
}

__global__ void k_dot_final(const double* __restrict__ part, double* __restrict__ out) {
  __shared__ double s[kDotBlocks];
  for (int i = threadIdx.x; i < kDotBlocks; i += blockDim.x) s[i] = part[i];
  __syncthreads();
  for (int w = kDotBlocks / 2; w > 0; w >>= 1) {
    for (int i = threadIdx.x; i < w; i += blockDim.x) s[i] += s[i + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) *out = s[0];
}

// y = x / d elementwise (IEEE division, as the reference's V = [b / beta], w / h_next, krylov.py:57,106)
// 16-byte accesses when both vectors are 16-byte aligned (the tail element, if any, by thread 0)
__global__ void k_div(long long n, const double* __restrict__ x, double d, double* __restrict__ y) {
  const long long stride = (long long)gridDim.x * blockDim.x, i0 = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if ((((unsigned long long)x | (unsigned long long)y) & 15) == 0) {
    const long long n2 = n >> 1;
    for (long long i = i0; i < n2; i += stride) {
      const double2 v = __ldg(reinterpret_cast<const double2*>(x) + i);
      reinterpret_cast<double2*>(y)[i] = make_double2(v.x / d, v.y / d);
    }
    if ((n & 1) && i0 == 0) y[n - 1] = x[n - 1] / d;
  } else {
    for (long long i = i0; i < n; i += stride) y[i] = x[i] / d;
  }
}

__global__ void k_axpy_dev(long long n, double sign, const double* __restrict__ coef, const double* __restrict__ x,
                           double* __restrict__ y) {
  const double a = sign * (*coef);
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    y[i] = fma(a, x[i], y[i]);
}

template <typename T>
__global__ void k_axpby(long long n, T alpha, const T* __restrict__ x, T beta, T* __restrict__ y) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    y[i] = beta == T(0) ? alpha * x[i] : fma(alpha, x[i], beta * y[i]);  // beta = 0 never reads y
}

// x = sum_i c_i v_i accumulated in term order exactly as x = 0; x = fma(c_i, v_i, 1.0 * x) (k_axpby with beta = 1),
// in one pass: reads the m vectors once and writes x once (krylov.py:120-124, the FGMRES solution update)
constexpr int kMaxTerms = SF_LINCOMB_MAX_TERMS;
struct LinComb {
  const double* v[kMaxTerms];
  double c[kMaxTerms];
};

__global__ void k_lincomb(long long n, int m, const LinComb lc, double* __restrict__ x) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    double acc = 0.0;
    for (int t = 0; t < m; ++t) acc = fma(lc.c[t], lc.v[t][i], 1.0 * acc);
    x[i] = acc;
  }
}

// y = A x for the coarse level's explicit inverse (A dense n x n fp64, row-major): one warp per row, lanes
// stride the columns, fixed xor-tree reduction (deterministic).  x is read in its storage type and, for the
// fp16 mode, demoted to binary16 first (multigrid.py:230-239: bs = demote16(bs)); y is rounded to its type.
template <typename X, typename Y>
__global__ void k_dense_apply(int n, const double* __restrict__ A, const X* __restrict__ x, int demote,
                              Y* __restrict__ y) {
  const int lane = threadIdx.x & 31;
  for (int row = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; row < n; row += (gridDim.x * blockDim.x) >> 5) {
    const double* a = A + (long long)row * n;
    double s = 0.0;
    for (int c = lane; c < n; c += 32) {
      double xv = (double)__ldg(&x[c]);
      if (demote) xv = (double)__half2float(__float2half_rn((float)xv));
      s = fma(__ldg(&a[c]), xv, s);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) y[row] = (Y)s;
  }
}

thread_local char g_err[256] = "";

// every entry point clears the buffer first, and every SF_EINVAL carries a message
int invalid(const char* what, const char* why) {
  snprintf(g_err, sizeof(g_err), "%s: %s", what, why);
  return SF_EINVAL;
}

int launched(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    snprintf(g_err, sizeof(g_err), "%s: %s", what, cudaGetErrorString(e));
    return SF_ECUDA;
  }
  return SF_OK;
}

}  // namespace

extern "C" {

const char* sf_vec_last_error(void) { return g_err; }

int sf_convert(long long n, const void* in, int in_dtype, void* out, int out_dtype, void* stream) {
  g_err[0] = 0;
  if (n < 0 || (!in && n) || (!out && n)) return invalid("sf_convert", "negative length or null vector");
  if (n == 0) return SF_OK;
  cudaStream_t st = (cudaStream_t)stream;
  int g = grid_for(n, 4);
  if (in_dtype == 0 && out_dtype == 1)
    k_convert<double, float><<<g, kThreads, 0, st>>>(n, (const double*)in, (float*)out);
  else if (in_dtype == 1 && out_dtype == 0)
    k_convert<float, double><<<g, kThreads, 0, st>>>(n, (const float*)in, (double*)out);
  else if (in_dtype == 0 && out_dtype == 0)
    k_convert<double, double><<<g, kThreads, 0, st>>>(n, (const double*)in, (double*)out);
  else if (in_dtype == 1 && out_dtype == 1)
    k_convert<float, float><<<g, kThreads, 0, st>>>(n, (const float*)in, (float*)out);
  else
    return invalid("sf_convert", "dtype codes must be 0 (f64) or 1 (f32)");
  return launched("sf_convert");
}

int sf_dot(long long n, const double* x, const double* y, double* out_dev, double* scratch, void* stream) {
  g_err[0] = 0;
  if (n < 0 || !out_dev || !scratch || (n && (!x || !y))) return invalid("sf_dot", "negative length or null pointer");
  cudaStream_t st = (cudaStream_t)stream;
  k_dot_partial<<<kDotBlocks, kThreads, 0, st>>>(n, x, y, scratch);
  k_dot_final<<<1, 1024, 0, st>>>(scratch, out_dev);
  return launched("sf_dot");
}

int sf_axpy_dot(long long n, double sign, const double* coef_dev, const double* x, double* w, const double* y,
                double* out_dev, double* scratch, void* stream) {
  g_err[0] = 0;
  if (n < 0 || !coef_dev || !out_dev || !scratch || (n && (!x || !w)))
    return invalid("sf_axpy_dot", "negative length or null pointer");
  cudaStream_t st = (cudaStream_t)stream;
  k_axpy_dot_partial<<<kDotBlocks, kThreads, 0, st>>>(n, sign, coef_dev, x, w, y, scratch);
  k_dot_final<<<1, 1024, 0, st>>>(scratch, out_dev);
  return launched("sf_axpy_dot");
}

int sf_dot2(long long n, const double* x1, const double* x2, const double* y, double* out1_dev, double* out2_dev,
            double* scratch2, void* stream) {
  g_err[0] = 0;
  if (n < 0 || !out1_dev || !out2_dev || !scratch2 || (n && (!x1 || !x2 || !y)))
    return invalid("sf_dot2", "negative length or null pointer");
  cudaStream_t st = (cudaStream_t)stream;
  k_dot2_partial<<<kDotBlocks, kThreads, 0, st>>>(n, x1, x2, y, scratch2, scratch2 + kDotBlocks);
  k_dot_final<<<1, 1024, 0, st>>>(scratch2, out1_dev);
  k_dot_final<<<1, 1024, 0, st>>>(scratch2 + kDotBlocks, out2_dev);
  return launched("sf_dot2");
}

int sf_lincomb(long long n, int m, const double* const* vecs, const double* coefs, double* out, void* stream) {
  g_err[0] = 0;
  if (n < 0 || !out) return invalid("sf_lincomb", "negative length or null output");
  if (m < 0 || m > kMaxTerms) return invalid("sf_lincomb", "term count must lie in [0, SF_LINCOMB_MAX_TERMS]");
  if (m && (!vecs || !coefs)) return invalid("sf_lincomb", "null term arrays");
  if (n == 0) return SF_OK;
  LinComb lc;
  for (int t = 0; t < m; ++t) {
    if (!vecs[t]) return invalid("sf_lincomb", "null term vector");
    lc.v[t] = vecs[t];
    lc.c[t] = coefs[t];
  }
  k_lincomb<<<grid_for(n, 4), kThreads, 0, (cudaStream_t)stream>>>(n, m, lc, out);
  return launched("sf_lincomb");
}

int sf_axpy_dev(long long n, double sign, const double* coef_dev, const double* x, double* y, void* stream) {
  g_err[0] = 0;
  if (n < 0 || !coef_dev || (n && (!x || !y))) return invalid("sf_axpy_dev", "negative length or null pointer");
  if (n == 0) return SF_OK;
  k_axpy_dev<<<grid_for(n, 4), kThreads, 0, (cudaStream_t)stream>>>(n, sign, coef_dev, x, y);
  return launched("sf_axpy_dev");
}

int sf_axpby(long long n, double alpha, const double* x, double beta, double* y, void* stream) {
  g_err[0] = 0;
  if (n < 0 || (n && (!x || !y))) return invalid("sf_axpby", "negative length or null vector");
  if (n == 0) return SF_OK;
  k_axpby<double><<<grid_for(n, 4), kThreads, 0, (cudaStream_t)stream>>>(n, alpha, x, beta, y);
  return launched("sf_axpby");
}

int sf_axpby_f32(long long n, float alpha, const float* x, float beta, float* y, void* stream) {
  g_err[0] = 0;
  if (n < 0 || (n && (!x || !y))) return invalid("sf_axpby_f32", "negative length or null vector");
  if (n == 0) return SF_OK;
  k_axpby<float><<<grid_for(n, 4), kThreads, 0, (cudaStream_t)stream>>>(n, alpha, x, beta, y);
  return launched("sf_axpby_f32");
}

int sf_div(long long n, const double* x, double d, double* y, void* stream) {
  g_err[0] = 0;
  if (n < 0 || (n && (!x || !y))) return invalid("sf_div", "negative length or null vector");
  if (n == 0) return SF_OK;
  k_div<<<grid_for(n, 4), kThreads, 0, (cudaStream_t)stream>>>(n, x, d, y);
  return launched("sf_div");
}

int sf_dense_apply(long long n, const double* A, const void* x, int x_dtype, int demote16, void* y, int y_dtype,
                   void* stream) {
  g_err[0] = 0;
  if (n < 0 || n > (1LL << 20) || (n && (!A || !x || !y)))
    return invalid("sf_dense_apply", "length outside [0, 2^20] or null pointer");
  if ((x_dtype != 0 && x_dtype != 1) || (y_dtype != 0 && y_dtype != 1))
    return invalid("sf_dense_apply", "dtype codes must be 0 (f64) or 1 (f32)");
  if (n == 0) return SF_OK;
  cudaStream_t st = (cudaStream_t)stream;
  const int nn = (int)n;
  long long blocks = (n * 32 + kThreads - 1) / kThreads;
  const int g = (int)(blocks < 148 * 8 ? blocks : 148 * 8);
  if (x_dtype == 0 && y_dtype == 0)
    k_dense_apply<double, double><<<g, kThreads, 0, st>>>(nn, A, (const double*)x, demote16, (double*)y);
  else if (x_dtype == 1 && y_dtype == 1)
    k_dense_apply<float, float><<<g, kThreads, 0, st>>>(nn, A, (const float*)x, demote16, (float*)y);
  else if (x_dtype == 0)
    k_dense_apply<double, float><<<g, kThreads, 0, st>>>(nn, A, (const double*)x, demote16, (float*)y);
  else
    k_dense_apply<float, double><<<g, kThreads, 0, st>>>(nn, A, (const float*)x, demote16, (double*)y);
  return launched("sf_dense_apply");
}

}  // extern "C"
