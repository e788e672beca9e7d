// FP64 / FP16 pipe micro-benchmark for B200 (sm_100a).
// Measures: DFMA throughput, DMMA (mma.sync.m8n8k4.f64) throughput, both
// interleaved in one kernel (are the pipes additive?), FFMA, and HMMA
// (mma.sync.m16n8k16 f16->f32).  Writes one line per test to stdout.
#include <cstdio>
#include <cuda_runtime.h>

#define ITERS 4096

__global__ void k_dfma(double* out, double s) {
  double a0 = threadIdx.x, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, a4 = a0 + 4, a5 = a0 + 5, a6 = a0 + 6, a7 = a0 + 7;
  const double m = s, c = 1e-9;
#pragma unroll 1
  for (int i = 0; i < ITERS; ++i) {
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      a0 = fma(a0, m, c); a1 = fma(a1, m, c); a2 = fma(a2, m, c); a3 = fma(a3, m, c);
      a4 = fma(a4, m, c); a5 = fma(a5, m, c); a6 = fma(a6, m, c); a7 = fma(a7, m, c);
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
}

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}

__global__ void k_dmma(double* out, double s) {
  double c[8][2];
#pragma unroll
  for (int i = 0; i < 8; ++i) { c[i][0] = 0; c[i][1] = 0; }
  double a = s * threadIdx.x, b = s + threadIdx.x;
#pragma unroll 1
  for (int i = 0; i < ITERS; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) dmma(c[j][0], c[j][1], a, b);
  }
  double t = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) t += c[i][0] + c[i][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = t;
}

__global__ void k_mixed(double* out, double s) {
  double c[4][2];
#pragma unroll
  for (int i = 0; i < 4; ++i) { c[i][0] = 0; c[i][1] = 0; }
  double a = s * threadIdx.x, b = s + threadIdx.x;
  double a0 = threadIdx.x, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3;
  const double m = s, cc = 1e-9;
#pragma unroll 1
  for (int i = 0; i < ITERS; ++i) {
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      dmma(c[j][0], c[j][1], a, b);
      a0 = fma(a0, m, cc); a1 = fma(a1, m, cc); a2 = fma(a2, m, cc); a3 = fma(a3, m, cc);
      a0 = fma(a0, m, cc); a1 = fma(a1, m, cc); a2 = fma(a2, m, cc); a3 = fma(a3, m, cc);
    }
  }
  double t = a0 + a1 + a2 + a3;
#pragma unroll
  for (int i = 0; i < 4; ++i) t += c[i][0] + c[i][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = t;
}

__global__ void k_ffma(float* out, float s) {
  float a[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) a[i] = threadIdx.x + i;
#pragma unroll 1
  for (int i = 0; i < ITERS; ++i) {
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
      for (int q = 0; q < 16; ++q) a[q] = fmaf(a[q], s, 1e-7f);
  }
  float t = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) t += a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = t;
}

__global__ void k_hmma(float* out, float s) {
  float c[8][4];
#pragma unroll
  for (int i = 0; i < 8; ++i) for (int j = 0; j < 4; ++j) c[i][j] = 0.f;
  unsigned a0 = 0x3c003c00u ^ threadIdx.x, a1 = a0, a2 = a0, a3 = a0, b0 = 0x3c003c00u, b1 = b0;
#pragma unroll 1
  for (int i = 0; i < ITERS; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j)
      asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
                   : "+f"(c[j][0]), "+f"(c[j][1]), "+f"(c[j][2]), "+f"(c[j][3])
                   : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
  }
  float t = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) for (int j = 0; j < 4; ++j) t += c[i][j];
  out[blockIdx.x * blockDim.x + threadIdx.x] = t * s;
}

template <typename F>
float time_it(F f) {
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  f(); cudaDeviceSynchronize();
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(e0); f(); cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
  }
  return best;
}

int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int blocks = sms * 8, threads = 256;
  double* dout; float* fout;
  cudaMalloc(&dout, sizeof(double) * blocks * threads);
  cudaMalloc(&fout, sizeof(float) * blocks * threads);
  double nthr = double(blocks) * threads;
  float ms;
  ms = time_it([&] { k_dfma<<<blocks, threads>>>(dout, 1.0000001); });
  printf("{\"test\":\"dfma\",\"ms\":%.4f,\"tflops\":%.3f}\n", ms, nthr * ITERS * 32 * 2 / (ms * 1e-3) / 1e12);
  ms = time_it([&] { k_dmma<<<blocks, threads>>>(dout, 1.0000001); });
  printf("{\"test\":\"dmma_m8n8k4\",\"ms\":%.4f,\"tflops\":%.3f}\n", ms, nthr / 32 * ITERS * 8 * 256 * 2 / (ms * 1e-3) / 1e12);
  ms = time_it([&] { k_mixed<<<blocks, threads>>>(dout, 1.0000001); });
  printf("{\"test\":\"dmma+dfma\",\"ms\":%.4f,\"tflops\":%.3f}\n", ms,
         (nthr / 32 * ITERS * 4 * 256 * 2 + nthr * ITERS * 32 * 2) / (ms * 1e-3) / 1e12);
  ms = time_it([&] { k_ffma<<<blocks, threads>>>(fout, 1.0000001f); });
  printf("{\"test\":\"ffma\",\"ms\":%.4f,\"tflops\":%.3f}\n", ms, nthr * ITERS * 64 * 2 / (ms * 1e-3) / 1e12);
  ms = time_it([&] { k_hmma<<<blocks, threads>>>(fout, 1.0f); });
  printf("{\"test\":\"hmma_m16n8k16_f32acc\",\"ms\":%.4f,\"tflops\":%.3f}\n", ms, nthr / 32 * ITERS * 8 * 4096 * 2 / (ms * 1e-3) / 1e12);
  cudaError_t err = cudaGetLastError();
  printf("{\"err\":\"%s\",\"sms\":%d}\n", cudaGetErrorString(err), sms);
  return 0;
}
