// Legacy tensor-path throughput on B200 (mma.sync f16 -> f32): m16n8k16 vs m16n8k8, and the
// mixed-precision FHFMA used by the binary16 split.  nvcc -gencode arch=compute_100a,code=sm_100a -O3
#include <cstdio>
#include <cuda_runtime.h>

template <int KIND>
__global__ void k(float* out, int iters) {
  float d[8][4] = {};
  unsigned a0 = threadIdx.x, a1 = a0 * 3, a2 = a0 * 5, a3 = a0 * 7, b0 = a0 ^ 0x3c003c00u, b1 = b0 + 1;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      if (KIND == 0)
        asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                     : "+f"(d[j][0]), "+f"(d[j][1]), "+f"(d[j][2]), "+f"(d[j][3])
                     : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
      else if (KIND == 1)
        asm volatile("mma.sync.aligned.m16n8k8.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};"
                     : "+f"(d[j][0]), "+f"(d[j][1]), "+f"(d[j][2]), "+f"(d[j][3])
                     : "r"(a0), "r"(a1), "r"(b0));
      else {
        unsigned short h = (unsigned short)(a0 + j);
#pragma unroll
        for (int q = 0; q < 4; ++q)
          asm volatile("fma.rn.f32.f16 %0, %1, %2, %0;" : "+f"(d[j][q]) : "h"(h), "h"((unsigned short)0xE800));
      }
    }
  }
  float s = 0;
#pragma unroll
  for (int j = 0; j < 8; ++j) s += d[j][0] + d[j][1] + d[j][2] + d[j][3];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int KIND>
void run(const char* name, float per_inst_flop) {
  float* out;
  cudaMalloc(&out, 148 * 8 * 512 * sizeof(float));
  int iters = 4096, blocks = 148 * 4, threads = 512;
  k<KIND><<<blocks, threads>>>(out, 16);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a);
  k<KIND><<<blocks, threads>>>(out, iters);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  int clk;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  double insts = (double)blocks * (threads / 32) * iters * 8 * (KIND == 2 ? 4 * 32 : 1);
  double cyc = ms * 1e-3 * clk * 1e3;
  printf("%s: %.3f ms, %.3f warp-inst/cycle/SM (at %d MHz nominal), %.1f TFLOP/s\n", name, ms, insts / cyc / 148 /
         (KIND == 2 ? 32 : 1), clk / 1000, insts * per_inst_flop / (ms * 1e-3) / 1e12);
  cudaFree(out);
}

int main() {
  run<0>("HMMA.16816.F32 (m16n8k16)", 16 * 8 * 16 * 2);
  run<1>("HMMA.1688.F32  (m16n8k8) ", 16 * 8 * 8 * 2);
  run<2>("FHFMA (fma.rn.f32.f16), thread-inst", 2);
  return 0;
}
