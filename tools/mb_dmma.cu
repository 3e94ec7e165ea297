// Does the FP64 tensor path (DMMA, mma.sync m8n8k4 f64) run beside the DFMA pipe?
// Measures DMMA-only, DFMA-only and mixed (half the warps each) throughput.
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}
// mode 0: all warps DMMA, 1: all warps DFMA, 2: even warps DMMA, odd warps DFMA
__global__ void k(int mode, int iters, double* out) {
  const int warp = threadIdx.x >> 5;
  const bool use_mma = mode == 0 || (mode == 2 && !(warp & 1));
  double acc[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) acc[i] = threadIdx.x * 1e-3 + i;
  const double a = 1.0000001, b = 0.9999999;
  if (use_mma) {
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int i = 0; i < 8; ++i) dmma(acc[2 * i], acc[2 * i + 1], a, b);
    }
  } else {
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int r = 0; r < 8; ++r)  // 8 x 16 = 128 FMA per thread = 8 DMMA-equivalents (256 FMA / 32 lanes each)
#pragma unroll
        for (int i = 0; i < 16; ++i) acc[i] = fma(acc[i], a, b);
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) s += acc[i];
  if (s == 1.2345) out[0] = s;
}

int main() {
  int nsm;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  double* out;
  cudaMalloc(&out, 8);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int iters = 1 << 14;
  for (int threads : {128, 256}) {
    for (int mode = 0; mode < 3; ++mode) {
      float best = 1e9;
      for (int r = 0; r < 4; ++r) {
        cudaEventRecord(e0);
        k<<<nsm * 4, threads>>>(mode, iters, out);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (r && ms < best) best = ms;
      }
      // per warp per iteration: DMMA 8 x 256 FMA, DFMA 128 x 32 FMA = 4096 FMA: equal work per warp
      const double fl = 2.0 * 4096.0 * iters * (threads / 32) * nsm * 4;
      printf("threads/CTA=%d mode=%s: %.2f TFLOP/s\n", threads, mode == 0 ? "DMMA " : mode == 1 ? "DFMA " : "mixed",
             fl / best / 1e9);
    }
  }
  return cudaGetLastError() == cudaSuccess ? 0 : 1;
}
