// mb_dmma_lat.cu -- latency of dependent mma.sync.m8n8k4.f64 (DMMA) and DFMA chains, one warp
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/mb_dmma_lat tools/mb_dmma_lat.cu
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}
template <int CH>
__global__ void k_lat(double a, double b, double* out, long long* cyc, int mode) {
  double d[CH][2];
  for (int c = 0; c < CH; ++c) d[c][0] = d[c][1] = threadIdx.x * 1e-3 + c;
  long long t0 = clock64();
  for (int it = 0; it < 128; ++it) {
#pragma unroll
    for (int c = 0; c < CH; ++c) {
      if (mode == 0) dmma(d[c][0], d[c][1], a, b);
      else { d[c][0] = fma(d[c][0], a, b); d[c][1] = fma(d[c][1], a, b); }
    }
  }
  long long t1 = clock64();
  double s = 0;
  for (int c = 0; c < CH; ++c) s += d[c][0] + d[c][1];
  out[threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
int main() {
  double* o; long long* c; cudaMalloc(&o, 1024 * 8); cudaMallocHost(&c, 8);
  for (int mode = 0; mode < 2; ++mode) {
#define RUN(CH) k_lat<CH><<<1, 32>>>(0.999, 1e-3, o, c, mode); cudaDeviceSynchronize(); k_lat<CH><<<1, 32>>>(0.999, 1e-3, o, c, mode); cudaDeviceSynchronize(); \
    printf("%s chains=%2d: %.1f cycles per step (%d ops per step)\n", mode ? "DFMA(2/lane)" : "DMMA", CH, c[0] / 128.0, CH);
    RUN(1) RUN(2) RUN(4) RUN(8) RUN(16)
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
