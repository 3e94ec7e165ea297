// DFMA throughput with coefficients streamed from the kernel-parameter constant bank
#include <cstdio>
#include <cuda_runtime.h>
template <int K> struct P { double c[K]; };
template <int K>
__global__ void __launch_bounds__(128) k(const P<K> p, double* out, int iters) {
  double x[8], a[16];
#pragma unroll
  for (int i = 0; i < 8; ++i) x[i] = threadIdx.x * 1e-3 + i;
#pragma unroll
  for (int i = 0; i < 16; ++i) a[i] = 0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int q = 0; q < K; ++q) a[q & 15] = fma(p.c[q], x[q & 7], a[q & 15]);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) s += a[i];
  if (s == 1.2345) out[0] = s;
}
template <int K> void run(int blocks_per_sm, int nsm) {
  P<K> p;
  for (int i = 0; i < K; ++i) p.c[i] = 1.0 + i * 1e-9;
  double* out; cudaMalloc(&out, 8);
  int iters = (1 << 20) / K;
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  float best = 1e9;
  for (int r = 0; r < 4; ++r) {
    cudaEventRecord(e0);
    k<K><<<nsm * blocks_per_sm, 128>>>(p, out, iters);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1); if (r && ms < best) best = ms;
  }
  double fl = 2.0 * K * (double)iters * 128 * nsm * blocks_per_sm;
  printf("K=%4d blocks/SM=%d: %.2f TFLOP/s\n", K, blocks_per_sm, fl / best / 1e9);
}
int main() {
  int nsm; cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  for (int b : {2, 4}) { run<32>(b, nsm); run<128>(b, nsm); run<256>(b, nsm); run<512>(b, nsm); run<1024>(b, nsm); }
  return 0;
}
