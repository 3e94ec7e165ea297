// mb_solve.cu -- throughput of the generic patch solve (solve_generic_sym, the
// fused sweep's reflection-basis Schur solve) in isolation: windows read from
// shared memory, results folded into a checksum, so the FP64 pipe utilisation of
// the solve's instruction stream alone can be compared with the sweep's.
//   PPT = patches per thread per iteration (1: as the sweep; 2: two windows whose
//   solves share every coefficient load), MINB = CTAs of 64 threads per SM.
#include "../include/svk.h"
#include <cuda_runtime.h>
#include <cstdio>
#include <cstring>
#include <vector>
#include "../paper_2401_06277_b200/csrc/stencil.cuh"
#include "../paper_2401_06277_b200/csrc/kernels_common.cuh"
#include "../paper_2401_06277_b200/csrc/sweep_fused.cuh"
using namespace svk;

template <int PPT, int MINB>
__global__ void __launch_bounds__(64, MINB) k_mb(const FusedFactors F, double* out, int iters) {
  __shared__ double win[32 * 51 * PPT];
  for (int q = threadIdx.x; q < 32 * 51 * PPT; q += 64) win[q] = 1e-3 * ((q * 7919) % 1000) - 0.5;
  __syncthreads();
  double acc = 0.0;
  for (int it = 0; it < iters; ++it) {
    double vx[PPT][25], vy[PPT][25], rp[PPT];
#pragma unroll
    for (int p = 0; p < PPT; ++p) {
      const double* w = win + (p * 32 + ((threadIdx.x + it) & 31)) * 51;
#pragma unroll
      for (int k = 0; k < 25; ++k) {
        vx[p][k] = w[k];
        vy[p][k] = w[25 + k];
      }
      rp[p] = w[50];
    }
#pragma unroll
    for (int p = 0; p < PPT; ++p) {
      const double dp = solve_generic_sym(vx[p], vy[p], rp[p], F);
      double s = dp;
#pragma unroll
      for (int k = 0; k < 25; ++k) s += vx[p][k] + vy[p][k];
      acc += s;
    }
  }
  if (acc == 1.2345) out[0] = acc;
}

template <int PPT, int MINB>
void run(const FusedFactors& F, int nsm) {
  double* out;
  cudaMalloc(&out, 8);
  const int iters = 2048 / PPT;
  const int blocks = nsm * MINB * 4;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float best = 1e9;
  for (int r = 0; r < 4; ++r) {
    cudaEventRecord(e0);
    k_mb<PPT, MINB><<<blocks, 64>>>(F, out, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (r && ms < best) best = ms;
  }
  cudaFuncAttributes a;
  cudaFuncGetAttributes(&a, k_mb<PPT, MINB>);
  const double solves = (double)blocks * 64 * iters * PPT;
  std::printf("{\"ppt\": %d, \"ctas_per_sm\": %d, \"regs\": %d, \"gsolves_per_s\": %.2f, \"err\": \"%s\"}\n", PPT, MINB,
              a.numRegs, solves / best / 1e6, cudaGetErrorString(cudaGetLastError()));
  cudaFree(out);
}

int main() {
  int nsm;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  FusedFactors F;
  double* f = reinterpret_cast<double*>(&F);
  for (int i = 0; i < (int)(sizeof(F) / 8); ++i) f[i] = 0.01 * ((i * 37) % 100) - 0.3;
  run<1, 4>(F, nsm);
  run<1, 6>(F, nsm);
  run<1, 8>(F, nsm);
  run<2, 4>(F, nsm);
  run<2, 3>(F, nsm);
  return 0;
}
