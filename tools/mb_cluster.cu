// mb_cluster.cu -- cost of a phase of the one-launch coarse V-cycle (small_cycle.cuh):
// a cluster of C CTAs x 256 threads runs P phases, each a cluster-wide loop over
// n points (K loads of the previous phase's output + 1 store per point) followed by
// barrier.cluster arrive.release / wait.acquire.  %globaltimer per phase.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/mb_cluster tools/mb_cluster.cu
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

__device__ __forceinline__ void csync(int mode) {
  if (mode == 0)
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
  else if (mode == 1)
    asm volatile("barrier.cluster.arrive.relaxed.aligned;\n\tbarrier.cluster.wait.aligned;\n" ::: "memory");
  else {
    asm volatile("fence.acq_rel.cluster;\n" ::: "memory");
    asm volatile("barrier.cluster.arrive.relaxed.aligned;\n\tbarrier.cluster.wait.aligned;\n" ::: "memory");
  }
}
__device__ __forceinline__ unsigned long long gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ unsigned crank() {
  unsigned r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}

__global__ void __launch_bounds__(256, 1) k_phases(double* a, double* b, int n, int K, int P, int mode,
                                                     unsigned long long* st) {
  const int nt = 16 * 256;  // launched with cluster 16
  const int gt = crank() * 256 + threadIdx.x;
  if (gt == 0) st[0] = gtime();
  for (int p = 0; p < P; ++p) {
    const double* src = (p & 1) ? b : a;
    double* dst = (p & 1) ? a : b;
    for (int q = gt; q < n; q += nt) {
      double s = 0.0;
#pragma unroll 8
      for (int k = 0; k < K; ++k) s += src[(q + 37 * k) % n];
      dst[q] = s * 0.5;
    }
    csync(mode);
    if (gt == 0) st[p + 1] = gtime();
  }
}

int main() {
  const int n = 1 << 14;
  double *a, *b;
  unsigned long long* st;
  cudaMalloc(&a, n * 8);
  cudaMalloc(&b, n * 8);
  cudaMemset(a, 0, n * 8);
  cudaMemset(b, 0, n * 8);
  cudaMallocHost(&st, 4096 * 8);
  cudaFuncSetAttribute(k_phases, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  for (int mode = 0; mode < 3; ++mode)
    for (int K : {0, 1, 25})
      for (int nn : {256, 2400, 16384}) {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(16);
        cfg.blockDim = dim3(256);
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = 16;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        const int P = 40;
        for (int rep = 0; rep < 2; ++rep) {
          cudaError_t e = cudaLaunchKernelEx(&cfg, k_phases, a, b, nn, K, P, mode, st);
          if (e != cudaSuccess) {
            printf("launch: %s\n", cudaGetErrorString(e));
            return 1;
          }
          cudaDeviceSynchronize();
        }
        printf("mode %d (%s) K=%2d n=%5d: %.2f us per phase (first %.2f)\n", mode,
               mode == 0 ? "arrive.release/wait.acquire" : mode == 1 ? "relaxed, no fence" : "fence.acq_rel.cluster + relaxed",
               K, nn, (st[P] - st[1]) / 1000.0 / (P - 1), (st[1] - st[0]) / 1000.0);
      }
  return 0;
}
