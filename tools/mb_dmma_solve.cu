// mb_dmma_solve.cu -- round-2 groundwork: the reflection-basis block products of
// the generic patch solve (EE 9x9, EO 6x6, OE 6x6, OO 4x4 per velocity component,
// DESIGN.md section 7) on the FP64 tensor path vs the DFMA path, operands in
// shared memory as a sweep kernel would hold them.
//
//   DFMA: one patch per lane, 50 transformed values loaded from shared memory,
//         338 FMAs with the block coefficients as kernel parameters, 50 stores.
//   DMMA: a quad of lanes per patch, 8 patches per mma.sync.m8n8k4.f64 (patches
//         along M, block inputs along K, block outputs along N), coefficients as
//         register-resident B fragments; per patch and component 11 DMMAs'
//         share; A fragments loaded from shared memory, D fragments stored back.
//
// Both variants process the same patches and the DMMA results are checked
// against the DFMA ones.  Prints patch solves per second for each.
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

struct Blocks {
  double ee[9][9], eo[6][6], oe[6][6], oo[4][4];
};
// block input / output positions in the transformed 25-vector (ty*5+tx)
__constant__ int c_pos[4][9] = {{0, 1, 2, 5, 6, 7, 10, 11, 12},
                                {3, 4, 8, 9, 13, 14, 0, 0, 0},
                                {15, 16, 17, 20, 21, 22, 0, 0, 0},
                                {18, 19, 23, 24, 0, 0, 0, 0, 0}};
__device__ __forceinline__ constexpr int nb_of(int blk) { return blk == 0 ? 9 : (blk == 3 ? 4 : 6); }
constexpr int kPatchesPerCTA = 128;  // 4 warps x 32 patches
constexpr int kStride = 53;          // doubles per patch-component row in smem (odd: fewer bank conflicts)

// static position tables (register-resident operands in the DFMA path)
template <int BLK>
__device__ __forceinline__ constexpr int posof(int q) {
  constexpr int P[4][9] = {{0, 1, 2, 5, 6, 7, 10, 11, 12},
                           {3, 4, 8, 9, 13, 14, 0, 0, 0},
                           {15, 16, 17, 20, 21, 22, 0, 0, 0},
                           {18, 19, 23, 24, 0, 0, 0, 0, 0}};
  return P[BLK][q];
}
template <int NB, int BLK>
__device__ __forceinline__ void mv(const double (&in)[25], double (&out)[25], const double (&B)[NB][NB]) {
  double s[NB];
#pragma unroll
  for (int r = 0; r < NB; ++r) s[r] = 0.0;
#pragma unroll
  for (int q = 0; q < NB; ++q) {
    const double x = in[posof<BLK>(q)];
#pragma unroll
    for (int r = 0; r < NB; ++r) s[r] = fma(B[r][q], x, s[r]);
  }
#pragma unroll
  for (int r = 0; r < NB; ++r) out[posof<BLK>(r)] = s[r];
}

__global__ void __launch_bounds__(128) k_dfma(const Blocks B, const double* __restrict__ gin, double* __restrict__ gout,
                                              int iters) {
  extern __shared__ double s_io[];  // in place: every block reads and writes only its own positions
  double* sout = s_io;
  double* sin_ = s_io;
  for (int q = threadIdx.x; q < kPatchesPerCTA * 2 * kStride; q += blockDim.x)
    sin_[q] = gin[(size_t)blockIdx.x * kPatchesPerCTA * 2 * kStride + q];
  __syncthreads();
  for (int it = 0; it < iters; ++it) {
    const int p = threadIdx.x;
#pragma unroll
    for (int c = 0; c < 2; ++c) {
      const double* in = sin_ + (p * 2 + c) * kStride;
      double* out = sout + (p * 2 + c) * kStride;
      double v[25], o[25];
#pragma unroll
      for (int k = 0; k < 25; ++k) v[k] = in[k];
      mv<9, 0>(v, o, B.ee);
      mv<6, 1>(v, o, B.eo);
      mv<6, 2>(v, o, B.oe);
      mv<4, 3>(v, o, B.oo);
#pragma unroll
      for (int k = 0; k < 25; ++k) out[k] = o[k];
    }
    __syncwarp();
  }
  __syncthreads();
  for (int q = threadIdx.x; q < kPatchesPerCTA * 2 * kStride; q += blockDim.x)
    gout[(size_t)blockIdx.x * kPatchesPerCTA * 2 * kStride + q] = sout[q];
}

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

// coefficient fragments: block blk, K-tile kt, N-tile nt: lane holds Blk[n][k] with
// k = 4 kt + (lane & 3), n = 8 nt + (lane >> 2) (zero outside the block)
__device__ __forceinline__ double coef(const Blocks& B, int blk, int k, int n) {
  const int nb = blk == 0 ? 9 : (blk == 3 ? 4 : 6);
  if (k >= nb || n >= nb) return 0.0;
  return blk == 0 ? B.ee[n][k] : blk == 1 ? B.eo[n][k] : blk == 2 ? B.oe[n][k] : B.oo[n][k];
}

__global__ void __launch_bounds__(128) k_dmma(const Blocks B, const double* __restrict__ gin, double* __restrict__ gout,
                                              int iters) {
  extern __shared__ double s_io[];  // in place: every block reads and writes only its own positions
  double* sout = s_io;
  double* sin_ = s_io;
  for (int q = threadIdx.x; q < kPatchesPerCTA * 2 * kStride; q += blockDim.x)
    sin_[q] = gin[(size_t)blockIdx.x * kPatchesPerCTA * 2 * kStride + q];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int qk = lane & 3, qm = lane >> 2;
  __syncthreads();
  // register-resident B fragments: EE 3 k-tiles x 2 n-tiles, EO/OE 2 x 1, OO 1 x 1
  double bee[3][2], beo[2], boe[2], boo;
#pragma unroll
  for (int kt = 0; kt < 3; ++kt)
#pragma unroll
    for (int nt = 0; nt < 2; ++nt) bee[kt][nt] = coef(B, 0, 4 * kt + qk, 8 * nt + qm);
#pragma unroll
  for (int kt = 0; kt < 2; ++kt) {
    beo[kt] = coef(B, 1, 4 * kt + qk, qm);
    boe[kt] = coef(B, 2, 4 * kt + qk, qm);
  }
  boo = coef(B, 3, qk, qm);
  __syncthreads();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int g = 0; g < 4; ++g) {  // 4 groups of 8 patches per warp
      const int p = warp * 32 + g * 8 + qm;
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        const double* in = sin_ + (p * 2 + c) * kStride;
        double* out = sout + (p * 2 + c) * kStride;
        auto A = [&](int blk, int k) {  // input k of block blk of patch p (0 beyond the block)
          return k < nb_of(blk) ? in[c_pos[blk][k]] : 0.0;
        };
        // EE: 2 n-tiles
        double d[2][2] = {{0.0, 0.0}, {0.0, 0.0}};
#pragma unroll
        for (int kt = 0; kt < 3; ++kt) {
          const double a = A(0, 4 * kt + qk);
          dmma(d[0][0], d[0][1], a, bee[kt][0]);
          dmma(d[1][0], d[1][1], a, bee[kt][1]);
        }
#pragma unroll
        for (int nt = 0; nt < 2; ++nt)
#pragma unroll
          for (int j = 0; j < 2; ++j) {
            const int n = 8 * nt + 2 * qk + j;
            if (n < 9) out[c_pos[0][n]] = d[nt][j];
          }
        // EO, OE, OO
        double e[2] = {0.0, 0.0}, f[2] = {0.0, 0.0}, h[2] = {0.0, 0.0};
#pragma unroll
        for (int kt = 0; kt < 2; ++kt) {
          dmma(e[0], e[1], A(1, 4 * kt + qk), beo[kt]);
          dmma(f[0], f[1], A(2, 4 * kt + qk), boe[kt]);
        }
        dmma(h[0], h[1], A(3, qk), boo);
#pragma unroll
        for (int j = 0; j < 2; ++j) {
          const int n = 2 * qk + j;
          if (n < 6) {
            out[c_pos[1][n]] = e[j];
            out[c_pos[2][n]] = f[j];
          }
          if (n < 4) out[c_pos[3][n]] = h[j];
        }
      }
    }
    __syncwarp();
  }
  __syncthreads();
  for (int q = threadIdx.x; q < kPatchesPerCTA * 2 * kStride; q += blockDim.x)
    gout[(size_t)blockIdx.x * kPatchesPerCTA * 2 * kStride + q] = sout[q];
}

int main() {
  int nsm;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  Blocks B;
  srand(1);
  auto rnd = [] { return (double)rand() / RAND_MAX - 0.5; };
  for (auto& r : B.ee) for (double& v : r) v = rnd();
  for (auto& r : B.eo) for (double& v : r) v = rnd();
  for (auto& r : B.oe) for (double& v : r) v = rnd();
  for (auto& r : B.oo) for (double& v : r) v = rnd();
  const int ctas = nsm * 2 * 8;  // 2 CTAs per SM x 8 waves
  const size_t n = (size_t)ctas * kPatchesPerCTA * 2 * kStride;
  double *in, *o1, *o2, *o3;
  cudaMalloc(&in, n * 8);
  cudaMalloc(&o3, n * 8);
  cudaMalloc(&o1, n * 8);
  cudaMalloc(&o2, n * 8);
  double* h = (double*)malloc(n * 8);
  for (size_t i = 0; i < n; ++i) h[i] = rnd();
  cudaMemcpy(in, h, n * 8, cudaMemcpyHostToDevice);
  cudaMemset(o1, 0, n * 8);
  cudaMemset(o2, 0, n * 8);
  const int iters = 2000;
  const int smem = kPatchesPerCTA * 2 * kStride * 8;
  cudaFuncSetAttribute(k_dfma, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(k_dmma, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  // correctness: one pass of each from the same input
  k_dfma<<<ctas, 128, smem>>>(B, in, o1, 1);
  k_dmma<<<ctas, 128, smem>>>(B, in, o2, 1);
  cudaDeviceSynchronize();
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float best[2] = {1e9f, 1e9f};
  for (int rep = 0; rep < 4; ++rep)
    for (int v = 0; v < 2; ++v) {
      cudaEventRecord(e0);
      if (v == 0) k_dfma<<<ctas, 128, smem>>>(B, in, o3, iters);
      else k_dmma<<<ctas, 128, smem>>>(B, in, o3, iters);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      if (rep && ms < best[v]) best[v] = ms;
    }
  double* a = (double*)malloc(n * 8);
  double* b = (double*)malloc(n * 8);
  cudaMemcpy(a, o1, n * 8, cudaMemcpyDeviceToHost);
  cudaMemcpy(b, o2, n * 8, cudaMemcpyDeviceToHost);
  double md = 0, ma = 0;
  for (size_t i = 0; i < n; ++i) {
    md = fmax(md, fabs(a[i] - b[i]));
    ma = fmax(ma, fabs(a[i]));
  }
  const double patches = (double)ctas * kPatchesPerCTA * iters;
  printf("{\"dfma_patch_solves_per_s\": %.4g, \"dmma_patch_solves_per_s\": %.4g, \"speedup\": %.3f, "
         "\"max_abs_diff\": %.3g, \"max_abs\": %.3g, \"err\": \"%s\"}\n",
         patches / (best[0] * 1e-3), patches / (best[1] * 1e-3), best[0] / best[1], md, ma,
         cudaGetErrorString(cudaGetLastError()));
  return 0;
}
