// krylov.cuh -- vector kernels for FGMRES: multi-dot products,
// multi-axpy and scaling over whole pitched vectors (padding entries are 0 and
// stay 0).  Reductions are deterministic: fixed grid, per-block partials, one
// fixed-order tree per result.
#pragma once
#include <cstdint>

namespace svk {

constexpr int kMaxM = 8;          // vectors per multi-dot / multi-axpy launch
constexpr int kRedThreads = 256;

struct VecPtrs {
  const double* p[kMaxM];
};

template <int M>
__device__ __forceinline__ void block_reduce_store(double (&acc)[M], double* __restrict__ partial, int stride) {
  __shared__ double sm[kRedThreads / 32][M];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
  for (int m = 0; m < M; ++m) {
    double v = acc[m];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
    if (lane == 0) sm[wid][m] = v;
  }
  __syncthreads();
  if (threadIdx.x < M) {
    double s = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) s += sm[w][threadIdx.x];
    partial[threadIdx.x * stride + blockIdx.x] = s;
  }
}

// partial[m*gridDim.x + block] = sum over this block's slice of v_m . w   (m < M)
template <int M>
__global__ void __launch_bounds__(kRedThreads) k_multidot(VecPtrs vs, int m_used, const double* __restrict__ w,
                                                          int64_t n, double* __restrict__ partial) {
  double acc[M];
#pragma unroll
  for (int m = 0; m < M; ++m) acc[m] = 0.0;
  const int64_t n2 = n >> 1;  // vectors are 16-byte aligned with even length
  const double2* w2 = reinterpret_cast<const double2*>(w);
  for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < n2; q += (int64_t)gridDim.x * blockDim.x) {
    const double2 wq = w2[q];
#pragma unroll
    for (int m = 0; m < M; ++m)
      if (m < m_used) {
        const double2 v = reinterpret_cast<const double2*>(vs.p[m])[q];
        acc[m] = fma(v.x, wq.x, acc[m]);
        acc[m] = fma(v.y, wq.y, acc[m]);
      }
  }
  block_reduce_store<M>(acc, partial, gridDim.x);
}

// out[m] (+)= sum_b partial[m*nb + b], one block per m, fixed order
__global__ void k_reduce_partials(const double* __restrict__ partial, int nb, double* __restrict__ out, int accumulate) {
  __shared__ double sm[kRedThreads];
  const int m = blockIdx.x;
  double s = 0.0;
  for (int b = threadIdx.x; b < nb; b += blockDim.x) s += partial[m * nb + b];
  sm[threadIdx.x] = s;
  __syncthreads();
  for (int o = blockDim.x / 2; o > 0; o >>= 1) {
    if (threadIdx.x < o) sm[threadIdx.x] += sm[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) out[m] = accumulate ? out[m] + sm[0] : sm[0];
}

// w += sign * sum_m coef[m] v_m   (coef in device memory)
__global__ void __launch_bounds__(256) k_multiaxpy(double* __restrict__ w, VecPtrs vs, int m_used,
                                                   const double* __restrict__ coef, double sign, int64_t n) {
  double c[kMaxM];
#pragma unroll
  for (int m = 0; m < kMaxM; ++m) c[m] = m < m_used ? sign * coef[m] : 0.0;
  const int64_t n2 = n >> 1;
  double2* w2 = reinterpret_cast<double2*>(w);
  for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < n2; q += (int64_t)gridDim.x * blockDim.x) {
    double2 a = w2[q];
#pragma unroll
    for (int m = 0; m < kMaxM; ++m)
      if (m < m_used) {
        const double2 v = reinterpret_cast<const double2*>(vs.p[m])[q];
        a.x = fma(c[m], v.x, a.x);
        a.y = fma(c[m], v.y, a.y);
      }
    w2[q] = a;
  }
}

// dst = alpha * src
__global__ void k_scale(double* __restrict__ dst, const double* __restrict__ src, double alpha, int64_t n) {
  for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < n; q += (int64_t)gridDim.x * blockDim.x)
    dst[q] = alpha * src[q];
}

}  // namespace svk

namespace svk {

// ---------------------------------------------------------------------------
// Fused classical Gram-Schmidt passes (CGS2) over a device array of basis
// pointers V[0..m), m <= kCgsMax.  Every pass reads each basis vector once:
//   k_cgs_dots  : part[i] = V_i . w                                   (i < m)
//   k_cgs_update: w_out = w - sum_i c_i V_i; DOTS: part[i] = V_i . w_out (i < m);
//                 always part[m] (DOTS) or part[0] = w_out . w_out
// Per-block partials (fixed grid) are reduced by k_reduce_partials in a fixed
// order, so results are deterministic.  One element per thread per iteration
// keeps the m basis values in registers between the update and the dots.
// ---------------------------------------------------------------------------
constexpr int kCgsMax = 32;
struct VecList {  // basis pointers by value (kernel-parameter space)
  const double* p[kCgsMax];
};

template <int MM>
__device__ __forceinline__ void block_reduce_store_n(const double (&acc)[MM], int m_used, double extra, int extra_at,
                                                     double* __restrict__ partial, int stride) {
  __shared__ double smr[kRedThreads / 32][MM + 1];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
  for (int m = 0; m <= MM; ++m) {
    const bool use = m < MM ? (m < m_used) : (extra_at >= 0);
    if (!use) continue;
    double v = m < MM ? acc[m] : extra;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
    if (lane == 0) smr[wid][m] = v;
  }
  __syncthreads();
  for (int m = threadIdx.x; m < m_used; m += blockDim.x) {
    double s = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) s += smr[w][m];
    partial[m * stride + blockIdx.x] = s;
  }
  if (extra_at >= 0 && threadIdx.x == 0) {
    double s = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) s += smr[w][MM];
    partial[extra_at * stride + blockIdx.x] = s;
  }
}

// part[i] = V_i . w for i < m <= MM (double2 streaming, high occupancy)
template <int MM>
__global__ void __launch_bounds__(kRedThreads) k_cgs_dots(const VecList V, int m, const double* __restrict__ w,
                                                          int64_t n, double* __restrict__ partial) {
  double acc[MM];
#pragma unroll
  for (int i = 0; i < MM; ++i) acc[i] = 0.0;
  const int64_t n2 = n >> 1;
  const double2* w2 = reinterpret_cast<const double2*>(w);
  for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < n2; q += (int64_t)gridDim.x * blockDim.x) {
    const double2 wq = w2[q];
#pragma unroll
    for (int i = 0; i < MM; ++i)
      if (i < m) {
        const double2 v = reinterpret_cast<const double2*>(V.p[i])[q];
        acc[i] = fma(v.x, wq.x, fma(v.y, wq.y, acc[i]));
      }
  }
  block_reduce_store_n<MM>(acc, m, 0.0, -1, partial, gridDim.x);
}

// w_out = w - sum_{i<m} c_i V_i (m <= kCgsMax); part[0] = w_out . w_out
__global__ void __launch_bounds__(kRedThreads) k_cgs_update(const VecList V, int m, const double* __restrict__ c,
                                                            const double* __restrict__ w, double* __restrict__ wout,
                                                            int64_t n, double* __restrict__ partial) {
  const int64_t n2 = n >> 1;
  const double2* w2 = reinterpret_cast<const double2*>(w);
  double2* o2 = reinterpret_cast<double2*>(wout);
  double nrm = 0.0;
  for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < n2; q += (int64_t)gridDim.x * blockDim.x) {
    double2 a = w2[q];
#pragma unroll 8
    for (int i = 0; i < m; ++i) {
      const double ci = __ldg(c + i);
      const double2 v = reinterpret_cast<const double2*>(V.p[i])[q];
      a.x = fma(-ci, v.x, a.x);
      a.y = fma(-ci, v.y, a.y);
    }
    o2[q] = a;
    nrm = fma(a.x, a.x, fma(a.y, a.y, nrm));
  }
  double dummy[1] = {0.0};
  block_reduce_store_n<1>(dummy, 0, nrm, 0, partial, gridDim.x);
}

// c[i] = raw[i] * scale[i]  (device), for i < m
__global__ void k_scale_coef(const double* __restrict__ raw, const double* __restrict__ scale, double* __restrict__ c,
                             int m) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < m) c[i] = raw[i] * scale[i];
}

}  // namespace svk
