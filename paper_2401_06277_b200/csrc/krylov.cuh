// krylov.cuh -- vector kernels for FGMRES: multi-dot products
// and multi-updates over the owned index segments of pitched vectors (padding
// entries are 0 and stay 0).  Reductions are deterministic: fixed grid, per-block partials, one
// fixed-order tree per result.
#pragma once
#include <cstdint>

namespace svk {

constexpr int kRedThreads = 256;

// out[m] (+)= sum_b partial[m*nb + b], one block per m, fixed order
__global__ void k_reduce_partials(const double* __restrict__ partial, int nb, double* __restrict__ out, int accumulate) {
  __shared__ double sm[kRedThreads];
  pdl_wait();
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
// Up to three contiguous index segments (in double2 units) of a vector: the
// owned rows of the u_x, u_y and p planes on a row slab, or the whole vector.
struct Seg3 {
  int64_t off2[3];
  int64_t cum2[4];
};
__device__ __forceinline__ int64_t seg_index(const Seg3& S, int64_t q) {
  // selects instead of a runtime index into the parameter (which would copy S to local memory)
  const bool a = q < S.cum2[1], b = q < S.cum2[2];
  const int64_t off = a ? S.off2[0] : (b ? S.off2[1] : S.off2[2]);
  const int64_t base = a ? 0 : (b ? S.cum2[1] : S.cum2[2]);
  return off + (q - base);
}

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
                                                          const Seg3 S, double* __restrict__ partial) {
  pdl_wait();
  double acc[MM];
#pragma unroll
  for (int i = 0; i < MM; ++i) acc[i] = 0.0;
  const int64_t n2 = S.cum2[3];
  const double2* w2 = reinterpret_cast<const double2*>(w);
  // KE elements per thread and pass (as k_cgs_update); elements past the ragged end
  // are masked by a zero weight vector entry
  constexpr int KE = MM <= 8 ? 4 : 2;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t q0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q0 < n2; q0 += KE * stride) {
    int64_t qq[KE];
    double2 wv[KE];
#pragma unroll
    for (int e = 0; e < KE; ++e) {
      const bool in = q0 + e * stride < n2;
      qq[e] = in ? seg_index(S, q0 + e * stride) : seg_index(S, q0);
      wv[e] = in ? w2[qq[e]] : make_double2(0.0, 0.0);
    }
#pragma unroll
    for (int i = 0; i < MM; ++i)
      if (i < m) {
        const double2* pv = reinterpret_cast<const double2*>(V.p[i]);
        double t = acc[i];
#pragma unroll
        for (int e = 0; e < KE; ++e) {
          const double2 v = pv[qq[e]];
          t = fma(v.x, wv[e].x, fma(v.y, wv[e].y, t));
        }
        acc[i] = t;
      }
  }
  block_reduce_store_n<MM>(acc, m, 0.0, -1, partial, gridDim.x);
}

// w_out = w - sum_{i<m} c_i V_i (m <= kCgsMax); part[0] = w_out . w_out
__global__ void __launch_bounds__(kRedThreads) k_cgs_update(const VecList V, int m, const double* __restrict__ c,
                                                            const double* __restrict__ w, double* __restrict__ wout,
                                                            const Seg3 S, double* __restrict__ partial) {
  pdl_wait();
  const int64_t n2 = S.cum2[3];
  const double2* w2 = reinterpret_cast<const double2*>(w);
  double2* o2 = reinterpret_cast<double2*>(wout);
  double nrm = 0.0;
  // KE elements per thread and pass: the per-vector pointer / coefficient loads are
  // shared and KE times the basis loads are in flight
  constexpr int KE = 4;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t q0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q0 < n2; q0 += KE * stride) {
    int64_t qq[KE];
    bool in[KE];
    double2 a[KE];
#pragma unroll
    for (int e = 0; e < KE; ++e) {
      in[e] = q0 + e * stride < n2;
      qq[e] = in[e] ? seg_index(S, q0 + e * stride) : seg_index(S, q0);
      a[e] = w2[qq[e]];
    }
#pragma unroll 4
    for (int i = 0; i < m; ++i) {
      const double ci = __ldg(c + i);
      const double2* pv = reinterpret_cast<const double2*>(V.p[i]);
#pragma unroll
      for (int e = 0; e < KE; ++e) {
        const double2 v = pv[qq[e]];
        a[e].x = fma(-ci, v.x, a[e].x);
        a[e].y = fma(-ci, v.y, a[e].y);
      }
    }
#pragma unroll
    for (int e = 0; e < KE; ++e)
      if (in[e]) {
        o2[qq[e]] = a[e];
        nrm = fma(a[e].x, a[e].x, fma(a[e].y, a[e].y, nrm));
      }
  }
  double dummy[1] = {0.0};
  block_reduce_store_n<1>(dummy, 0, nrm, 0, partial, gridDim.x);
}

// c[i] = raw[i] * scale[i]  (device), for i < m
__global__ void k_scale_coef(const double* __restrict__ raw, const double* __restrict__ scale, double* __restrict__ c,
                             int m) {
  pdl_wait();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < m) c[i] = raw[i] * scale[i];
}

}  // namespace svk
