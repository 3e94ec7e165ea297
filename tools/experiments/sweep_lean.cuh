// MEASURED AND REJECTED (round 2; kept as a record, not built): 2.07 ms at 4096^2
// with 5 CTAs/SM (200 registers, spills) and 1.76 ms at 4 CTAs/SM (254
// registers, no spills) against 1.44 ms for k_vanka_fused: reading b and the
// output's x_in with LDG instead of staging them by TMA costs more than the
// extra CTA buys.  It was included from csrc/ and selected with SVK_SWEEP_LEAN=1.
//
// sweep_lean.cuh -- the fused Vanka sweep (alg:vk) with leaner shared
// memory, so that 5 CTAs (10 warps) fit an SM instead of 4 (8 warps).
//
// Same strips, steps, residual, patch solve and owner-computes accumulation as
// k_vanka_fused<false> (sweep_fused.cuh); what moves out of shared memory:
//  * b (velocity and pressure) is read from global memory where the residual
//    uses it -- each value is used once, so a ring only staged it;
//  * x_in of the output rows (and of the pressure output) is read from global
//    memory (L2: TMA brought those rows on chip one to two steps earlier), so the
//    x ring need not keep the two row pairs behind the residual window: 5 pairs
//    instead of 6;
//  * the p ring keeps 5 rows (slot = row mod 5) instead of 8.
// 41 KB of rings per 2-warp CTA (56 KB before); registers <= 204 (5 CTAs per SM).
#pragma once
#include "sweep_fused.cuh"

namespace svk {
namespace fl {
constexpr int XPR = 5, PR = 5, RR = fz::RR, RPR = 4;
constexpr int OXS = 0;
constexpr int OPS = OXS + XPR * 4 * fz::WX;
constexpr int ORS = OPS + PR * fz::PXS;
constexpr int ORP = ORS + RR * 2 * fz::W;
constexpr int OMB = ORP + RPR * fz::PWID;  // 2 mbarriers
constexpr int kSmemBytes = (OMB + 2) * 8;
#ifndef SVK_LEAN_MINB
#define SVK_LEAN_MINB 5
#endif
constexpr int kMinB = SVK_LEAN_MINB;
#ifndef SVK_LEAN_MAXNREG
#define SVK_LEAN_MAXNREG 200
#endif
static_assert(kMinB * fz::kNT * SVK_LEAN_MAXNREG <= 65536, "registers for kMinB CTAs per SM");
static_assert((OPS * 8) % 128 == 0 && (ORS * 8) % 16 == 0, "TMA smem alignment");
static_assert(kMinB * (kSmemBytes + 1024) <= 232448, "kMinB CTAs per SM");
}  // namespace fl

__device__ __forceinline__ int fl_xpair(int p) { return fl::OXS + pmod(p, fl::XPR) * 4 * fz::WX; }
__device__ __forceinline__ int fl_prow(int r) { return fl::OPS + pmod(r, fl::PR) * fz::PXS; }
__device__ __forceinline__ int fl_rrow(int j, int c) { return fl::ORS + pmod(j, fl::RR) * 2 * fz::W + c * fz::W; }
__device__ __forceinline__ int fl_rprow(int r) { return fl::ORP + (r & 3) * fz::PWID; }
// ring adapter for the residual: x / p rows from shared memory, b from global memory
struct RingFl {
  const double* b;  // the level's b vector
  int64_t bux, buy, bpo, pu, pp;  // b planes (pointer offsets) and pitches
  int rc0;          // lattice column of residual column set 0 (2 kx0 - 4)
  int pc0;          // node column of pressure residual column 0 (kx0 - 2)
  __device__ __forceinline__ int x(int j, int c) const {
    return fl_xpair((j - 1) >> 1) + c * 2 * fz::WX + ((j - 1) & 1) * fz::WX;
  }
  __device__ __forceinline__ int p(int r) const { return fl_prow(r); }
  // The ring's columns cover the whole strip; columns / rows outside the grid
  // read 0 (their residuals are never used by a patch, as in the TMA zero fill).
  __device__ __forceinline__ double2 b2(const double*, int j, int c, int t, int lat) const {
    const int col = rc0 + 2 * t;
    if (j < 0 || j >= lat || col < 0 || col + 1 >= (int)pu) return make_double2(0.0, 0.0);
    return __ldg(reinterpret_cast<const double2*>(b + (c ? buy : bux) + (int64_t)j * pu + col));
  }
  __device__ __forceinline__ double bp1(const double*, int r, int t, int np) const {
    const int col = pc0 + t;
    if (r < 0 || r >= np || col < 0 || col >= np) return 0.0;
    return __ldg(b + bpo + (int64_t)r * pp + col);
  }
};
// bind the grid extents (the residual code calls b2 / bp1 with ring arguments only)
struct RingFlBound {
  RingFl r;
  int lat, np;
  __device__ __forceinline__ int x(int j, int c) const { return r.x(j, c); }
  __device__ __forceinline__ int p(int q) const { return r.p(q); }
  __device__ __forceinline__ double2 b2(const double* sm, int j, int c, int t) const { return r.b2(sm, j, c, t, lat); }
  __device__ __forceinline__ double bp1(const double* sm, int q, int t) const { return r.bp1(sm, q, t, np); }
};

// residual rows 2sp+1, 2sp+2 and pressure row sp+1 into the residual rings
__device__ __forceinline__ void fl_residual(double* sm, const LevelGeom& g, const FusedFactors& F, int sp, int kx0,
                                            const RingFlBound& rg, double (&pm)[3][3], bool first) {
  ResWin win;
  load_res_win<0, 4, 2, 2>(sm, rg, sp, win);  // x rows 0..4; p row 2 (rows 0..1 carried in pm)
  if (first) load_res_win<0, -1, 0, 1>(sm, rg, sp, win);
  else {
#pragma unroll
    for (int r = 0; r < 2; ++r)
#pragma unroll
      for (int q = 0; q < 3; ++q) win.Pm[r][q] = pm[r + 1][q];
  }
#pragma unroll
  for (int r = 0; r < 3; ++r)
#pragma unroll
    for (int q = 0; q < 3; ++q) pm[r][q] = win.Pm[r][q];
  const ResVals R = residual_from_win<false, false, RingFlBound, false>(sm, g, F, sp, kx0, rg, win);
  const int t = threadIdx.x;
#pragma unroll
  for (int comp = 0; comp < 2; ++comp) {
    sts2(sm + fl_rrow(2 * sp + 1, comp) + 2 * t, R.u[comp][0], R.u[comp][1]);
    sts2(sm + fl_rrow(2 * sp + 2, comp) + 2 * t, R.u[comp][2], R.u[comp][3]);
  }
  sm[fl_rprow(sp + 1) + t] = R.p;
}

// __maxnreg__ rather than __launch_bounds__(64, 5): ptxas then settles at 168
// registers (with spills), while 5 CTAs x 64 threads x 200 registers fit the SM
__global__ void __maxnreg__(SVK_LEAN_MAXNREG) k_vanka_fused_lean(const FusedArgs A, const FusedFactors F,
                                                                         const __grid_constant__ FusedMaps M,
                                                                         const double* __restrict__ xin,
                                                                         const double* __restrict__ bvec) {
  extern __shared__ __align__(1024) double sm[];
  const LevelGeom& g = A.g;
  const int N = g.N, lat = g.lat;
  const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
  const int kx0 = blockIdx.x * fz::kNOUT;
  const int y0 = g.r0 + blockIdx.y * A.chunk;
  const int y1 = min(y0 + A.chunk, g.r1);
  if (y0 >= y1) return;
  const int xc0 = 2 * kx0 - 6, pc0 = kx0 - 4;
  const int sB = y0 - 1, sE = y1;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sm + fl::OMB);
  unsigned phases = 0u;
  const RingFlBound rg{RingFl{bvec, g.oux, g.ouy, g.op, g.pu, g.pp, 2 * kx0 - 4, kx0 - 2}, lat, N + 1};

  if (t == 0) {
    mbar_init(&bars[0], 1);
    mbar_init(&bars[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  pdl_wait();
  // prologue: x pairs sB-3 .. sB+1 (rows 2sB-5 .. 2sB+4), p rows sB-2 .. sB+1 -> barrier 0
  if (t == 0) {
    mbar_expect_tx(&bars[0], 5 * fz::kXBytes + 4 * fz::kPBytes);
    for (int p = sB - 3; p <= sB + 1; ++p) tma_load_3d(sm + fl_xpair(p), &M.xv, xc0, 2 * p + 1, 0, &bars[0]);
    for (int r = sB - 2; r <= sB + 1; ++r) tma_load_2d(sm + fl_prow(r), &M.xp, pc0, r, &bars[0]);
  }
  mbar_wait(&bars[0], 0u);
  phases ^= 1u;
  {
    double pm0[3][3];
    fl_residual(sm, g, F, sB - 2, kx0, rg, pm0, true);
    fl_residual(sm, g, F, sB - 1, kx0, rg, pm0, true);
  }
  __syncthreads();
  // data of step sB: p row sB+2 -> barrier 1 (x pairs up to sB+1 are in)
  if (t == 0) {
    mbar_expect_tx(&bars[1], fz::kPBytes);
    tma_load_2d(sm + fl_prow(sB + 2), &M.xp, pc0, sB + 2, &bars[1]);
  }

  const int pi = fz::kOWN * warp + lane;
  const int kxp = kx0 - 1 + pi;
  const bool owner = lane >= 1 && lane <= fz::kOWN;
  double carry[3][2][2];
#pragma unroll
  for (int r = 0; r < 3; ++r)
#pragma unroll
    for (int c = 0; c < 2; ++c) carry[r][c][0] = carry[r][c][1] = 0.0;
  const int i0 = 2 * kxp;
  const bool cin0 = i0 >= 1 && i0 <= lat - 2, cin1 = i0 + 1 <= lat - 2;
  double wgt[2][2];
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int b = 0; b < 2; ++b)
      wgt[a][b] = (b ? cin1 : cin0)
                      ? (A.scalar_w ? A.omega : A.omega * (a ? 0.5 : 1.0 / 3.0) * (b ? 0.5 : 1.0 / 3.0))
                      : 0.0;
  const bool colout = owner && 2 * kxp < g.pu;
  const int64_t du = g.ouy - g.oux;
  double pmw[3][3];
  for (int s = sB; s <= sE; ++s) {
    // data of step s (x pair s+1, p row s+2) arrived on barrier (s-sB+1)&1; prefetch
    // step s+1 (x pair s+2 -> slot of pair s-3, read last by step s-2's residual;
    // p row s+3 -> slot of row s-2, read last by step s-2's residual: every thread
    // has passed the barrier of step s-1, so finished step s-1's residual)
    const int bi = (s - sB + 1) & 1;
    mbar_wait(&bars[bi], (phases >> bi) & 1u);
    phases ^= 1u << bi;
    if (t == (((s - sB) & 1) << 5) % fz::kNT && s < sE) {
      uint64_t* nbar = &bars[(s - sB) & 1];
      mbar_expect_tx(nbar, fz::kXBytes + fz::kPBytes);
      tma_load_3d(sm + fl_xpair(s + 2), &M.xv, xc0, 2 * s + 5, 0, nbar);
      tma_load_2d(sm + fl_prow(s + 3), &M.xp, pc0, s + 3, nbar);
    }
    fl_residual(sm, g, F, s, kx0, rg, pmw, s == sB);
    __syncthreads();

    double vx[25], vy[25];
    double dp = 0.0;
    const bool valid = kxp >= 0 && kxp <= N && s >= 0 && s <= N;
    const bool generic = kxp >= 2 && kxp <= N - 2 && s >= 2 && s <= N - 2;
    if (valid && generic) {
#pragma unroll
      for (int oy = 0; oy < 5; ++oy) {
        const double* ru = sm + fl_rrow(2 * s - 2 + oy, 0) + 2 * pi;
        const double* rv = sm + fl_rrow(2 * s - 2 + oy, 1) + 2 * pi;
        const double2 u01 = lds2(ru), u23 = lds2(ru + 2), v01 = lds2(rv), v23 = lds2(rv + 2);
        vx[oy * 5 + 0] = u01.x; vx[oy * 5 + 1] = u01.y; vx[oy * 5 + 2] = u23.x; vx[oy * 5 + 3] = u23.y;
        vx[oy * 5 + 4] = ru[4];
        vy[oy * 5 + 0] = v01.x; vy[oy * 5 + 1] = v01.y; vy[oy * 5 + 2] = v23.x; vy[oy * 5 + 3] = v23.y;
        vy[oy * 5 + 4] = rv[4];
      }
      dp = solve_generic_sym(vx, vy, sm[fl_rprow(s) + pi + 1], F);
    } else if (valid) {
      const int64_t nb = bd_count(N), bix = bd_index(kxp, s, N);
#pragma unroll
      for (int q = 0; q < 25; ++q) {
        vx[q] = A.bd[q * nb + bix];
        vy[q] = A.bd[(25 + q) * nb + bix];
      }
      dp = A.bd[50 * nb + bix];
    } else {
#pragma unroll
      for (int q = 0; q < 25; ++q) {
        vx[q] = 0.0;
        vy[q] = 0.0;
      }
    }
    const int ny = s - 1;
    const bool rowout = colout && ny >= y0 && ny < y1;
    // x_in of the outputs from global memory (L2), issued ahead of the shuffles
    double2 xo[2][2];
    if (rowout) {
#pragma unroll
      for (int c = 0; c < 2; ++c)
#pragma unroll
        for (int rr = 0; rr < 2; ++rr) {
          const int j = min(2 * ny + rr, lat - 1);
          xo[c][rr] = __ldg(reinterpret_cast<const double2*>(xin + g.oux + c * du + (int64_t)j * g.pu + i0));
        }
    }
    if (owner && s >= y0 && s < y1 && kxp < g.pp) {
      const double xp = __ldg(xin + g.op + (int64_t)s * g.pp + kxp);
      A.xout[g.op + (int64_t)s * g.pp + kxp] = kxp <= N ? fma(A.omega, dp, xp) : 0.0;
    }
    double* const ou_row = A.xout + g.oux + i0 + (int64_t)(2 * ny) * g.pu;
#pragma unroll
    for (int c = 0; c < 2; ++c) {
      const double* v = c ? vy : vx;
      double S0[5], S1[5];
#pragma unroll
      for (int oy = 0; oy < 5; ++oy) {
        const double r0 = __shfl_down_sync(0xffffffffu, v[oy * 5 + 0], 1);
        const double r1 = __shfl_down_sync(0xffffffffu, v[oy * 5 + 1], 1);
        const double l4 = __shfl_up_sync(0xffffffffu, v[oy * 5 + 4], 1);
        S0[oy] = oy < 3 ? carry[oy][c][0] + v[oy * 5 + 2] + l4 + r0 : v[oy * 5 + 2] + l4 + r0;
        S1[oy] = oy < 3 ? carry[oy][c][1] + v[oy * 5 + 3] + r1 : v[oy * 5 + 3] + r1;
      }
#pragma unroll
      for (int r = 0; r < 3; ++r) {
        carry[r][c][0] = S0[r + 2];
        carry[r][c][1] = S1[r + 2];
      }
      if (rowout) {
        double* const oc = ou_row + c * du;
#pragma unroll
        for (int rr = 0; rr < 2; ++rr) {
          const int j = 2 * ny + rr;
          if (j > lat - 1) continue;
          const bool jin = j >= 1 && j <= lat - 2;
          const double2 x = xo[c][rr];
          const double w0 = jin ? wgt[rr][0] : 0.0, w1 = jin ? wgt[rr][1] : 0.0;
          *reinterpret_cast<double2*>(oc + rr * g.pu) = make_double2(fma(w0, S0[rr], x.x), fma(w1, S1[rr], x.y));
        }
      }
    }
  }
}

inline int launch_fused_sweep_lean(const LevelGeom& g, const FusedFactors& F, const FusedArgs& A0, const double* xin,
                                   const double* b, int nsm, cudaStream_t s) {
  static bool attr_done[64] = {false};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev >= 0 && dev < 64 && !attr_done[dev]) {
    cudaFuncSetAttribute(k_vanka_fused_lean, cudaFuncAttributeMaxDynamicSharedMemorySize, fl::kSmemBytes);
    attr_done[dev] = true;
  }
  const int ncover = (int)std::max<int64_t>(g.pu / 2, g.pp);
  const int nstrips = (ncover + fz::kNOUT - 1) / fz::kNOUT;
  FusedArgs A = A0;
  A.chunk = fused_chunk(g, nstrips, nsm);  // (sized for 4 CTAs per SM; 5 fit)
  FusedMaps M;
  std::memset(&M, 0, sizeof(M));
  if (!make_vel_map(&M.xv, g, xin, fz::WX) || !make_p_map(&M.xp, g, xin, fz::PXW)) return -2;
  const dim3 grid(nstrips, (g.r1 - g.r0 + A.chunk - 1) / A.chunk);
  launch_pdl(k_vanka_fused_lean, grid, dim3(fz::kNT), fl::kSmemBytes, s, A, F, M, xin, b);
  return 0;
}

}  // namespace svk
