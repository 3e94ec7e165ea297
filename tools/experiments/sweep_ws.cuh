// MEASURED AND REJECTED (round 2; kept as a record, not built): at 4096^2 this
// kernel took 1.99 ms (2 CTAs/SM, 250 registers) and 2.56 ms (3 CTAs/SM, 168
// registers, spills) against 1.44 ms for k_vanka_fused: the solver warps are
// the critical path and fewer warps solve.  It was
// included from csrc/ and selected with SVK_SWEEP_WS=1.
//
// sweep_ws.cuh -- warp-specialised variant of the fused Vanka sweep (alg:vk,
// P:262-271; the same arithmetic as k_vanka_fused<false>, so the same results
// up to nothing: every value is computed by the same code in the same order).
//
// k_vanka_fused runs every phase of a step (residual, CTA barrier, patch solve,
// accumulation / output) in both of its warps; with 2 warps per scheduler the
// FP64 pipe idles whenever both are in an FP64-light phase (DESIGN.md section 7,
// profiles/r2_sweep_regions.txt).  Here a CTA of 3 warps splits the work:
//  * warp 2 (the residual warp) owns the TMA rings of x, p, b and computes the
//    residual rows of a step for all 128 ring columns (two column sets per
//    lane) into the residual ring, then arrives on res_full[step];
//  * warps 0 and 1 (the solver warps, the lane -> patch map of k_vanka_fused)
//    wait on res_full, copy their patch windows into registers, arrive on
//    consumed[step], solve, accumulate with warp shuffles and store x_out; the
//    x_in they add to is read from global memory (L2), not from the x ring.
// No CTA barrier: the residual warp runs up to two steps ahead (residual ring of
// 9 lattice rows, 4 pressure rows; it waits on consumed[step-3] before
// overwriting), so the three warps of a CTA -- and 12 warps per SM at 168
// registers -- drift freely and overlap their FP64-light and FP64-heavy phases.
// Step barriers are indexed (step - sB) & 3 with phase parity ((step - sB) >> 2) & 1,
// so no barrier is reused before every waiter has passed its previous phase.
#pragma once
#include "sweep_fused.cuh"

namespace svk {
namespace fw {
constexpr int kSolverWarps = fz::kWarps;           // 2: the patch layout of k_vanka_fused
constexpr int kNT = 32 * (kSolverWarps + 1);       // + the residual warp
#ifndef SVK_WS_MINB
#define SVK_WS_MINB 3
#endif
constexpr int kMinB = SVK_WS_MINB;                 // CTAs per SM (3: 9 warps, <= 224 registers; 4: 12 warps, 168)
constexpr int XPR = 4, PR = 4, BPR = 2, RR = 9, RPR = 4;
constexpr int OXS = 0;
constexpr int OPS = OXS + XPR * 4 * fz::WX;
constexpr int OBS = OPS + PR * fz::PXS;
constexpr int OBP = OBS + BPR * 4 * fz::W;
constexpr int ORS = OBP + 2 * fz::PWID;
constexpr int ORP = ORS + RR * 2 * fz::W;
constexpr int OMB = ORP + RPR * fz::PWID;           // 2 TMA + 4 res_full + 4 consumed mbarriers
constexpr int kSmemBytes = (OMB + 10) * 8;
static_assert((OPS * 8) % 128 == 0 && (OBS * 8) % 128 == 0 && (OBP * 8) % 128 == 0, "TMA smem alignment");
static_assert(kMinB * (kSmemBytes + 1024) <= 232448, "kMinB CTAs per SM");
}  // namespace fw

__device__ __forceinline__ int fw_xpair(int p) { return fw::OXS + (p & 3) * 4 * fz::WX; }
__device__ __forceinline__ int fw_prow(int r) { return fw::OPS + (r & 3) * fz::PXS; }
__device__ __forceinline__ int fw_bpair(int p) { return fw::OBS + (p & 1) * 4 * fz::W; }
__device__ __forceinline__ int fw_bprow(int r) { return fw::OBP + (r & 1) * fz::PWID; }
__device__ __forceinline__ int fw_rrow(int j, int c) { return fw::ORS + pmod(j, fw::RR) * 2 * fz::W + c * fz::W; }
__device__ __forceinline__ int fw_rprow(int r) { return fw::ORP + (r & 3) * fz::PWID; }
struct RingFw {
  static __device__ __forceinline__ int x(int j, int c) {
    return fw_xpair((j - 1) >> 1) + c * 2 * fz::WX + ((j - 1) & 1) * fz::WX;
  }
  static __device__ __forceinline__ int p(int r) { return fw_prow(r); }
  static __device__ __forceinline__ int b(int j, int c) {
    return fw_bpair((j - 1) >> 1) + c * 2 * fz::W + ((j - 1) & 1) * fz::W;
  }
  static __device__ __forceinline__ int bp(int r) { return fw_bprow(r); }
};
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}

// residual rows 2sp+1, 2sp+2 and pressure row sp+1 of ring column set t (0..63)
__device__ __forceinline__ void fw_residual_cols(double* sm, const LevelGeom& g, const FusedFactors& F, int sp,
                                                 int kx0, int t) {
  const RingFw rg{};
  ResWin w;
  load_res_win<0, 4, 0, 2>(sm, rg, sp, w, t);
  const ResVals R = residual_from_win<false, false, RingFw, false>(sm, g, F, sp, kx0, rg, w, t);
#pragma unroll
  for (int comp = 0; comp < 2; ++comp) {
    sts2(sm + fw_rrow(2 * sp + 1, comp) + 2 * t, R.u[comp][0], R.u[comp][1]);
    sts2(sm + fw_rrow(2 * sp + 2, comp) + 2 * t, R.u[comp][2], R.u[comp][3]);
  }
  sm[fw_rprow(sp + 1) + t] = R.p;
}

__global__ void __launch_bounds__(fw::kNT, fw::kMinB) k_vanka_fused_ws(const FusedArgs A, const FusedFactors F,
                                                                       const __grid_constant__ FusedMaps M,
                                                                       const double* __restrict__ xin) {
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
  uint64_t* tbar = reinterpret_cast<uint64_t*>(sm + fw::OMB);  // [2] TMA
  uint64_t* full = tbar + 2;                                    // [4] residual rows of a step written
  uint64_t* cons = tbar + 6;                                    // [4] a step's windows copied by the solvers
  if (t == 0) {
    mbar_init(&tbar[0], 1);
    mbar_init(&tbar[1], 1);
    for (int k = 0; k < 4; ++k) {
      mbar_init(&full[k], 32);
      mbar_init(&cons[k], 32 * fw::kSolverWarps);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  pdl_wait();

  if (warp == fw::kSolverWarps) {
    // ===================== residual warp =====================
    unsigned phases = 0u;
    // prologue: x pairs sB-3 .. sB, p rows sB-2 .. sB+1, b pairs sB-2, sB-1, b_p rows sB-1, sB
    if (lane == 0) {
      mbar_expect_tx(&tbar[0], 4 * fz::kXBytes + 4 * fz::kPBytes + 2 * fz::kBBytes + 2 * fz::kBPBytes);
      for (int p = sB - 3; p <= sB; ++p) tma_load_3d(sm + fw_xpair(p), &M.xv, xc0, 2 * p + 1, 0, &tbar[0]);
      for (int r = sB - 2; r <= sB + 1; ++r) tma_load_2d(sm + fw_prow(r), &M.xp, pc0, r, &tbar[0]);
      for (int p = sB - 2; p <= sB - 1; ++p) tma_load_3d(sm + fw_bpair(p), &M.bv, xc0 + 2, 2 * p + 1, 0, &tbar[0]);
      for (int r = sB - 1; r <= sB; ++r) tma_load_2d(sm + fw_bprow(r), &M.bp, kx0 - 2, r, &tbar[0]);
    }
    mbar_wait(&tbar[0], 0u);
    phases ^= 1u;
    for (int sp = sB - 2; sp <= sB - 1; ++sp) {
      fw_residual_cols(sm, g, F, sp, kx0, lane);
      fw_residual_cols(sm, g, F, sp, kx0, lane + 32);
    }
    __syncwarp();
    // data of step sB: x pair sB+1, p row sB+2, b pair sB, b_p row sB+1 -> tbar[1]
    if (lane == 0) {
      mbar_expect_tx(&tbar[1], fz::kXBytes + fz::kPBytes + fz::kBBytes + fz::kBPBytes);
      tma_load_3d(sm + fw_xpair(sB + 1), &M.xv, xc0, 2 * sB + 3, 0, &tbar[1]);
      tma_load_2d(sm + fw_prow(sB + 2), &M.xp, pc0, sB + 2, &tbar[1]);
      tma_load_3d(sm + fw_bpair(sB), &M.bv, xc0 + 2, 2 * sB + 1, 0, &tbar[1]);
      tma_load_2d(sm + fw_bprow(sB + 1), &M.bp, kx0 - 2, sB + 1, &tbar[1]);
    }
    for (int s = sB; s <= sE; ++s) {
      const int bi = (s - sB + 1) & 1;
      mbar_wait(&tbar[bi], (phases >> bi) & 1u);
      phases ^= 1u << bi;
      __syncwarp();  // every lane has finished step s-1 (the slots refilled below were read then)
      if (lane == 0 && s < sE) {  // data of step s+1: x pair s+2, p row s+3, b pair s+1, b_p row s+2
        uint64_t* nb = &tbar[bi ^ 1];
        mbar_expect_tx(nb, fz::kXBytes + fz::kPBytes + fz::kBBytes + fz::kBPBytes);
        tma_load_3d(sm + fw_xpair(s + 2), &M.xv, xc0, 2 * s + 5, 0, nb);
        tma_load_2d(sm + fw_prow(s + 3), &M.xp, pc0, s + 3, nb);
        tma_load_3d(sm + fw_bpair(s + 1), &M.bv, xc0 + 2, 2 * s + 3, 0, nb);
        tma_load_2d(sm + fw_bprow(s + 2), &M.bp, kx0 - 2, s + 2, nb);
      }
      // rows 2s+1, 2s+2 (and pressure row s+1) reuse the slots of step s-3's window
      if (s - 3 >= sB) {
        const int q = s - 3 - sB;
        mbar_wait(&cons[q & 3], (unsigned)((q >> 2) & 1));
      }
      fw_residual_cols(sm, g, F, s, kx0, lane);
      fw_residual_cols(sm, g, F, s, kx0, lane + 32);
      mbar_arrive(&full[(s - sB) & 3]);
    }
    return;
  }

  // ===================== solver warps =====================
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
  double wgt[2][2];  // [row parity][column parity], column mask folded in (as k_vanka_fused)
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int b = 0; b < 2; ++b)
      wgt[a][b] = (b ? cin1 : cin0)
                      ? (A.scalar_w ? A.omega : A.omega * (a ? 0.5 : 1.0 / 3.0) * (b ? 0.5 : 1.0 / 3.0))
                      : 0.0;
  const bool colout = owner && 2 * kxp < g.pu;
  const int64_t du = g.ouy - g.oux;
  for (int s = sB; s <= sE; ++s) {
    const int q = s - sB;
    mbar_wait(&full[q & 3], (unsigned)((q >> 2) & 1));
    double vx[25], vy[25];
    double dp = 0.0;
    const bool valid = kxp >= 0 && kxp <= N && s >= 0 && s <= N;
    const bool generic = kxp >= 2 && kxp <= N - 2 && s >= 2 && s <= N - 2;
    double rp = 0.0;
    if (valid && generic) {
#pragma unroll
      for (int oy = 0; oy < 5; ++oy) {  // window rows 2s-2+oy, columns 2kxp-2.. = ring columns 2pi ..
        const double* ru = sm + fw_rrow(2 * s - 2 + oy, 0) + 2 * pi;
        const double* rv = sm + fw_rrow(2 * s - 2 + oy, 1) + 2 * pi;
        const double2 u01 = lds2(ru), u23 = lds2(ru + 2), v01 = lds2(rv), v23 = lds2(rv + 2);
        vx[oy * 5 + 0] = u01.x; vx[oy * 5 + 1] = u01.y; vx[oy * 5 + 2] = u23.x; vx[oy * 5 + 3] = u23.y;
        vx[oy * 5 + 4] = ru[4];
        vy[oy * 5 + 0] = v01.x; vy[oy * 5 + 1] = v01.y; vy[oy * 5 + 2] = v23.x; vy[oy * 5 + 3] = v23.y;
        vy[oy * 5 + 4] = rv[4];
      }
      rp = sm[fw_rprow(s) + pi + 1];
    }
    mbar_arrive(&cons[q & 3]);  // this step's windows are in registers
    const int ny = s - 1;
    const bool rowout = colout && ny >= y0 && ny < y1;
    // x_in of this step's outputs from global memory (L2), issued before the solve
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
    const bool pout = owner && s >= y0 && s < y1 && kxp < g.pp;
    const double xpv = pout ? __ldg(xin + g.op + (int64_t)s * g.pp + kxp) : 0.0;
    if (valid && generic) {
      dp = solve_generic_sym(vx, vy, rp, F);
    } else if (valid) {  // precomputed by k_boundary_patches
      const int64_t nb = bd_count(N), bix = bd_index(kxp, s, N);
#pragma unroll
      for (int k = 0; k < 25; ++k) {
        vx[k] = A.bd[k * nb + bix];
        vy[k] = A.bd[(25 + k) * nb + bix];
      }
      dp = A.bd[50 * nb + bix];
    } else {
#pragma unroll
      for (int k = 0; k < 25; ++k) {
        vx[k] = 0.0;
        vy[k] = 0.0;
      }
    }
    if (pout) A.xout[g.op + (int64_t)s * g.pp + kxp] = kxp <= N ? fma(A.omega, dp, xpv) : 0.0;
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

inline int launch_fused_sweep_ws(const LevelGeom& g, const FusedFactors& F, const FusedArgs& A0, const double* xin,
                                 const double* b, int nsm, cudaStream_t s) {
  static bool attr_done[64] = {false};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev >= 0 && dev < 64 && !attr_done[dev]) {
    cudaFuncSetAttribute(k_vanka_fused_ws, cudaFuncAttributeMaxDynamicSharedMemorySize, fw::kSmemBytes);
    attr_done[dev] = true;
  }
  const int ncover = (int)std::max<int64_t>(g.pu / 2, g.pp);
  const int nstrips = (ncover + fz::kNOUT - 1) / fz::kNOUT;
  FusedArgs A = A0;
  A.chunk = fused_chunk(g, nstrips, nsm);
  FusedMaps M;
  std::memset(&M, 0, sizeof(M));
  if (!make_vel_map(&M.bv, g, b) || !make_p_map(&M.bp, g, b, fz::PWID)) return -2;
  if (!make_vel_map(&M.xv, g, xin, fz::WX) || !make_p_map(&M.xp, g, xin, fz::PXW)) return -2;
  const dim3 grid(nstrips, (g.r1 - g.r0 + A.chunk - 1) / A.chunk);
  launch_pdl(k_vanka_fused_ws, grid, dim3(fw::kNT), fw::kSmemBytes, s, A, F, M, xin);
  return 0;
}

}  // namespace svk
