// residual_strip.cuh -- residual r = b - A x (alg:mg line 3), the FGMRES
// operator y = A x, and the fused residual + restriction r_c = P^T (b - A x)
// (alg:mg lines 3-4) as streaming strip kernels.
//
// Same machinery as the fused Vanka sweep (sweep_fused.cuh): a CTA of 128
// threads owns a strip of 120 node columns and a chunk of rows, x / p / b rows
// arrive by TMA into shared-memory rings, and `fused_residual_vals` evaluates the
// stencil of two lattice rows and one pressure row per step into registers.
// MODE 0 stores them directly; MODE 1 restricts them on the fly: coarse lattice
// row C needs fine rows 2C-3 .. 2C+3 (1D Q2 interpolation transpose: weights
// -1/8, 3/8, 1, 3/8, -1/8 around an even coarse index, 3/4, 1, 3/4 around an odd
// one) and coarse pressure row C' fine rows 2C'-1 .. 2C'+1 (1/2, 1, 1/2).  The x
// direction combines a thread's columns with its neighbours' odd columns (one
// exchange row per step), the y direction accumulates register carries over the
// coarse rows still open, so the fine residual never touches HBM or a ring.
#pragma once
#include "sweep_fused.cuh"

namespace svk {

// Rings of the residual kernels: TMA data two steps ahead (three mbarriers), so
// x keeps 6 row pairs (3 in use + 2 in flight), p 8 rows, b 4 pairs, b_p 4 rows.
namespace rz {
constexpr int XPR = 6;                        // x pairs (width fz::WX)
constexpr int OXS = 0;
constexpr int OPS = OXS + XPR * 4 * fz::WX;   // p rows (8), as the sweep
constexpr int OBS = OPS + 8 * fz::PXS;        // b pairs (4)
constexpr int OBP = OBS + 4 * 4 * fz::W;      // b_p rows (4)
constexpr int ORS = OBP + 4 * fz::PWID;       // MODE 1 exchange rows: [step parity][5][128]
constexpr int OMB = ORS + 2 * 5 * fz::kNT;    // 3 mbarriers
constexpr int kSmemBytes = (OMB + 4) * 8;
static_assert((OBS * 8) % 128 == 0 && (OBP * 8) % 128 == 0, "TMA smem alignment");
static_assert(fz::kMinB * (kSmemBytes + 1024) <= 232448, "kMinB CTAs per SM");
}  // namespace rz
__device__ __forceinline__ int rz_bpair(int p) { return rz::OBS + (p & 3) * 4 * fz::W; }
__device__ __forceinline__ int rz_prow(int r) { return rz::OPS + (r & 7) * fz::PXS; }
__device__ __forceinline__ int rz_xpair(int p) { return rz::OXS + pmod(p, rz::XPR) * 4 * fz::WX; }
struct RingRz {
  static __device__ __forceinline__ int x(int j, int c) {
    return rz_xpair((j - 1) >> 1) + c * 2 * fz::WX + ((j - 1) & 1) * fz::WX;
  }
  static __device__ __forceinline__ int p(int r) { return rz_prow(r); }
  static __device__ __forceinline__ int b(int j, int c) {
    return rz_bpair((j - 1) >> 1) + c * 2 * fz::W + ((j - 1) & 1) * fz::W;
  }
  static __device__ __forceinline__ int bp(int r) { return rz::OBP + (r & 3) * fz::PWID; }
  SVK_RING_B_FROM_SMEM
};

// the same ring with the x-pair slots of step sp advanced incrementally (RingFzS)
struct RingRzStep {
  RingSlots<rz::XPR, rz::OXS> S;
  int sp;
  __device__ __forceinline__ int x(int j, int c) const { return S.xr(j - 2 * sp, c); }
  __device__ __forceinline__ int p(int r) const { return rz_prow(r); }
  __device__ __forceinline__ int b(int j, int c) const { return RingRz::b(j, c); }
  __device__ __forceinline__ int bp(int r) const { return RingRz::bp(r); }
  SVK_RING_B_FROM_SMEM
};

struct ResidArgs {
  LevelGeom g;   // fine level
  LevelGeom gc;  // coarse level (MODE 1)
  int chunk;     // rows per CTA: fine node rows (MODE 0) or coarse node rows (MODE 1)
  double* out;   // r / A x on the fine level (MODE 0) or r_c on the coarse level (MODE 1)
};

template <bool NOB, int MODE>
__global__ void __launch_bounds__(fz::kNT, fz::kMinB) k_residual_strip(const ResidArgs R, const FusedFactors F,
                                                               const __grid_constant__ FusedMaps M) {
  extern __shared__ __align__(1024) double sm[];
  const LevelGeom& g = R.g;
  const int N = g.N, lat = g.lat;
  const int t = threadIdx.x;
  const int kx0 = blockIdx.x * fz::kNOUT;
  const int xc0 = 2 * kx0 - 6, pc0 = kx0 - 4;
  int spB, spE, Y0 = 0, Y1 = 0, y0 = 0, y1 = 0;
  if (MODE == 0) {
    y0 = g.r0 + blockIdx.y * R.chunk;
    y1 = min(y0 + R.chunk, g.r1);
    if (y0 >= y1) return;
    spB = y0 - 1;
    spE = y1 - 1;
  } else {
    Y0 = R.gc.r0 + blockIdx.y * R.chunk;
    Y1 = min(Y0 + R.chunk, R.gc.r1);
    if (Y0 >= Y1) return;
    spB = 2 * Y0 - 2;
    spE = 2 * Y1;
  }
  uint64_t* bars = reinterpret_cast<uint64_t*>(sm + rz::OMB);
  unsigned phases = 0u;  // bit b: parity of mbarrier b
  if (t == 0) {
    mbar_init(&bars[0], 1);
    mbar_init(&bars[1], 1);
    mbar_init(&bars[2], 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  pdl_wait();
  // data of step sp: x pairs up to sp+1, p rows up to sp+2, b pair sp, b_p row sp+1
  auto issue = [&](int sp, uint64_t* bar, bool first) {
    const unsigned nx = first ? 3 : 1;
    mbar_expect_tx(bar, nx * (fz::kXBytes + fz::kPBytes) + (NOB ? 0u : fz::kBBytes + fz::kBPBytes));
    for (int p = sp + 2 - (int)nx; p <= sp + 1; ++p) tma_load_3d(sm + rz_xpair(p), &M.xv, xc0, 2 * p + 1, 0, bar);
    for (int r = sp + 3 - (int)nx; r <= sp + 2; ++r) tma_load_2d(sm + rz_prow(r), &M.xp, pc0, r, bar);
    if (!NOB) {
      tma_load_3d(sm + rz_bpair(sp), &M.bv, xc0 + 2, 2 * sp + 1, 0, bar);
      tma_load_2d(sm + RingRz::bp(sp + 1), &M.bp, kx0 - 2, sp + 1, bar);
    }
  };
  if (t == 0) {  // the first two steps
    issue(spB, &bars[0], true);
    issue(spB + 1, &bars[1], false);
  }
  double rc_carry[2][3] = {{0.0, 0.0, 0.0}, {0.0, 0.0, 0.0}};  // MODE 1: open coarse rows sp-1 .. sp+1
  double pc_carry[2] = {0.0, 0.0};                              // MODE 1: open coarse pressure rows
  int slot = 0;                                                 // (sp - spB) % 3
  RingSlots<rz::XPR, rz::OXS> S = RingSlots<rz::XPR, rz::OXS>::at(spB);
  // stencil windows rolled across steps: x rows 2sp+2..2sp+4 and p rows sp+1..sp+2
  // of step sp are rows 0..2 / 0..1 of step sp+1, so each step loads 2 x rows and
  // 1 p row from shared memory instead of 5 and 3
  ResWin win;
  for (int sp = spB; sp <= spE; ++sp) {
    const RingRzStep rg{S, sp};
    auto step_residual = [&]() {
      if (sp == spB) load_res_win<0, 2, 0, 1>(sm, rg, sp, win);
      load_res_win<3, 4, 2, 2>(sm, rg, sp, win);
      return residual_from_win<false, NOB, RingRzStep, true>(sm, g, F, sp, kx0, rg, win);
    };
    mbar_wait(&bars[slot], (phases >> slot) & 1u);
    phases ^= 1u << slot;
    // prefetch step sp+2 (x pair sp+3 -> slot of sp-3, p row sp+4 -> slot of sp-4,
    // b pair sp+2 -> slot of sp-2, b_p row sp+3 -> slot of sp-1): every thread has
    // passed the barrier of step sp-1, i.e. finished the residual of step sp-1.
    const int nslot = slot == 0 ? 2 : slot - 1;  // (sp + 2 - spB) % 3
    if (t == (((sp - spB) & 1) << 5) % fz::kNT) issue(sp + 2, &bars[nslot], false);  // issuer alternates warps
    if (MODE == 0) {
      // lattice rows 2sp+1, 2sp+2 and pressure row sp+1 straight from registers:
      // thread t in [2, 122) owns node column kx0-2+t (lattice columns 2kx, 2kx+1)
      const ResVals V = step_residual();
      const int kx = kx0 - 2 + t, i0 = 2 * kx;
      if (t >= 2 && t < fz::kNOUT + 2) {
        const double sg = NOB ? -1.0 : 1.0;  // NOB: the values are -A x
#pragma unroll
        for (int rr = 0; rr < 2; ++rr) {
          const int j = 2 * sp + 1 + rr;
          if (j < 2 * y0 || j >= 2 * y1 || j > lat - 1 || i0 >= g.pu) continue;
#pragma unroll
          for (int c = 0; c < 2; ++c)
            *reinterpret_cast<double2*>(R.out + (c ? g.ouy : g.oux) + (int64_t)j * g.pu + i0) =
                make_double2(sg * V.u[c][2 * rr], sg * V.u[c][2 * rr + 1]);
        }
        const int pr = sp + 1;
        if (pr >= y0 && pr < y1 && kx < g.pp) R.out[g.op + (int64_t)pr * g.pp + kx] = sg * V.p;
      }
      __syncthreads();  // ring slots of x / p / b are reused by the next prefetch
    } else {
      // Restriction r_c = P^T r in registers: x first (the odd-column neighbours
      // come through a small double-buffered exchange row), then y with carries
      // over the three coarse lattice rows still open (like the sweep's
      // accumulation).  Thread t in [2, 122) owns coarse lattice column a =
      // kx0-2+t (its even fine column 2a sits on it) and, for even a, the coarse
      // pressure column a/2.  1D P^T weights around fine 2C: C even: -1/8, 3/8,
      // 1, 3/8, -1/8 at offsets -3, -1, 0, 1, 3; C odd: 3/4, 1, 3/4 at -1, 0, 1;
      // pressure: 1/2, 1, 1/2 around fine node 2C'.
      const ResVals V = step_residual();
      double* xb = sm + rz::ORS + (sp & 1) * 5 * fz::kNT;
      xb[0 * fz::kNT + t] = V.u[0][1];
      xb[1 * fz::kNT + t] = V.u[0][3];
      xb[2 * fz::kNT + t] = V.u[1][1];
      xb[3 * fz::kNT + t] = V.u[1][3];
      xb[4 * fz::kNT + t] = V.p;
      __syncthreads();
      const LevelGeom& gc = R.gc;
      const int a = kx0 - 2 + t;
      const int tm1 = max(t - 1, 0), tm2 = max(t - 2, 0), tp1 = min(t + 1, fz::kNT - 1);
      // y weights of fine rows j0 = 2sp+1 and j1 = 2sp+2 for coarse rows sp-1 .. sp+2
      const double w_m1 = ((sp - 1) & 1) ? 0.0 : -0.125;  // j0 = 2(sp-1)+3
      const double w_0 = (sp & 1) ? 0.75 : 0.375;         // j0 = 2sp+1
      const double w_p1 = ((sp + 1) & 1) ? 0.75 : 0.375;  // j0 = 2(sp+1)-1
      const double w_p2 = ((sp + 2) & 1) ? 0.0 : -0.125;  // j0 = 2(sp+2)-3
      const int C = sp - 1;  // coarse lattice row completed by this step
      const bool emit = t >= 2 && t < fz::kNOUT + 2 && C >= 2 * Y0 && C < 2 * Y1 && C <= gc.lat - 1 && a < gc.pu;
      const bool inside = C >= 1 && C <= gc.lat - 2 && a >= 1 && a <= gc.lat - 2;
#pragma unroll
      for (int comp = 0; comp < 2; ++comp) {
        double q[2];
#pragma unroll
        for (int rr = 0; rr < 2; ++rr) {
          const double* ro = xb + (comp * 2 + rr) * fz::kNT;
          const double e = V.u[comp][2 * rr], o1 = V.u[comp][2 * rr + 1], om1 = ro[tm1];
          q[rr] = (a & 1) ? e + 0.75 * (om1 + o1) : e + 0.375 * (om1 + o1) - 0.125 * (ro[tm2] + ro[tp1]);
        }
        const double done = rc_carry[comp][0] + w_m1 * q[0];
        rc_carry[comp][0] = rc_carry[comp][1] + w_0 * q[0];
        rc_carry[comp][1] = rc_carry[comp][2] + w_p1 * q[0] + q[1];
        rc_carry[comp][2] = w_p2 * q[0];
        if (emit) R.out[(comp ? gc.ouy : gc.oux) + (int64_t)C * gc.pu + a] = inside ? done : 0.0;
      }
      // pressure: fine node row nr = sp+1
      {
        const double qp = (a & 1) ? 0.0 : 0.5 * xb[4 * fz::kNT + tm1] + V.p + 0.5 * xb[4 * fz::kNT + tp1];
        const int nr = sp + 1;
        if (!(nr & 1)) {
          pc_carry[0] += qp;
        } else {
          const int Cp = (nr - 1) >> 1, cp = a >> 1;
          const double done = pc_carry[0] + 0.5 * qp;
          pc_carry[0] = pc_carry[1] + 0.5 * qp;
          pc_carry[1] = 0.0;
          if (!(a & 1) && t >= 2 && t < fz::kNOUT + 2 && Cp >= Y0 && Cp < Y1 && Cp <= gc.N && cp < gc.pp)
            R.out[gc.op + (int64_t)Cp * gc.pp + cp] = cp <= gc.N ? done : 0.0;
        }
      }
    }
    slot = slot == 2 ? 0 : slot + 1;
    S.advance();
    roll_res_win(win);
  }
  // the two last prefetches (steps spE+1, spE+2) must land before the shared memory is released
  mbar_wait(&bars[slot], (phases >> slot) & 1u);
  phases ^= 1u << slot;
  slot = slot == 2 ? 0 : slot + 1;
  mbar_wait(&bars[slot], (phases >> slot) & 1u);
}

// MODE 0: out = b - A x (NOB = false) or A x (NOB = true) on level g.
// MODE 1: out = P^T (b - A x) on the coarse level gc (Dirichlet rows zeroed).
inline int launch_residual_strip(const LevelGeom& g, const LevelGeom* gc, const FusedFactors& F, const double* x,
                                 const double* b, double* out, int nsm, cudaStream_t s) {
  static bool attr_done[64] = {false};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev >= 0 && dev < 64 && !attr_done[dev]) {
    cudaFuncSetAttribute(k_residual_strip<false, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, rz::kSmemBytes);
    cudaFuncSetAttribute(k_residual_strip<true, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, rz::kSmemBytes);
    cudaFuncSetAttribute(k_residual_strip<false, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, rz::kSmemBytes);
    attr_done[dev] = true;
  }
  FusedMaps M;
  std::memset(&M, 0, sizeof(M));
  if (!make_vel_map(&M.xv, g, x, fz::WX) || !make_p_map(&M.xp, g, x, fz::PXW)) return -2;
  if (b && (!make_vel_map(&M.bv, g, b) || !make_p_map(&M.bp, g, b, fz::PWID))) return -2;
  const int ncover = (int)std::max<int64_t>(g.pu / 2, g.pp);
  const int nstrips = (ncover + fz::kNOUT - 1) / fz::kNOUT;
  ResidArgs R{g, gc ? *gc : g, 0, out};
  if (!gc) {
    R.chunk = fused_chunk(g, nstrips, nsm);
    const dim3 grid(nstrips, (g.r1 - g.r0 + R.chunk - 1) / R.chunk);
    if (b) launch_pdl(k_residual_strip<false, 0>, grid, dim3(fz::kNT), rz::kSmemBytes, s, R, F, M);
    else launch_pdl(k_residual_strip<true, 0>, grid, dim3(fz::kNT), rz::kSmemBytes, s, R, F, M);
  } else {
    if (!b) return -1;
    // coarse strips must cover the coarse pitch too: strip k owns coarse lattice columns [120k, 120k+120)
    const int ncov = (int)std::max<int64_t>(std::max<int64_t>(g.pu / 2, g.pp), gc->pu);
    const int ns = (ncov + fz::kNOUT - 1) / fz::kNOUT;
    R.chunk = std::max(1, fused_chunk(*gc, ns, nsm) / 2 + 1);
    const dim3 grid(ns, (gc->r1 - gc->r0 + R.chunk - 1) / R.chunk);
    launch_pdl(k_residual_strip<false, 1>, grid, dim3(fz::kNT), rz::kSmemBytes, s, R, F, M);
  }
  return 0;
}

}  // namespace svk
