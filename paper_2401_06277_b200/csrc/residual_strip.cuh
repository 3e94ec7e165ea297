// residual_strip.cuh -- residual r = b - A x (alg:mg line 3), the FGMRES
// operator y = A x, and the fused residual + restriction r_c = P^T (b - A x)
// (alg:mg lines 3-4) as streaming strip kernels.
//
// Same machinery as the fused Vanka sweep (sweep_fused.cuh): a CTA of 128
// threads owns a strip of 120 node columns and a chunk of rows, x / p / b rows
// arrive by TMA into shared-memory rings, and `fused_residual` evaluates the
// stencil of two lattice rows and one pressure row per step into a residual
// ring.  The residual ring is then either written out (MODE 0) or restricted on
// the fly (MODE 1): coarse lattice row C needs fine rows 2C-3 .. 2C+3 (1D Q2
// interpolation transpose: weights -1/8, 3/8, 1, 3/8, -1/8 around an even coarse
// index, 3/4, 1, 3/4 around an odd one) and coarse pressure row C' fine rows
// 2C'-1 .. 2C'+1 (1/2, 1, 1/2), so the fine residual never touches HBM.
#pragma once
#include "sweep_fused.cuh"

namespace svk {

namespace rz {
constexpr int RR = 8;                         // residual ring rows (2C-3 .. 2C+3 plus the row being written)
constexpr int ORS = fz::ORS;
constexpr int ORP = ORS + RR * 2 * fz::W;
constexpr int OMB = ORP + 4 * fz::PWID;
constexpr int kSmemBytes = (OMB + 2) * 8;
}  // namespace rz

struct ResidArgs {
  LevelGeom g;   // fine level
  LevelGeom gc;  // coarse level (MODE 1)
  int chunk;     // rows per CTA: fine node rows (MODE 0) or coarse node rows (MODE 1)
  double* out;   // r / A x on the fine level (MODE 0) or r_c on the coarse level (MODE 1)
};

template <bool NOB, int MODE>
__global__ void __launch_bounds__(fz::kNT, 2) k_residual_strip(const ResidArgs R, const FusedFactors F,
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
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  // data of the first step: x pairs spB-1 .. spB+1, p rows spB .. spB+2, b pair spB, b_p row spB+1
  if (t == 0) {
    const unsigned bytes = 3 * fz::kXBytes + 3 * fz::kPBytes + (NOB ? 0u : fz::kBBytes + fz::kBPBytes);
    mbar_expect_tx(&bars[0], bytes);
    for (int p = spB - 1; p <= spB + 1; ++p) tma_load_3d(sm + xpair(p), &M.xv, xc0, 2 * p + 1, 0, &bars[0]);
    for (int r = spB; r <= spB + 2; ++r) tma_load_2d(sm + prow(r), &M.xp, pc0, r, &bars[0]);
    if (!NOB) {
      tma_load_3d(sm + bpair(spB), &M.bv, xc0 + 2, 2 * spB + 1, 0, &bars[0]);
      tma_load_2d(sm + bprow(spB + 1), &M.bp, kx0 - 2, spB + 1, &bars[0]);
    }
  }
  auto rrow8 = [&](int j, int c) { return rz::ORS + (j & (rz::RR - 1)) * 2 * fz::W + c * fz::W; };
  auto rprow4 = [&](int r) { return rz::ORP + (r & 3) * fz::PWID; };
  for (int sp = spB; sp <= spE; ++sp) {
    const int k = sp - spB;
    mbar_wait(&bars[k & 1], (phases >> (k & 1)) & 1u);
    phases ^= 1u << (k & 1);
    if (t == 0) {  // prefetch step sp+1: x pair sp+2, p row sp+3, b pair sp+1, b_p row sp+2
      uint64_t* nb = &bars[(k + 1) & 1];
      mbar_expect_tx(nb, fz::kXBytes + fz::kPBytes + (NOB ? 0u : fz::kBBytes + fz::kBPBytes));
      tma_load_3d(sm + xpair(sp + 2), &M.xv, xc0, 2 * sp + 5, 0, nb);
      tma_load_2d(sm + prow(sp + 3), &M.xp, pc0, sp + 3, nb);
      if (!NOB) {
        tma_load_3d(sm + bpair(sp + 1), &M.bv, xc0 + 2, 2 * sp + 3, 0, nb);
        tma_load_2d(sm + bprow(sp + 2), &M.bp, kx0 - 2, sp + 2, nb);
      }
    }
    fused_residual<false, NOB, rz::RR, rz::ORS, rz::ORP>(sm, g, F, sp, kx0);
    __syncthreads();
    if (MODE == 0) {
      // lattice rows 2sp+1, 2sp+2 and pressure row sp+1, owned columns only;
      // thread t < 120 owns node column kx0+t = ring columns 2t+4, 2t+5
      if (t < fz::kNOUT) {
        const int kx = kx0 + t, i0 = 2 * kx;
        const double sg = NOB ? -1.0 : 1.0;  // NOB: the ring holds -A x
#pragma unroll
        for (int rr = 1; rr <= 2; ++rr) {
          const int j = 2 * sp + rr;
          if (j < 2 * y0 || j >= 2 * y1 || j > lat - 1 || i0 >= g.pu) continue;
#pragma unroll
          for (int c = 0; c < 2; ++c) {
            const double2 v = lds2(sm + rrow8(j, c) + 2 * t + 4);
            *reinterpret_cast<double2*>(R.out + (c ? g.ouy : g.oux) + (int64_t)j * g.pu + i0) =
                make_double2(sg * v.x, sg * v.y);
          }
        }
        const int pr = sp + 1;
        if (pr >= y0 && pr < y1 && kx < g.pp) R.out[g.op + (int64_t)pr * g.pp + kx] = sg * sm[rprow4(pr) + t + 2];
      }
    } else {
      const LevelGeom& gc = R.gc;
      // coarse lattice row C = sp-1 is complete (fine rows 2C-3 .. 2C+3 = 2sp-5 .. 2sp+1)
      const int C = sp - 1;
      if (t < fz::kNOUT && C >= 2 * Y0 && C < 2 * Y1 && C <= gc.lat - 1) {
        const int c = kx0 + t;  // coarse lattice column; fine columns 2c-3 .. 2c+3 = ring 2t+1 .. 2t+7
        if (c < gc.pu) {
          const bool inside = C >= 1 && C <= gc.lat - 2 && c >= 1 && c <= gc.lat - 2;
          const int ro = (C & 1) ? 1 : 3;  // row offsets -ro .. ro
          const int co = (c & 1) ? 1 : 3;
#pragma unroll
          for (int comp = 0; comp < 2; ++comp) {
            double acc = 0.0;
            if (inside) {
#pragma unroll
              for (int dy = -3; dy <= 3; ++dy) {
                if (dy < -ro || dy > ro) continue;
                // 1D weights of P^T: even coarse index (-1/8, 0, 3/8, 1, 3/8, 0, -1/8); odd (3/4, 1, 3/4)
                const double wy = (C & 1) ? (dy == 0 ? 1.0 : 0.75)
                                          : (dy == 0 ? 1.0 : ((dy & 1) ? ((dy == -1 || dy == 1) ? 0.375 : -0.125) : 0.0));
                if (wy == 0.0) continue;
                const double* fr = sm + rrow8(2 * C + dy, comp) + 2 * t + 4;  // fine column 2c -> ring 2t+4
                double sx = 0.0;
                if (c & 1) {
                  sx = 0.75 * fr[-1] + fr[0] + 0.75 * fr[1];
                } else {
                  sx = -0.125 * fr[-3] + 0.375 * fr[-1] + fr[0] + 0.375 * fr[1] - 0.125 * fr[3];
                }
                acc = fma(wy, sx, acc);
              }
            }
            R.out[(comp ? gc.ouy : gc.oux) + (int64_t)C * gc.pu + c] = acc;
          }
        }
      }
      // coarse pressure row C' = sp/2 (fine rows sp-1 .. sp+1) for even sp
      if (!(sp & 1)) {
        const int Cp = sp >> 1;
        const int cp = (kx0 >> 1) + t;  // coarse node; fine nodes 2cp-1 .. 2cp+1 = r_p ring 2t+1 .. 2t+3
        if (t < fz::kNOUT / 2 && Cp >= Y0 && Cp < Y1 && Cp <= gc.N && cp < gc.pp) {
          double acc = 0.0;
          if (cp <= gc.N) {
#pragma unroll
            for (int dy = -1; dy <= 1; ++dy) {
              const double* fr = sm + rprow4(2 * Cp + dy) + 2 * t + 2;
              acc = fma(dy ? 0.5 : 1.0, 0.5 * fr[-1] + fr[0] + 0.5 * fr[1], acc);
            }
          }
          R.out[gc.op + (int64_t)Cp * gc.pp + cp] = acc;
        }
      }
    }
    __syncthreads();
  }
  mbar_wait(&bars[(spE - spB + 1) & 1], (phases >> ((spE - spB + 1) & 1)) & 1u);
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
  if (!make_vel_map(&M.xv, g, x) || !make_p_map(&M.xp, g, x, fz::PXW)) return -2;
  if (b && (!make_vel_map(&M.bv, g, b) || !make_p_map(&M.bp, g, b, fz::PWID))) return -2;
  const int ncover = (int)std::max<int64_t>(g.pu / 2, g.pp);
  const int nstrips = (ncover + fz::kNOUT - 1) / fz::kNOUT;
  ResidArgs R{g, gc ? *gc : g, 0, out};
  if (!gc) {
    R.chunk = fused_chunk(g, nstrips, nsm);
    const dim3 grid(nstrips, (g.r1 - g.r0 + R.chunk - 1) / R.chunk);
    if (b) k_residual_strip<false, 0><<<grid, fz::kNT, rz::kSmemBytes, s>>>(R, F, M);
    else k_residual_strip<true, 0><<<grid, fz::kNT, rz::kSmemBytes, s>>>(R, F, M);
  } else {
    if (!b) return -1;
    // coarse strips must cover the coarse pitch too: strip k owns coarse lattice columns [120k, 120k+120)
    const int ncov = (int)std::max<int64_t>(std::max<int64_t>(g.pu / 2, g.pp), gc->pu);
    const int ns = (ncov + fz::kNOUT - 1) / fz::kNOUT;
    R.chunk = std::max(1, fused_chunk(*gc, ns, nsm) / 2 + 1);
    const dim3 grid(ns, (gc->r1 - gc->r0 + R.chunk - 1) / R.chunk);
    k_residual_strip<false, 1><<<grid, fz::kNT, rz::kSmemBytes, s>>>(R, F, M);
  }
  return 0;
}

}  // namespace svk
