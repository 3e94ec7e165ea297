// small_cycle.cuh -- the V-cycle's coarse levels (N <= SVK_SMALL_N, below the
// finest level) in ONE launch: one thread-block cluster runs alg:mg
// from the top small level down to the level-0 solve and back up, phase by
// phase, with a cluster barrier between dependent phases.
//
// Why: on the levels <= 256^2 every strip kernel of the V-cycle is latency-bound
// (8-15 us per launch whatever the level size, six launches per level: boundary
// patches, x = 0 sweep, residual + restriction, prolongation, boundary patches,
// sweep), so the levels 256^2 .. 4^2 cost ~0.4 ms of a ~5.4 ms 4096^2 V-cycle for
// ~0.1% of its work.  Here each phase is a cluster-wide grid-stride loop over
// points or patches of one level, and a phase boundary costs one cluster barrier
// (barrier.cluster arrive.release / wait.acquire, ~0.6 us: tools/mb_cluster.cu)
// instead of a kernel launch.  Measured: the levels 16^2,
// 8^2, 4^2 take 71 us in one launch against ~125 us as 13 launches; a phase costs
// 2-7 us here, so above 16^2 the per-kernel path is faster.
//
// Same operator, same steps as the strip kernels (alg:vk, alg:mg), in the
// unfused form of the paper's kernel split (alg:vk_kernels):
//   residual r = b - A x (masked, k_residual's stencils)            [phase]
//   patch solves delta_i = A_i^{-1} V_i r by the group's dense inverse on the
//     FP64 tensor path: one warp per (tile of <= 16 patches of one group, n8 tile
//     of the 51 slots), 13 k-steps of mma.sync.m8n8k4.f64 -- a warp issues a DMMA
//     only every ~25-35 cycles, so a tile's 7 slot tiles go to 7 warps  [phase]
//   x_out = x_in + W sum_i V_i^T delta_i (owner gathers, fixed order) [phase]
//   restriction r_c = P^T r, prolongation x += P e_c, level-0 min-norm solve.
// Point phases: one warp per lattice / pressure row (no 64-bit index division),
// every load of a point issued before its arithmetic; the stencil rows the lanes
// index by their own parity come from shared memory (divergent __constant__ reads
// serialise).  SVK_DEBUG_SMALL=2 (with SVK_GRAPHS=0) prints %globaltimer per phase.
// Data produced inside the launch is ordered by the barrier's release/acquire
// (the acquire invalidates the SM's L1), so phases read it with plain loads.
#pragma once

namespace svk {

constexpr int kScThreads = 256;
constexpr int kScMaxLevels = 9;

struct ScLevel {
  LevelGeom g;
  const double* dinv;   // the level's 25 padded group inverses
  const BdTile* tiles;  // every patch of the level in tiles (make_sc_tiles)
  int ntiles;
  double* b;  // right-hand side (top level: the caller's b; below: ws_b)
  double* x;  // iterate (top level: the caller's x; below: ws_x)
  double* r;  // residual workspace (ws_r)
};
struct ScArgs {
  ScLevel lv[kScMaxLevels];  // levels 0 .. top
  int top;
  double nu, omega;
  int scalar_w, nu_pre, nu_post, sweeps3;
  const double* cmat;        // level-0 bordered pseudo-inverse (k_coarse_build / k_coarse_invert)
  const int* cidx;
  int cni;
  double* d;                 // patch corrections, slot-major: d[s * np + p], np of the top level
  unsigned long long* stamps;  // development aid (SVK_DEBUG_SMALL=2): %globaltimer after each barrier
};

__device__ __forceinline__ void sc_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}
__device__ __forceinline__ unsigned sc_rank() {
  unsigned r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ unsigned sc_ncta() {
  unsigned r;
  asm volatile("mov.u32 %0, %%cluster_nctarank;" : "=r"(r));
  return r;
}

// loads of data written earlier in the launch: plain (L1-cached) loads -- the
// cluster barrier's acquire invalidates the L1 (CCTL.IVALL in the SASS)
#define LDX(p) (*(p))

// the 1D stencil rows the residual needs, copied from c_st into shared memory at
// kernel start: the lanes of a warp index them by their own lattice parity, and
// divergent __constant__ reads serialise (each distinct address is a separate
// constant-cache access, a miss an L2 round trip)
struct ScStencil {
  double KR[2][5], MR[2][5], CC[2][3], GC[2][3], CR[3][5], GR[3][5];
};

struct ScThreads {
  int gt, nt;  // cluster-wide thread index / count
  int gw, nw;  // cluster-wide warp index / count
  int lane;
};

// (L u)(i, j) + (B^T p)(i, j) at an interior lattice point with every load of the
// 5x5 / 3x3 windows issued up front (one memory round trip per point).  Same
// products and summation order as lap_at / gradp_at: the taps lap_at skips (odd
// parity: offsets +-2) carry the exact zeros KR[1][0,4] = MR[1][0,4] = 0, so the
// sum is bitwise the same; their clamped loads only keep addresses in range.
__device__ __forceinline__ double sc_ax_vel(const LevelGeom& g, const ScStencil& cs, double nu, const double* x, int plane,
                                            int i, int j) {
  const int pi = i & 1, pj = j & 1, lat = g.lat;
  const double* u = x + (plane ? g.ouy : g.oux);
  double U[5][5];
#pragma unroll
  for (int bb = 0; bb < 5; ++bb) {
    const int jj = min(max(j + bb - 2, 0), lat - 1);
#pragma unroll
    for (int aa = 0; aa < 5; ++aa) U[bb][aa] = u[(int64_t)jj * g.pu + min(max(i + aa - 2, 0), lat - 1)];
  }
  // B^T p: pressure nodes ky0 .. ky0+nky-1, kx0 .. kx0+nkx-1 (gradp_at)
  const int ky0 = pj ? (j - 1) >> 1 : (j >> 1) - 1, nky = pj ? 2 : 3;
  const int kx0 = pi ? (i - 1) >> 1 : (i >> 1) - 1, nkx = pi ? 2 : 3;
  double P[3][3];
#pragma unroll
  for (int ty = 0; ty < 3; ++ty)
#pragma unroll
    for (int tx = 0; tx < 3; ++tx)
      P[ty][tx] = x[g.op + (int64_t)min(ky0 + ty, g.N) * g.pp + min(kx0 + tx, g.N)];  // unused taps: clamped
  double s = 0.0;
#pragma unroll
  for (int bb = 0; bb < 5; ++bb) {
    const double my = cs.MR[pj][bb], ky = cs.KR[pj][bb];
#pragma unroll
    for (int aa = 0; aa < 5; ++aa) s += (my * cs.KR[pi][aa] + ky * cs.MR[pi][aa]) * U[bb][aa];
  }
  double sp = 0.0;
#pragma unroll
  for (int ty = 0; ty < 3; ++ty) {
    if (ty >= nky) continue;
    const double cy = plane == 0 ? cs.CC[pj][ty] : cs.GC[pj][ty];
    if (cy == 0.0) continue;
    double t = 0.0;
#pragma unroll
    for (int tx = 0; tx < 3; ++tx)
      if (tx < nkx) t += (plane == 0 ? cs.GC[pi][tx] : cs.CC[pi][tx]) * P[ty][tx];
    sp += cy * t;
  }
  return nu * s + -g.h * sp;
}
// (B u)(kx, ky) with the 5x5 windows of both components loaded up front (div_at order)
__device__ __forceinline__ double sc_ax_p(const LevelGeom& g, const ScStencil& cs, const double* x, int kx, int ky) {
  const int N = g.N, lat = g.lat;
  const int cx = kx == 0 ? 0 : (kx == N ? 2 : 1), cy = ky == 0 ? 0 : (ky == N ? 2 : 1);
  double U[5][5], V[5][5];
#pragma unroll
  for (int oy = 0; oy < 5; ++oy) {
    const int j = 2 * ky - 2 + oy;
#pragma unroll
    for (int ox = 0; ox < 5; ++ox) {
      const int i = 2 * kx - 2 + ox;
      const int64_t o = (int64_t)min(max(j, 0), lat - 1) * g.pu + min(max(i, 0), lat - 1);
      U[oy][ox] = x[g.oux + o];  // outside taps are skipped below; the clamped load keeps it in range
      V[oy][ox] = x[g.ouy + o];
    }
  }
  double s = 0.0;
#pragma unroll
  for (int oy = 0; oy < 5; ++oy) {
    const int j = 2 * ky - 2 + oy;
    if (j < 0 || j >= lat) continue;
    const double cyc = cs.CR[cy][oy], gyc = cs.GR[cy][oy];
#pragma unroll
    for (int ox = 0; ox < 5; ++ox) {
      const int i = 2 * kx - 2 + ox;
      if (i < 0 || i >= lat) continue;
      s += cyc * cs.GR[cx][ox] * U[oy][ox] + gyc * cs.CR[cx][ox] * V[oy][ox];
    }
  }
  return -g.h * s;
}

// every entry of a level vector: one warp per lattice / pressure row, lanes along
// the row (no 64-bit index division), fv(plane, j, i, offset) / fp(j, i, offset)
template <class Fv, class Fp>
__device__ __forceinline__ void sc_for_points(const LevelGeom& g, const ScThreads& T, Fv fv, Fp fp) {
  const int nrows = 2 * g.lat + g.N + 1;
  for (int row = T.gw; row < nrows; row += T.nw) {
    if (row < 2 * g.lat) {
      const int plane = row >= g.lat ? 1 : 0, j = row - plane * g.lat;
      const int64_t base = (plane ? g.ouy : g.oux) + (int64_t)j * g.pu;
      for (int i = T.lane; i < g.pu; i += 32) fv(plane, j, i, base + i);
    } else {
      const int j = row - 2 * g.lat;
      const int64_t base = g.op + (int64_t)j * g.pp;
      for (int i = T.lane; i < g.pp; i += 32) fp(j, i, base + i);
    }
  }
}

// r = b - A x (x == nullptr: r = b), masked to 0 on Dirichlet rows and padding (k_residual)
__device__ __noinline__ void sc_residual(const ScLevel& L, const ScStencil& cs, double nu, const double* x, double* r,
                                         const ScThreads& T) {
  const LevelGeom g = L.g;
  const double* b = L.b;
  const int N = g.N, lat = g.lat;
  sc_for_points(
      g, T,
      [&](int plane, int j, int i, int64_t o) {
        if (i >= lat || i == 0 || j == 0 || i == lat - 1 || j == lat - 1) {
          r[o] = 0.0;
          return;
        }
        const double bo = b[o];
        r[o] = x ? bo - sc_ax_vel(g, cs, nu, x, plane, i, j) : bo;
      },
      [&](int j, int i, int64_t o) {
        if (i > N) {
          r[o] = 0.0;
          return;
        }
        const double bo = b[o];
        r[o] = x ? bo - sc_ax_p(g, cs, x, i, j) : bo;
      });
}

// delta_i = A_i^{-1} V_i r for every patch of the level, slot-major into d: one
// warp per tile (<= 16 patches of one group; generic patches in row segments),
// D = R Ai^T on DMMA (patches along M, slots along N, window slots along K; as
// k_boundary_patches).  The straight-line reflection-basis solve of the strip
// kernels is not used here: executed once per thread it is instruction-fetch
// bound (~40 KB of code per phase), the DMMA tile loop is a few hundred bytes.
__device__ __noinline__ void sc_patches(const ScLevel& L, const double* r, double* d, const ScThreads& T) {
  const LevelGeom& g = L.g;
  const int N = g.N, lat = g.lat;
  const int64_t np = (int64_t)(N + 1) * (N + 1);
  const int gq = T.lane >> 2, t4 = T.lane & 3;
  // one task per (tile, n8 tile of slots): 13 k-steps, two independent m8 chains; DMMA
  // chains are latency-bound, so the 7 slot tiles of a tile go to 7 warps
  for (int task = T.gw; task < 7 * L.ntiles; task += T.nw) {
    const BdTile tl = L.tiles[task / 7];
    const int nt = task % 7;
    const double* Ai = L.dinv + (size_t)tl.grp * kGroupStride;
    double a[2][13], bf[13];
    const int sb = 8 * nt + gq;  // B[k][n] = Ai[n][k], n = slot
#pragma unroll
    for (int kt = 0; kt < 13; ++kt) {
      const int c = 4 * kt + t4;
      bf[kt] = (sb < kSlots && c < kSlots) ? __ldg(Ai + sb * kSlots + c) : 0.0;
    }
    // A fragments for patches gq and 8 + gq: window slot c of the patch
#pragma unroll
    for (int mt = 0; mt < 2; ++mt) {
      const int pi = 8 * mt + gq;
      const int kx = tl.kx + pi * tl.dx, ky = tl.ky + pi * tl.dy;
      const bool pin = pi < tl.n;
      const int kxc = pin ? kx : tl.kx, kyc = pin ? ky : tl.ky;  // a valid patch for the address
#pragma unroll
      for (int kt = 0; kt < 13; ++kt) {  // every load issued (clamped address), then masked
        const int c = 4 * kt + t4;
        int64_t off;
        bool ok;
        if (c < 50) {
          const int comp = c / 25, oy = (c % 25) / 5, ox = c % 5;
          const int i = 2 * kxc - 2 + ox, j = 2 * kyc - 2 + oy;
          ok = i >= 1 && j >= 1 && i <= lat - 2 && j <= lat - 2;  // Dirichlet / outside: not a patch unknown
          off = (comp ? g.ouy : g.oux) + (int64_t)min(max(j, 0), lat - 1) * g.pu + min(max(i, 0), lat - 1);
        } else {
          ok = c == 50;
          off = p_at(g, kxc, kyc);
        }
        const double v = LDX(r + off);
        a[mt][kt] = (pin && ok) ? v : 0.0;
      }
    }
    double acc[2][2] = {{0.0, 0.0}, {0.0, 0.0}};
#pragma unroll
    for (int kt = 0; kt < 13; ++kt) {
      dmma_m8n8k4(acc[0][0], acc[0][1], a[0][kt], bf[kt]);
      dmma_m8n8k4(acc[1][0], acc[1][1], a[1][kt], bf[kt]);
    }
#pragma unroll
    for (int mt = 0; mt < 2; ++mt)
#pragma unroll
      for (int jj = 0; jj < 2; ++jj) {
        const int pi = 8 * mt + gq, s = 8 * nt + 2 * t4 + jj;  // C[m][n]: m = patch, n = slot
        if (pi >= tl.n || s >= kSlots) continue;
        const int kx = tl.kx + pi * tl.dx, ky = tl.ky + pi * tl.dy;
        d[(int64_t)s * np + (int64_t)ky * (N + 1) + kx] = acc[mt][jj];
      }
  }
}

// x_out = x_in + W sum_i V_i^T delta_i, in place (k_vanka_update; xzero: x_in = 0)
__device__ __noinline__ void sc_update(const ScLevel& L, double omega, int scalar_w, bool xzero, const double* d,
                                       const ScThreads& T) {
  const LevelGeom g = L.g;
  const int N = g.N, lat = g.lat;
  const int64_t np = (int64_t)(N + 1) * (N + 1);
  double* x = L.x;
  sc_for_points(
      g, T,
      [&](int plane, int j, int i, int64_t o) {
        if (i >= lat) {
          x[o] = 0.0;
          return;
        }
        const double xin = xzero ? 0.0 : LDX(x + o);
        if (i == 0 || j == 0 || i == lat - 1 || j == lat - 1) {
          x[o] = xin;
          return;
        }
        const int kx0 = max(0, (i - 1) >> 1), kx1 = min(N, (i + 2) >> 1);
        const int ky0 = max(0, (j - 1) >> 1), ky1 = min(N, (j + 2) >> 1);
        double v[3][3];  // all loads first, then the sum in the k_vanka_update order
#pragma unroll
        for (int a = 0; a < 3; ++a)
#pragma unroll
          for (int c = 0; c < 3; ++c) {
            const int ky = ky0 + a, kx = kx0 + c;
            const int slot = plane * 25 + (j - 2 * ky + 2) * 5 + (i - 2 * kx + 2);
            const bool in = ky <= ky1 && kx <= kx1;
            v[a][c] = LDX(d + (in ? (int64_t)slot * np + (int64_t)ky * (N + 1) + kx : 0));  // unused: skipped
          }
        double s = 0.0;
#pragma unroll
        for (int a = 0; a < 3; ++a)
#pragma unroll
          for (int c = 0; c < 3; ++c)
            if (ky0 + a <= ky1 && kx0 + c <= kx1) s += v[a][c];
        const int mult = (kx1 - kx0 + 1) * (ky1 - ky0 + 1);
        x[o] = xin + (scalar_w ? omega : omega / mult) * s;
      },
      [&](int j, int i, int64_t o) {
        if (i > N) {
          x[o] = 0.0;
          return;
        }
        const double xin = xzero ? 0.0 : LDX(x + o);
        x[o] = xin + omega * LDX(d + 50 * np + (int64_t)j * (N + 1) + i);
      });
}

// r_c = P^T r_f, coarse Dirichlet rows and padding set to 0 (k_restrict)
__device__ __noinline__ void sc_restrict(const LevelGeom& gfr, const LevelGeom& gcr, const double* rf, double* rc,
                                         const ScThreads& T) {
  const LevelGeom gf = gfr, gc = gcr;
  sc_for_points(
      gc, T,
      [&](int plane, int j, int i, int64_t o) {
        if (i < 1 || j < 1 || i >= gc.lat - 1 || j >= gc.lat - 1) {
          rc[o] = 0.0;
          return;
        }
        int fx[5], fy[5];
        double wx[5], wy[5];
        const int nx = p2col(i, fx, wx), ny = p2col(j, fy, wy);
        const double* r = rf + (plane ? gf.ouy : gf.oux);
        double v[5][5];  // all loads first, then the k_restrict order
#pragma unroll
        for (int b = 0; b < 5; ++b)
#pragma unroll
          for (int a = 0; a < 5; ++a)  // unused taps (b >= ny or a >= nx): clamped load, skipped below
            v[b][a] = LDX(r + (int64_t)fy[min(b, ny - 1)] * gf.pu + fx[min(a, nx - 1)]);
        double s = 0.0;
#pragma unroll
        for (int b = 0; b < 5; ++b) {
          if (b >= ny) continue;
          double t = 0.0;
#pragma unroll
          for (int a = 0; a < 5; ++a)
            if (a < nx) t += wx[a] * v[b][a];
          s += wy[b] * t;
        }
        rc[o] = s;
      },
      [&](int j, int i, int64_t o) {
        if (i > gc.N) {
          rc[o] = 0.0;
          return;
        }
        const double* r = rf + gf.op;
        double v[3][3];
#pragma unroll
        for (int b = 0; b < 3; ++b)
#pragma unroll
          for (int a = 0; a < 3; ++a)  // fine nodes outside 0..N: clamped load, skipped below
            v[b][a] = LDX(r + (int64_t)min(max(2 * j + b - 1, 0), gf.N) * gf.pp + min(max(2 * i + a - 1, 0), gf.N));
        double s = 0.0;
#pragma unroll
        for (int b = -1; b <= 1; ++b) {
          const int fj = 2 * j + b;
          if (fj < 0 || fj > gf.N) continue;
          const double wy = b ? 0.5 : 1.0;
#pragma unroll
          for (int a = -1; a <= 1; ++a) {
            const int fi = 2 * i + a;
            if (fi < 0 || fi > gf.N) continue;
            s += wy * (a ? 0.5 : 1.0) * v[b + 1][a + 1];
          }
        }
        rc[o] = s;
      });
}

// x_f += P e_c (prolong_q2_at / prolong_q1_at with L2 loads): one unit per coarse
// element and velocity component (4x4 fine points) or per coarse pressure node (2x2)
__device__ __noinline__ void sc_prolong(const LevelGeom& gf, const LevelGeom& gc, const double* ec, double* xf, const ScThreads& T) {
  const int ne = gc.N * gc.N, nn = (gc.N + 1) * (gc.N + 1);
  for (int q = T.gt; q < 2 * ne + nn; q += T.nt) {
    if (q < 2 * ne) {
      const int comp = q >= ne ? 1 : 0, e = q - comp * ne, ex = e % gc.N, ey = e / gc.N;
      const double* ep = ec + (comp ? gc.ouy : gc.oux) + (int64_t)(2 * ey) * gc.pu + 2 * ex;
      double tx[3][4];
#pragma unroll
      for (int rr = 0; rr < 3; ++rr) {
        const double c0 = LDX(ep + (int64_t)rr * gc.pu), c1 = LDX(ep + (int64_t)rr * gc.pu + 1),
                     c2 = LDX(ep + (int64_t)rr * gc.pu + 2);
        tx[rr][0] = ex == 0 ? 0.0 : c0;  // fine column 0 is Dirichlet
        tx[rr][1] = 0.375 * c0 + 0.75 * c1 - 0.125 * c2;
        tx[rr][2] = c1;
        tx[rr][3] = -0.125 * c0 + 0.75 * c1 + 0.375 * c2;
      }
      double* f = xf + (comp ? gf.ouy : gf.oux) + (int64_t)(4 * ey) * gf.pu + 4 * ex;
#pragma unroll
      for (int m = 0; m < 4; ++m) {
        const int j = 4 * ey + m;
        if (j < 1 || j >= gf.lat - 1) continue;
        const double w0 = m == 0 ? 1.0 : m == 1 ? 0.375 : m == 2 ? 0.0 : -0.125;
        const double w1 = m == 0 ? 0.0 : m == 1 ? 0.75 : m == 2 ? 1.0 : 0.75;
        const double w2 = m == 0 ? 0.0 : m == 1 ? -0.125 : m == 2 ? 0.0 : 0.375;
        double* row = f + (int64_t)m * gf.pu;
#pragma unroll
        for (int c = 0; c < 4; ++c) row[c] = LDX(row + c) + (w0 * tx[0][c] + w1 * tx[1][c] + w2 * tx[2][c]);
      }
    } else {
      const int n = q - 2 * ne, ax = n % (gc.N + 1), ay = n / (gc.N + 1);
      const double* e = ec + gc.op + (int64_t)ay * gc.pp + ax;
      const bool rx = ax < gc.N, ry = ay < gc.N;
      const double c00 = LDX(e), c10 = rx ? LDX(e + 1) : 0.0, c01 = ry ? LDX(e + gc.pp) : 0.0,
                   c11 = rx && ry ? LDX(e + gc.pp + 1) : 0.0;
#pragma unroll
      for (int dy = 0; dy < 2; ++dy) {
        const int j = 2 * ay + dy;
        if (j > gf.N) continue;
        const double l = dy ? 0.5 * (c00 + c01) : c00, rr = dy ? 0.5 * (c10 + c11) : c10;
        double* f = xf + gf.op + (int64_t)j * gf.pp + 2 * ax;
        f[0] = LDX(f) + l;
        if (rx) f[1] = LDX(f + 1) + 0.5 * (l + rr);
      }
    }
  }
}

__global__ void __launch_bounds__(kScThreads, 1) k_small_cycle(const __grid_constant__ ScArgs A) {
  __shared__ ScStencil scs;
  if (threadIdx.x == 0) {
    for (int a = 0; a < 2; ++a)
      for (int k = 0; k < 5; ++k) {
        scs.KR[a][k] = c_st.KR[a][k];
        scs.MR[a][k] = c_st.MR[a][k];
      }
    for (int a = 0; a < 2; ++a)
      for (int k = 0; k < 3; ++k) {
        scs.CC[a][k] = c_st.CC[a][k];
        scs.GC[a][k] = c_st.GC[a][k];
      }
    for (int a = 0; a < 3; ++a)
      for (int k = 0; k < 5; ++k) {
        scs.CR[a][k] = c_st.CR[a][k];
        scs.GR[a][k] = c_st.GR[a][k];
      }
  }
  __syncthreads();
  pdl_wait();
  ScThreads T;
  T.nt = (int)(sc_ncta() * blockDim.x);
  T.gt = (int)(sc_rank() * blockDim.x + threadIdx.x);
  T.nw = T.nt >> 5;
  T.gw = T.gt >> 5;
  T.lane = threadIdx.x & 31;
  int nst = 0;
  auto stamp = [&]() {
    if (A.stamps && T.gt == 0) {
      unsigned long long t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      A.stamps[nst] = t;
    }
    ++nst;
  };
  stamp();
  auto zero = [&](const ScLevel& L) {
    for (int64_t q = T.gt; q < L.g.len; q += T.nt) L.x[q] = 0.0;
  };
  // one relaxation sweep on level l, in place on lv[l].x (alg:vk)
  auto sweep = [&](int l, bool xzero) {
    const ScLevel& L = A.lv[l];
    const double* src = L.b;
    if (!xzero) {
      sc_residual(L, scs, A.nu, L.x, L.r, T);
      src = L.r;
    }
    if (!xzero) {
      sc_sync();  // residual complete
      stamp();
    }
    sc_patches(L, src, A.d, T);
    sc_sync();
    stamp();
    sc_update(L, A.omega, A.scalar_w, xzero, A.d, T);
    sc_sync();
    stamp();
  };
  for (int l = A.top; l >= 1; --l) {  // alg:mg down: relax, residual, restriction
    const ScLevel& L = A.lv[l];
    if (A.nu_pre == 0) {
      zero(L);
      sc_sync();
    stamp();
    }
    for (int k = 0; k < A.nu_pre; ++k) sweep(l, k == 0);
    sc_residual(L, scs, A.nu, L.x, L.r, T);
    sc_sync();
    stamp();
    sc_restrict(L.g, A.lv[l - 1].g, L.r, A.lv[l - 1].b, T);
    sc_sync();
    stamp();
  }
  {  // level 0: A_0^{-1} (minimum-norm, reading 3) or three sweeps from zero
    const ScLevel& L = A.lv[0];
    if (A.sweeps3) {
      sweep(0, true);
      sweep(0, false);
      sweep(0, false);
    } else {
      zero(L);
      sc_sync();
    stamp();
      const int n = A.cni + 1;
      for (int rr = T.gw; rr < A.cni; rr += T.nw) {  // one warp per row (k_coarse_apply)
        double s = 0.0;
        // the level-0 system has 98 + 25 = 123 unknowns: 4 columns per lane, loads first
        double mv[4], bv[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int c = T.lane + 32 * u, cc = min(c, A.cni - 1);
          mv[u] = c < A.cni ? A.cmat[(int64_t)rr * n + cc] : 0.0;
          bv[u] = LDX(L.b + A.cidx[cc]);
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) s = fma(mv[u], bv[u], s);
        for (int c = T.lane + 128; c < A.cni; c += 32) s = fma(A.cmat[(int64_t)rr * n + c], LDX(L.b + A.cidx[c]), s);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        if (T.lane == 0) L.x[A.cidx[rr]] = s;
      }
      sc_sync();
    stamp();
    }
  }
  for (int l = 1; l <= A.top; ++l) {  // alg:mg up: correction, relax
    sc_prolong(A.lv[l].g, A.lv[l - 1].g, A.lv[l - 1].x, A.lv[l].x, T);
    sc_sync();
    stamp();
    for (int k = 0; k < A.nu_post; ++k) sweep(l, false);
  }
}

}  // namespace svk
