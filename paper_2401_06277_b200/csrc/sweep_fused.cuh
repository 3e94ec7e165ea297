// sweep_fused.cuh -- structured patch factors and the fused Vanka sweep kernel.
//
// Generic patch (both axis categories 2, i.e. 2 <= kx,ky <= N-2): the 51
// unknowns are u_x and u_y on the full 5x5 lattice window around node k plus
// p_k, and the patch matrix is (A_i = V_i A V_i^T)
//     A_i = [[Lw, 0, bx^T], [0, Lw, by^T], [bx, by, 0]]
// with Lw = nu (M_w (x) K_w + K_w (x) M_w) (the same for both components,
// h-independent) and bx = -h C^_w (x) G_w, by = -h G_w (x) C^_w.
// It is solved exactly by the Schur complement on the pressure unknown:
//     dp = (cx.rx + cy.ry - rp) / sigma,   c = Lw^{-1} b^T,  sigma = bx.cx + by.cy
//     du = Lw^{-1} rx - cx dp,   dv = Lw^{-1} ry - cy dp
// and Lw^{-1} is applied in the even/odd (reflection) basis of each axis: the
// window matrices are symmetric under o -> 4-o, so with
//     e = (v0+v4, v1+v3, v2),  d = (v0-v4, v1-v3)
// Lw^{-1} is block diagonal with blocks EE 9x9, EO 6x6, OE 6x6, OO 4x4
// (169 FMA instead of 625), and bx lives only in EO, by only in OE.
#pragma once
#include <cuda.h>
#include <algorithm>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "stencil.cuh"

namespace svk {

// transformed per-axis index: 0:e0 1:e1 2:e2 (even) 3:d0 4:d1 (odd)
struct FusedFactors {
  double bee[9][9];   // EE block (ty in {0,1,2}, tx in {0,1,2}); row/col index ty*3+tx
  double beo[6][6];   // EO: ty in {0,1,2}, tx in {3,4}; index ty*2+(tx-3)
  double boe[6][6];   // OE: ty in {3,4}, tx in {0,1,2}; index (ty-3)*3+tx
  double boo[4][4];   // OO: ty in {3,4}, tx in {3,4}; index (ty-3)*2+(tx-3)
  double chx[6];      // hat c_x in EO (dp = (chx . rhat_x(EO) + chy . rhat_y(OE) - rp) * inv_sigma)
  double chy[6];      // hat c_y in OE
  double cpx[6];      // correction of the EO output block of u_x: yhat -= cpx * dp
  double cpy[6];      // correction of the OE output block of u_y
  double inv_sigma;
  double pad;
  // interior stencils of the residual, scaled (nu, h) for this level:
  double L2D[2][2][5][5];  // [row parity][col parity][b+2][a+2]: nu (M_b K_a + K_b M_a)
  double GX[2][2][3][3];   // B_x^T p: -h C^col[py][ty] Gcol[px][tx]
  double GY[2][2][3][3];   // B_y^T p: -h Gcol[py][ty] C^col[px][tx]
  double PBX[5][5];        // B_x at an interior pressure node: -h C^row[oy] G row[ox]
  double PBY[5][5];        // B_y: -h G row[oy] C^row[ox]
};
constexpr int kFacStride = (int)(sizeof(FusedFactors) / sizeof(double));
}  // namespace svk
#include "stencil_gen.cuh"
namespace svk {

// One CTA per level: build Lw, bx, by of the generic window, invert Lw, and
// form the transformed blocks.  Output scaling folds the 1/2 of the inverse
// transform into the rows, so that du = unsplit(yhat) with adds only:
//   v0 = E0 + D0, v4 = E0 - D0, v1 = E1 + D1, v3 = E1 - D1, v2 = E2.
__global__ void k_factor_setup(const int* __restrict__ Ns, double nu, double* __restrict__ out,
                               int* __restrict__ status) {
  const int l = blockIdx.x;
  const int N = Ns[l];
  const double h = 1.0 / N;
  __shared__ double Lw[25 * 25], colk[25], bx[25], by[25], cx[25], cy[25];
  __shared__ double Tm[25 * 25], Lt[25 * 25];
  __shared__ int perm[25];
  __shared__ int flag;
  const int tid = threadIdx.x;
  // generic node (kx,ky) = (2,2) on a level with N >= 4 (windows fully interior)
  const int kx = 2, ky = 2;
  if (tid == 0) flag = 0;
  for (int q = tid; q < 625; q += blockDim.x) {
    const int r = q / 25, c = q % 25;
    Dof a{0, 2 * kx - 2 + r % 5, 2 * ky - 2 + r / 5}, b{0, 2 * kx - 2 + c % 5, 2 * ky - 2 + c / 5};
    Lw[q] = a_entry(a, b, N, nu, h);
  }
  for (int q = tid; q < 25; q += blockDim.x) {
    Dof v0{0, 2 * kx - 2 + q % 5, 2 * ky - 2 + q / 5}, v1{1, 2 * kx - 2 + q % 5, 2 * ky - 2 + q / 5}, p{2, kx, ky};
    bx[q] = a_entry(p, v0, N, nu, h);
    by[q] = a_entry(p, v1, N, nu, h);
  }
  __syncthreads();
  if (!gj_invert(Lw, 25, 25, perm, colk, &flag)) {
    if (tid == 0) atomicExch(status, 1);
    return;
  }
  // c = Lw^{-1} b^T
  for (int q = tid; q < 25; q += blockDim.x) {
    double sx = 0, sy = 0;
    for (int t = 0; t < 25; ++t) {
      sx += Lw[q * 25 + t] * bx[t];
      sy += Lw[q * 25 + t] * by[t];
    }
    cx[q] = sx;
    cy[q] = sy;
  }
  // 1D transform T5 (rows: e0,e1,e2,d0,d1 over v0..v4) and its inverse
  const double T5[5][5] = {{1, 0, 0, 0, 1}, {0, 1, 0, 1, 0}, {0, 0, 1, 0, 0}, {1, 0, 0, 0, -1}, {0, 1, 0, -1, 0}};
  const double Ti5[5][5] = {{.5, 0, 0, .5, 0}, {0, .5, 0, 0, .5}, {0, 0, 1, 0, 0}, {0, .5, 0, 0, -.5}, {.5, 0, 0, -.5, 0}};
  const double S5[5] = {.5, .5, 1, .5, .5};  // output row scaling folded into the blocks
  // Tm = T (x) T with 2D index (ty,tx) <- (vy,vx): Tm[(ty*5+tx)][(vy*5+vx)]
  for (int q = tid; q < 625; q += blockDim.x) {
    const int r = q / 25, c = q % 25;
    Tm[q] = T5[r / 5][c / 5] * T5[r % 5][c % 5];
  }
  __syncthreads();
  // Lt = T Lw^{-1}
  for (int q = tid; q < 625; q += blockDim.x) {
    const int r = q / 25, c = q % 25;
    double s = 0;
    for (int t = 0; t < 25; ++t) s += Tm[r * 25 + t] * Lw[t * 25 + c];
    Lt[q] = s;
  }
  __syncthreads();
  FusedFactors* F = reinterpret_cast<FusedFactors*>(out + (size_t)l * kFacStride);
  // B = S (T Lw^{-1} T^{-1}) restricted to the four parity blocks
  for (int q = tid; q < 625; q += blockDim.x) {
    const int r = q / 25, c = q % 25;
    double s = 0;
    for (int t = 0; t < 25; ++t) s += Lt[r * 25 + t] * (Ti5[t / 5][c / 5] * Ti5[t % 5][c % 5]);
    s *= S5[r / 5] * S5[r % 5];
    const int ry = r / 5, rx = r % 5, cy_ = c / 5, cx_ = c % 5;
    const bool rye = ry < 3, rxe = rx < 3, cye = cy_ < 3, cxe = cx_ < 3;
    if (rye != cye || rxe != cxe) continue;  // zero by symmetry
    if (rye && rxe) F->bee[ry * 3 + rx][cy_ * 3 + cx_] = s;
    else if (rye && !rxe) F->beo[ry * 2 + rx - 3][cy_ * 2 + cx_ - 3] = s;
    else if (!rye && rxe) F->boe[(ry - 3) * 3 + rx][(cy_ - 3) * 3 + cx_] = s;
    else F->boo[(ry - 3) * 2 + rx - 3][(cy_ - 3) * 2 + cx_ - 3] = s;
  }
  // chat = T^{-T} c (dot with rhat = T r reproduces c . r); cpx = S T c
  if (tid < 25) {
    const int ty = tid / 5, tx = tid % 5;
    double hx = 0, hy = 0, px = 0, py = 0;
    for (int v = 0; v < 25; ++v) {
      const double ti = Ti5[v / 5][ty] * Ti5[v % 5][tx];  // (T^{-1})^T[tid][v] = T^{-1}[v][tid]
      hx += ti * cx[v];
      hy += ti * cy[v];
      const double tm = Tm[tid * 25 + v];
      px += tm * cx[v];
      py += tm * cy[v];
    }
    px *= S5[ty] * S5[tx];
    py *= S5[ty] * S5[tx];
    if (ty < 3 && tx >= 3) {
      F->chx[ty * 2 + tx - 3] = hx;
      F->cpx[ty * 2 + tx - 3] = px;
    }
    if (ty >= 3 && tx < 3) {
      F->chy[(ty - 3) * 3 + tx] = hy;
      F->cpy[(ty - 3) * 3 + tx] = py;
    }
  }
  __syncthreads();
  // Enforce the identities the symmetry-shared solve (solve_gen.cuh) relies on,
  // bitwise: B symmetric and invariant under the axis swap s(ty,tx) = (tx,ty)
  // (Lw = nu(M (x) K + K (x) M) is), chy = s(chx), cpy = s(cpx) (b_y = s(b_x)).
  // Each orbit is replaced by its mean (a change at the rounding level).
  if (tid == 0) {
    auto at = [&](int r, int c) -> double* {
      const int ry = r / 5, rx = r % 5, cy_ = c / 5, cx_ = c % 5;
      if (ry < 3 && rx < 3) return &F->bee[ry * 3 + rx][cy_ * 3 + cx_];
      if (ry < 3) return &F->beo[ry * 2 + rx - 3][cy_ * 2 + cx_ - 3];
      if (rx < 3) return &F->boe[(ry - 3) * 3 + rx][(cy_ - 3) * 3 + cx_];
      return &F->boo[(ry - 3) * 2 + rx - 3][(cy_ - 3) * 2 + cx_ - 3];
    };
    auto sg = [](int r) { return (r % 5) * 5 + r / 5; };
    for (int r = 0; r < 25; ++r)
      for (int c = 0; c < 25; ++c) {
        if ((r / 5 < 3) != (c / 5 < 3) || (r % 5 < 3) != (c % 5 < 3)) continue;
        const int mr[4] = {r, c, sg(r), sg(c)}, mc[4] = {c, r, sg(c), sg(r)};
        bool rep = true;
        for (int m = 1; m < 4; ++m) rep = rep && (r * 25 + c <= mr[m] * 25 + mc[m]);
        if (!rep) continue;
        const double avg = ((*at(mr[0], mc[0]) + *at(mr[1], mc[1])) + (*at(mr[2], mc[2]) + *at(mr[3], mc[3]))) * 0.25;
        for (int m = 0; m < 4; ++m) *at(mr[m], mc[m]) = avg;
      }
    for (int a = 0; a < 3; ++a)
      for (int b = 0; b < 2; ++b) {
        const double h2 = 0.5 * (F->chx[a * 2 + b] + F->chy[b * 3 + a]);
        const double p2 = 0.5 * (F->cpx[a * 2 + b] + F->cpy[b * 3 + a]);
        F->chx[a * 2 + b] = F->chy[b * 3 + a] = h2;
        F->cpx[a * 2 + b] = F->cpy[b * 3 + a] = p2;
      }
  }
  for (int q = tid; q < 100; q += blockDim.x) {
    const int py = q / 50, px = (q / 25) % 2, b = (q / 5) % 5, a = q % 5;
    F->L2D[py][px][b][a] = nu * (c_st.MR[py][b] * c_st.KR[px][a] + c_st.KR[py][b] * c_st.MR[px][a]);
  }
  for (int q = tid; q < 36; q += blockDim.x) {
    const int py = q / 18, px = (q / 9) % 2, ty = (q / 3) % 3, tx = q % 3;
    F->GX[py][px][ty][tx] = -h * c_st.CC[py][ty] * c_st.GC[px][tx];
    F->GY[py][px][ty][tx] = -h * c_st.GC[py][ty] * c_st.CC[px][tx];
  }
  for (int q = tid; q < 25; q += blockDim.x) {
    const int oy = q / 5, ox = q % 5;
    F->PBX[oy][ox] = -h * c_st.CR[1][oy] * c_st.GR[1][ox];
    F->PBY[oy][ox] = -h * c_st.GR[1][oy] * c_st.CR[1][ox];
  }
  __syncthreads();
  // Identities the shared-coefficient stencils (stencil_gen.cuh) rely on, made
  // bitwise: L2D depends on (|db|, |da|) only (reflection-symmetric 1D Q2
  // stencils) and L2D[py][px][b][a] = L2D[px][py][a][b]; PBY = PBX^T.
  if (tid == 0) {
    double L0[2][2][5][5];
    for (int q = 0; q < 100; ++q) (&L0[0][0][0][0])[q] = (&F->L2D[0][0][0][0])[q];
    for (int py = 0; py < 2; ++py)
      for (int px = 0; px < 2; ++px)
        for (int bi = 0; bi < 5; ++bi)
          for (int ai = 0; ai < 5; ++ai) {
            const int b = abs(bi - 2), a = abs(ai - 2);
            int kp = py, kq = px, k1 = b, k2 = a;
            if (py == 0 && px == 1) { kp = 1; kq = 0; k1 = a; k2 = b; }
            else if (py == px) { k1 = min(a, b); k2 = max(a, b); }
            F->L2D[py][px][bi][ai] = L0[kp][kq][k1 + 2][k2 + 2];
          }
    for (int oy = 0; oy < 5; ++oy)
      for (int ox = 0; ox < 5; ++ox) F->PBY[oy][ox] = F->PBX[ox][oy];
  }
  if (tid == 0) {
    double s = 0;
    for (int t = 0; t < 25; ++t) s += bx[t] * cx[t] + by[t] * cy[t];
    F->inv_sigma = 1.0 / s;
    F->pad = 0;
    if (s == 0.0) atomicExch(status, 1);
  }
}


// =============================================================================
// Boundary patches (some axis category != 2: kx or ky in {0, 1, N-1, N}).
// They are only O(N) of the (N+1)^2 patches but have 24 different matrices
// without the reflection symmetry, so they are solved up front by this small
// kernel -- one CTA of 256 threads per tile of 16 patches of one group: the
// window residuals on the tile's band, then the dense padded group inverse
// applied on the FP64 tensor path -- and their corrections are stored
// slot-major in `bd`.
// The fused kernel then loads them instead of diverging into a dense solve.
// Boundary patch numbering: rows ky in {0,1,N-1,N} first (4 x (N+1)), then
// columns kx in {0,1,N-1,N} for 2 <= ky <= N-2 (4 x (N-3)); nb = 8N - 8.
// =============================================================================
__host__ __device__ __forceinline__ int bd_axis(int k, int N) { return k <= 1 ? k : k - (N - 3); }
__host__ __device__ __forceinline__ int64_t bd_count(int N) { return 8 * (int64_t)N - 8; }
__host__ __device__ __forceinline__ int64_t bd_index(int kx, int ky, int N) {
  if (ky <= 1 || ky >= N - 1) return (int64_t)bd_axis(ky, N) * (N + 1) + kx;
  return 4 * (int64_t)(N + 1) + (int64_t)bd_axis(kx, N) * (N - 3) + (ky - 2);
}

// Tiles of boundary patches that share one group (category pair): patches
// (kx + q dx, ky + q dy), q < n.  One CTA per tile stages the group's padded
// inverse in shared memory once (instead of once per patch), evaluates the
// tile's window residuals, then applies the inverse (same summation order as a
// per-patch dense product).
struct BdTile {
  int kx, ky, dx, dy, n, grp;
};
#ifndef SVK_BD_TILE
#define SVK_BD_TILE 16
#endif
#ifndef SVK_BD_MINB
#define SVK_BD_MINB 3
#endif
constexpr int kBdTile = SVK_BD_TILE, kBdThreads = 256;
inline std::vector<BdTile> make_bd_tiles(int N) {
  std::vector<BdTile> t;
  auto seg = [&](int kx, int ky, int dx, int dy, int n) {
    for (int q0 = 0; q0 < n; q0 += kBdTile)
      t.push_back(BdTile{kx + q0 * dx, ky + q0 * dy, dx, dy, std::min(kBdTile, n - q0), pcat(ky, N) * 5 + pcat(kx, N)});
  };
  const int rows[4] = {0, 1, N - 1, N};
  for (int ky : rows) {
    seg(0, ky, 1, 0, 1);
    seg(1, ky, 1, 0, 1);
    seg(2, ky, 1, 0, N - 3);
    seg(N - 1, ky, 1, 0, 1);
    seg(N, ky, 1, 0, 1);
  }
  for (int kx : rows) seg(kx, 2, 0, 1, N - 3);
  return t;
}

// The tile's windows cover a band of 5 x (2n+3) lattice points (both components)
// plus its n pressure nodes: the residual is evaluated once per band point
// (phase 1), gathered into per-patch windows (phase 2), then the dense group
// inverse is applied (phase 3).  Dirichlet / outside points carry 0 (they are
// excluded from the patch unknowns, P:469 reading 7).
// x != 0: the band plus its 2-point stencil halo of x (9 x (2n+7) lattice points
// per component, 5 x (n+4) pressure nodes) is first staged in shared memory, so
// that each x value is read from memory once instead of by every stencil that
// touches it (the residual then uses lap_f / gradp_f / div_f on the stage, the
// same arithmetic as lap_at / gradp_at / div_at).  Every global load of the tile
// (group inverse, x stage, b on the band) is issued in one phase.
// Phase 3 is a small dense contraction, D[p][s] = sum_c R[p][c] Ai[s][c] (16
// patches x 51 slots x 51), run on the FP64 tensor path: mma.sync m8n8k4 f64
// (DMMA), patches along M (2 tiles), slots along N (7 tiles, one per warp),
// slots along K (13 steps), fragments read straight from shared memory.
constexpr int kBdBandW = 2 * kBdTile + 3;  // band length along the tile
constexpr int kBdStA = kBdBandW + 4;       // staged length along (stencil halo 2 + 2)
static_assert(kBdTile == 16, "the DMMA apply tiles 16 patches as two m8 tiles");
static_assert(kBdThreads >= 7 * 32, "one warp per n8 tile of the 51 slots");
__device__ __forceinline__ void dmma_m8n8k4(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}
__global__ void __launch_bounds__(kBdThreads, SVK_BD_MINB) k_boundary_patches(LevelGeom g, double nu, const double* __restrict__ dinv,
                                                         const BdTile* __restrict__ tiles,
                                                         const double* __restrict__ x, const double* __restrict__ b,
                                                         double* __restrict__ bd) {
  constexpr int T = kBdTile, RS = 53;  // odd row stride: few bank conflicts on the fragment loads
  constexpr int NBAND = 2 * 5 * kBdBandW;
  constexpr int NXS = 2 * 9 * kBdStA, NPS = 5 * (T + 4);
  __shared__ double Ai[kGroupStride];
  __shared__ double rv[T * RS];
  __shared__ double band[NBAND + T];  // [comp][5 across][kBdBandW along] + pressure residuals (b first)
  __shared__ double xs[NXS + NPS];    // x != 0: [comp][9 across][kBdStA along] + [5 across][T + 4 along]
  pdl_wait();
  const int N = g.N, lat = g.lat;
  const int64_t nb = bd_count(N);
  const BdTile tl = tiles[blockIdx.x];
  const int ylo = tl.ky + (tl.n - 1) * tl.dy;
  if (max(tl.ky, ylo) < g.r0 - 1 || min(tl.ky, ylo) > g.r1) return;  // patch rows a slab uses: r0-1 .. r1
  const double* A = dinv + (size_t)tl.grp * kGroupStride;
  // band origin: lattice point (2 kx - 2, 2 ky - 2) of the tile's first patch; "along" = tile direction
  const int i0 = 2 * tl.kx - 2, j0 = 2 * tl.ky - 2;
  const int nalong = 2 * tl.n + 3;
  // stage: lattice (i, j) <-> [across][along] from (i0 - 2, j0 - 2); nodes from (kx - 2, ky - 2).
  // Rows a slab-local vector does not hold are never read by the band's stencils
  // (the stencils of band rows outside the slab's patch rows are skipped below).
  const int jlo = 2 * (g.r0 - 1) - 4, jhi = 2 * g.r1 + 4;
  // ---- phase 0: every global load of the tile, all in flight at once (registers
  //      first, then shared memory: loop-carried load->store pairs would expose one
  //      L2 round trip per iteration) ----
  // b on the band (0 where the residual is not formed: Dirichlet / outside / beyond the slab)
  auto band_ij = [&](int q, int& comp, int& i, int& j, bool& ok) {
    comp = q / (5 * kBdBandW);
    const int rem = q % (5 * kBdBandW), ac = rem / kBdBandW, al = rem % kBdBandW;
    i = i0 + (tl.dx ? al : ac);
    j = j0 + (tl.dx ? ac : al);
    // only rows of the patches this slab solves (ky in r0-1 .. r1): a column
    // tile may reach beyond them, and a slab-local vector holds no rows there
    const bool jslab = j >= 2 * (g.r0 - 1) - 2 && j <= 2 * g.r1 + 2;
    ok = al < nalong && jslab && i >= 1 && j >= 1 && i <= lat - 2 && j <= lat - 2;
  };
  constexpr int NA = (kGroupStride + kBdThreads - 1) / kBdThreads;
  constexpr int NX = (NXS + NPS + kBdThreads - 1) / kBdThreads;
  constexpr int NB = (NBAND + T + kBdThreads - 1) / kBdThreads;
  double va[NA], vx[NX], vb[NB];
#pragma unroll
  for (int u = 0; u < NA; ++u) {
    const int q = threadIdx.x + u * kBdThreads;
    va[u] = q < kGroupStride ? __ldg(A + q) : 0.0;
  }
#pragma unroll
  for (int u = 0; u < NX; ++u) {
    const int q = threadIdx.x + u * kBdThreads;
    double v = 0.0;
    if (x && q < NXS) {
      const int comp = q / (9 * kBdStA), rem = q % (9 * kBdStA), ac = rem / kBdStA, al = rem % kBdStA;
      const int i = i0 - 2 + (tl.dx ? al : ac), j = j0 - 2 + (tl.dx ? ac : al);
      if (i >= 0 && j >= 0 && i < lat && j < lat && j >= jlo && j <= jhi)
        v = x[(comp ? g.ouy : g.oux) + (int64_t)j * g.pu + i];
    } else if (x && q < NXS + NPS) {
      const int r = q - NXS, ac = r / (T + 4), al = r % (T + 4);
      const int kx = tl.kx - 2 + (tl.dx ? al : ac), ky = tl.ky - 2 + (tl.dx ? ac : al);
      if (kx >= 0 && ky >= 0 && kx <= N && ky <= N && 2 * ky >= jlo && 2 * ky <= jhi) v = x[p_at(g, kx, ky)];
    }
    vx[u] = v;
  }
#pragma unroll
  for (int u = 0; u < NB; ++u) {
    const int q = threadIdx.x + u * kBdThreads;
    double v = 0.0;
    if (q < NBAND) {
      int comp, i, j;
      bool ok;
      band_ij(q, comp, i, j, ok);
      if (ok) v = b[(comp ? g.ouy : g.oux) + (int64_t)j * g.pu + i];
    } else if (q - NBAND < tl.n && tl.ky + (q - NBAND) * tl.dy >= g.r0 - 1 && tl.ky + (q - NBAND) * tl.dy <= g.r1) {
      const int pi = q - NBAND;
      v = b[p_at(g, tl.kx + pi * tl.dx, tl.ky + pi * tl.dy)];
    }
    vb[u] = v;
  }
#pragma unroll
  for (int u = 0; u < NA; ++u) {
    const int q = threadIdx.x + u * kBdThreads;
    if (q < kGroupStride) Ai[q] = va[u];
  }
#pragma unroll
  for (int u = 0; u < NX; ++u) {
    const int q = threadIdx.x + u * kBdThreads;
    if (x && q < NXS + NPS) xs[q] = vx[u];
  }
#pragma unroll
  for (int u = 0; u < NB; ++u) {
    const int q = threadIdx.x + u * kBdThreads;
    if (q < NBAND + T) band[q] = vb[u];
  }
  // ---- phase 1: r = b - A x on the band ----
  if (x) {
    __syncthreads();
    auto XS = [&](int comp, int i, int j) -> double {
      const int ai = i - (i0 - 2), aj = j - (j0 - 2);
      return xs[comp * 9 * kBdStA + (tl.dx ? aj * kBdStA + ai : ai * kBdStA + aj)];
    };
    auto PS = [&](int kx, int ky) -> double {
      const int ax = kx - (tl.kx - 2), ay = ky - (tl.ky - 2);
      return xs[NXS + (tl.dx ? ay * (T + 4) + ax : ax * (T + 4) + ay)];
    };
    // stage strides: lattice (i, j) -> xs[comp * 9 kBdStA + (i - i0 + 2) si + (j - j0 + 2) sj]
    const int si = tl.dx ? 1 : kBdStA, sj = tl.dx ? kBdStA : 1;
    const int pxs = tl.dx ? 1 : T + 4, pys = tl.dx ? T + 4 : 1;  // pressure stage strides
    for (int q = threadIdx.x; q < NBAND + T; q += blockDim.x) {
      if (q < NBAND) {
        int comp, i, j;
        bool ok;
        band_ij(q, comp, i, j, ok);
        if (ok) {
          // (L u + B^T p)(i, j) with the whole 5x5 / 3x3 stage windows read first: the
          // products and summation order of lap_f / gradp_f; the taps lap_f skips (odd
          // parity, offsets +-2) carry the exact zeros KR[1][0,4] = MR[1][0,4] = 0
          const int pi = i & 1, pj = j & 1;
          const double* xc = xs + comp * 9 * kBdStA + (i - i0 + 2) * si + (j - j0 + 2) * sj;
          double U[5][5];
#pragma unroll
          for (int bb = 0; bb < 5; ++bb)
#pragma unroll
            for (int aa = 0; aa < 5; ++aa) U[bb][aa] = xc[(aa - 2) * si + (bb - 2) * sj];
          const int ky0 = pj ? (j - 1) >> 1 : (j >> 1) - 1, nky = pj ? 2 : 3;
          const int kx0 = pi ? (i - 1) >> 1 : (i >> 1) - 1, nkx = pi ? 2 : 3;
          const double* pc = xs + NXS + (kx0 - (tl.kx - 2)) * pxs + (ky0 - (tl.ky - 2)) * pys;
          double P[3][3];
#pragma unroll
          for (int ty = 0; ty < 3; ++ty)
#pragma unroll
            for (int tx = 0; tx < 3; ++tx) P[ty][tx] = pc[min(tx, nkx - 1) * pxs + min(ty, nky - 1) * pys];
          double sl = 0.0;
#pragma unroll
          for (int bb = 0; bb < 5; ++bb) {
            const double my = c_st.MR[pj][bb], ky = c_st.KR[pj][bb];
#pragma unroll
            for (int aa = 0; aa < 5; ++aa) sl += (my * c_st.KR[pi][aa] + ky * c_st.MR[pi][aa]) * U[bb][aa];
          }
          double sp = 0.0;
#pragma unroll
          for (int ty = 0; ty < 3; ++ty) {
            if (ty >= nky) continue;
            const double cy = comp == 0 ? c_st.CC[pj][ty] : c_st.GC[pj][ty];
            if (cy == 0.0) continue;
            double t = 0.0;
#pragma unroll
            for (int tx = 0; tx < 3; ++tx)
              if (tx < nkx) t += (comp == 0 ? c_st.GC[pi][tx] : c_st.CC[pi][tx]) * P[ty][tx];
            sp += cy * t;
          }
          band[q] -= nu * sl + -g.h * sp;
        }
      } else if (q - NBAND < tl.n && tl.ky + (q - NBAND) * tl.dy >= g.r0 - 1 && tl.ky + (q - NBAND) * tl.dy <= g.r1) {
        const int pi = q - NBAND;
        band[q] -= div_f(XS, N, tl.kx + pi * tl.dx, tl.ky + pi * tl.dy, g.h);
      }
    }
  }
  __syncthreads();
  // ---- phase 2: per-patch windows R[p][slot] ----
  for (int q = threadIdx.x; q < T * kSlots; q += blockDim.x) {
    const int pi = q % T, s = q / T;
    double r = 0.0;
    if (pi < tl.n) {
      if (s < 50) {  // window (oy, ox) of patch pi: band across = oy (row tile) / ox, along = 2 pi + ox / oy
        const int comp = s / 25, oy = (s % 25) / 5, ox = s % 5;
        const int ac = tl.dx ? oy : ox, al = 2 * pi + (tl.dx ? ox : oy);
        r = band[comp * 5 * kBdBandW + ac * kBdBandW + al];
      } else {
        r = band[NBAND + pi];
      }
    }
    rv[pi * RS + s] = r;
  }
  __syncthreads();
  // ---- phase 3: D = R Ai^T on DMMA; warp w computes slots 8w .. 8w+7 of all 16 patches ----
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp >= 7) return;
  const int gq = lane >> 2, t4 = lane & 3;
  const int sb = 8 * warp + gq;  // B fragment: B[k][n] = Ai[n][k], n = slot 8w + (lane >> 2)
  double d[2][2] = {{0.0, 0.0}, {0.0, 0.0}};
#pragma unroll
  for (int kt = 0; kt < 13; ++kt) {
    const int c = 4 * kt + t4;  // K index (slot of the residual window)
    const double bfr = (sb < kSlots && c < kSlots) ? Ai[sb * kSlots + c] : 0.0;
    const double a0 = c < kSlots ? rv[gq * RS + c] : 0.0;        // A[m][k] = R[patch gq][c]
    const double a1 = c < kSlots ? rv[(8 + gq) * RS + c] : 0.0;  // patches 8 + gq
    dmma_m8n8k4(d[0][0], d[0][1], a0, bfr);
    dmma_m8n8k4(d[1][0], d[1][1], a1, bfr);
  }
#pragma unroll
  for (int mt = 0; mt < 2; ++mt)
#pragma unroll
    for (int jj = 0; jj < 2; ++jj) {
      const int pi = 8 * mt + gq, s = 8 * warp + 2 * t4 + jj;  // C[m][n]: m = patch, n = slot
      if (pi >= tl.n || s >= kSlots) continue;
      const int kx = tl.kx + pi * tl.dx, ky = tl.ky + pi * tl.dy;
      if (ky < g.r0 - 1 || ky > g.r1) continue;
      bd[(int64_t)s * nb + bd_index(kx, ky, N)] = d[mt][jj];
    }
}

// =============================================================================
// Fused additive Vanka sweep (alg:vk) -- one kernel per sweep:
//   x_out = x_in + W sum_i V_i^T A_i^{-1} V_i (b - A x_in)
//
// Layout of the work ("owner computes", no atomics, deterministic):
//  * a CTA of kNT threads (default 64 = 2 warps) owns a STRIP of kNOUT = 30 kWarps
//    node columns starting at kx0 and a CHUNK of node rows [y0, y1); it streams
//    upward through the chunk one node row (= one patch row = two lattice rows)
//    per step, keeping rings of rows in shared memory, filled by TMA one step
//    ahead (out-of-range rows / columns zero-filled) and completed on two
//    mbarriers: x (6 row pairs, both components), p (8 node rows), b (2 pairs),
//    b_p (2 rows), residual (7 lattice rows), pressure residual (4 rows).
//  * step s: (1) thread 0 issues the TMA loads of step s+1; (2) residual
//    r = b - A x on lattice rows 2s+1, 2s+2 (thread t: lattice columns rc0+2t,
//    rc0+2t+1, both components) and the pressure residual of node row s+1, into
//    the residual rings; (3) one CTA barrier; (4) lane l of warp w solves patch
//    pi = 30w + l, node column kx0-1+pi, exactly: generic patches by the
//    symmetry-shared reflection-basis Schur solve (solve_gen.cuh), boundary
//    patches from k_boundary_patches' output; (5) owner-computes accumulation in
//    registers (carries over three lattice rows, neighbouring patch columns via
//    warp shuffles; lanes 0 and 31 are ghost patches, so warps never exchange
//    partial sums) and x_out = x_in + W sum on lattice rows 2s-2, 2s-1, which are
//    now complete.
//  * patches and residuals at a strip edge are recomputed by both neighbouring
//    strips (2 patch columns per 30 kWarps node columns).
// =============================================================================
namespace fz {
// strip geometry: kWarps warps x 32 patch columns; warp w covers patches 30w .. 30w+31
// of the strip and owns the middle 30 (lanes 0 and 31 are ghosts), so warps
// accumulate independently.  Strip = 30 kWarps + 2 distinct patches, 30 kWarps owned
// node columns.  Default 2 warps (SVK_STRIP_THREADS=64): 4 CTAs/SM, barriers over
// 2 warps only (measured 3.5% faster than 4-warp strips at 2 CTAs/SM).
#ifndef SVK_STRIP_THREADS
#define SVK_STRIP_THREADS 64
#endif
constexpr int kNT = SVK_STRIP_THREADS, kWarps = kNT / 32, kOWN = 30, kNOUT = kWarps * kOWN;
constexpr int kMinB = 256 / kNT;  // CTAs per SM the rings and registers are sized for
constexpr int W = 2 * kNT;        // ring row width (doubles): x columns xc0..xc0+W-1, r/b columns rc0..rc0+W-1
constexpr int PWID = kNT;         // b_p / r_p row width: node columns from kx0-2
constexpr int PXW = kNT + 8;      // p ring box width: node columns pc0 = kx0-4 .. kx0+kNT+3
constexpr int PXS = (PXW + 15) / 16 * 16;  // p ring row stride (TMA smem destinations are 128-byte aligned)
// (TMA box starts must be 16-byte aligned in the innermost dimension: every
//  box origin here is an even column.)  Ring depths let warps drift up to one
//  step apart with a single barrier per step (see the WAR notes in the kernel).
// x ring: row PAIRS (2p+1, 2p+2), each [comp][2 rows][WX].  The residual of the
// last ghost patch column reads x up to two lattice columns beyond 2 kNT, which
// 128-thread strips cover with idle threads; narrower strips get 4 extra columns
// (TMA boxes stop at 256, hence none for 128; 4 keeps pairs 128-byte aligned).
constexpr int WX = kNT >= 128 ? W : W + 4;
constexpr int XPR = 6;
constexpr int PR = 8;             // p ring rows
constexpr int BPR = 2;            // b ring row pairs
constexpr int RR = 7;             // residual ring rows, each [comp][W]
constexpr int RPR = 4;            // pressure-residual ring rows
constexpr int OXS = 0;
constexpr int OPS = OXS + XPR * 4 * WX;
constexpr int OBS = OPS + PR * PXS;
constexpr int OBP = OBS + BPR * 4 * W;
constexpr int ORS = OBP + 2 * PWID;
constexpr int ORP = ORS + RR * 2 * W;
constexpr int OMB = ORP + RPR * PWID;  // 2 mbarriers
constexpr int kSmemBytes = (OMB + 2) * 8;
constexpr unsigned kXBytes = 4 * WX * 8, kPBytes = PXW * 8, kBBytes = 4 * W * 8, kBPBytes = PWID * 8;
static_assert(kMinB * (kSmemBytes + 1024) <= 232448, "kMinB sweep CTAs per SM");
}  // namespace fz

struct FusedArgs {
  LevelGeom g;
  double omega;
  int scalar_w;
  int chunk;            // node rows per CTA
  const double* bd;     // boundary-patch corrections (k_boundary_patches), slot-major
  double* xout;
};
struct FusedMaps {      // TMA descriptors (host-encoded per launch)
  CUtensorMap xv;       // x velocity planes: dims {lat, lat, 2}, box {256, 2, 2}
  CUtensorMap xp;       // x pressure plane:  dims {N+1, N+1},  box {128, 1}
  CUtensorMap bv;       // b velocity planes
  CUtensorMap bp;       // b pressure plane
};

__device__ __forceinline__ int pmod(int a, int m) {
  const int r = a % m;
  return r < 0 ? r + m : r;
}
__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, int c0, int c1, int c2, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];\n" ::"r"(
          smem_u32(dst)),
      "l"(map), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int c0, int c1, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];\n" ::"r"(
          smem_u32(dst)),
      "l"(map), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
}

// ring offsets (doubles from the smem base)
__device__ __forceinline__ int xpair(int p) { return fz::OXS + pmod(p, fz::XPR) * 4 * fz::WX; }
// x lattice row j, component c: pair (j-1)>>1, row-in-pair (j-1)&1, layout [comp][row][W]
__device__ __forceinline__ int xrow(int j, int c) {
  return xpair((j - 1) >> 1) + c * 2 * fz::WX + ((j - 1) & 1) * fz::WX;
}
__device__ __forceinline__ int prow(int r) { return fz::OPS + (r & 7) * fz::PXS; }
__device__ __forceinline__ int bpair(int p) { return fz::OBS + (p & 1) * 4 * fz::W; }
__device__ __forceinline__ int brow(int j, int c) { return bpair((j - 1) >> 1) + c * 2 * fz::W + ((j - 1) & 1) * fz::W; }
__device__ __forceinline__ int bprow(int r) { return fz::OBP + (r & 1) * fz::PWID; }
__device__ __forceinline__ int rrow(int j, int c) { return fz::ORS + pmod(j, fz::RR) * 2 * fz::W + c * fz::W; }
__device__ __forceinline__ int rprow(int r) { return fz::ORP + (r & 3) * fz::PWID; }

__device__ __forceinline__ double2 lds2(const double* p) { return *reinterpret_cast<const double2*>(p); }
__device__ __forceinline__ void sts2(double* p, double a, double b) { *reinterpret_cast<double2*>(p) = make_double2(a, b); }

// Residual on lattice rows 2sp+1 (odd) and 2sp+2 (even) at lattice columns
// c0 = rc0 + 2t (even) and c0+1, both components, and the pressure residual at
// node (kx0-2+t, sp+1).  Reads x rows 2sp..2sp+4, p rows sp..sp+2, b rows
// 2sp+1, 2sp+2 (pair sp), b_p row sp+1.  Each stencil coefficient is loaded once
// and used for both components; the whole 5x5 windows are loaded first.
struct ResVals {
  double u[2][4];  // [comp][(j0,c0), (j0,c0+1), (j1,c0), (j1,c0+1)], 0 on Dirichlet / outside points
  double p;        // pressure residual at node (kx0-2+t, sp+1), 0 outside
};
// ring layout of the sweep kernel (x 6 pairs, p 8 rows, b 2 pairs, b_p 2 rows)
// b values of residual column set t (lattice columns rc0 + 2t, +1 / node kx0-2+t)
// from the ring's b rows; a ring may instead read them from global memory
#define SVK_RING_B_FROM_SMEM                                                                       \
  __device__ __forceinline__ double2 b2(const double* sm, int j, int c, int t) const {            \
    return lds2(sm + b(j, c) + 2 * t);                                                           \
  }                                                                                              \
  __device__ __forceinline__ double bp1(const double* sm, int r, int t) const { return sm[bp(r) + t]; }
struct RingFz {
  static __device__ __forceinline__ int x(int j, int c) { return xrow(j, c); }
  static __device__ __forceinline__ int p(int r) { return prow(r); }
  static __device__ __forceinline__ int b(int j, int c) { return brow(j, c); }
  static __device__ __forceinline__ int bp(int r) { return bprow(r); }
  SVK_RING_B_FROM_SMEM
};
// MASK = false (the fused sweep): Dirichlet / boundary-pressure rows are not
// masked -- generic patches, the only readers of these residuals, have windows
// strictly inside the domain (2 <= kx, ky <= N-2), so those values are never used.
// The stencil windows of one residual step: x rows 2sp..2sp+4 (lattice columns
// c0-2 .. c0+2, both components) and p rows sp..sp+2 (nodes kx0-3+t .. kx0-1+t).
struct ResWin {
  double U[5][5], V[5][5], Pm[3][3];
};
// load x window rows R0..R1 and p window rows P0..P1 of step sp
template <int R0, int R1, int P0, int P1, class RG>
__device__ __forceinline__ void load_res_win(const double* sm, const RG& rg, int sp, ResWin& w, int t) {
#pragma unroll
  for (int r = R0; r <= R1; ++r) {
    const double* xu = sm + rg.x(2 * sp + r, 0) + 2 * t;
    const double* xv = sm + rg.x(2 * sp + r, 1) + 2 * t;
    const double2 u01 = lds2(xu), u23 = lds2(xu + 2), v01 = lds2(xv), v23 = lds2(xv + 2);
    w.U[r][0] = u01.x; w.U[r][1] = u01.y; w.U[r][2] = u23.x; w.U[r][3] = u23.y; w.U[r][4] = xu[4];
    w.V[r][0] = v01.x; w.V[r][1] = v01.y; w.V[r][2] = v23.x; w.V[r][3] = v23.y; w.V[r][4] = xv[4];
  }
#pragma unroll
  for (int r = P0; r <= P1; ++r) {
    const double* pr = sm + rg.p(sp + r) + t + 1;
#pragma unroll
    for (int q = 0; q < 3; ++q) w.Pm[r][q] = pr[q];
  }
}
template <int R0, int R1, int P0, int P1, class RG>
__device__ __forceinline__ void load_res_win(const double* sm, const RG& rg, int sp, ResWin& w) {
  load_res_win<R0, R1, P0, P1, RG>(sm, rg, sp, w, (int)threadIdx.x);
}
// step sp -> sp+1 with the overlapping rows kept in registers (x rows 2..4 -> 0..2, p rows 1..2 -> 0..1)
__device__ __forceinline__ void roll_res_win(ResWin& w) {
#pragma unroll
  for (int r = 0; r < 3; ++r)
#pragma unroll
    for (int c = 0; c < 5; ++c) {
      w.U[r][c] = w.U[r + 2][c];
      w.V[r][c] = w.V[r + 2][c];
    }
#pragma unroll
  for (int r = 0; r < 2; ++r)
#pragma unroll
    for (int q = 0; q < 3; ++q) w.Pm[r][q] = w.Pm[r + 1][q];
}
template <bool XZERO, bool NOB = false, class RG = RingFz, bool MASK = true>
__device__ __forceinline__ ResVals residual_from_win(const double* sm, const LevelGeom& g, const FusedFactors& F,
                                                     int sp, int kx0, const RG& rg, const ResWin& w,
                                                     int t = -1) {
  if (t < 0) t = threadIdx.x;
  const int N = g.N, lat = g.lat;
  const int c0 = 2 * kx0 - 4 + 2 * t;
  const int j0 = 2 * sp + 1, j1 = 2 * sp + 2;
  const bool c0ok = c0 >= 1 && c0 <= lat - 2, c1ok = c0 + 1 >= 1 && c0 + 1 <= lat - 2;
  const bool j0ok = j0 >= 1 && j0 <= lat - 2, j1ok = j1 >= 1 && j1 <= lat - 2;
  const int na = kx0 - 2 + t, nrow = sp + 1;
  const bool pok = na >= 0 && na <= N && nrow >= 0 && nrow <= N;
  double ax[8];  // (A x) at (j0,c0) (j0,c0+1) (j1,c0) (j1,c0+1) for u_x [0..3] and u_y [4..7]
#pragma unroll
  for (int q = 0; q < 8; ++q) ax[q] = 0.0;
  double bu = 0.0;
  if (!XZERO) {
    const double (&U)[5][5] = w.U;
    const double (&V)[5][5] = w.V;
    const double (&Pm)[3][3] = w.Pm;
    stencil_L_sym(U, V, ax, F);  // shared-coefficient form (stencil_gen.cuh)
    const bool pint = na >= 1 && na <= N - 1 && nrow >= 1 && nrow <= N - 1;
    if (pint || !MASK) {  // B u on the interior pressure-row pattern (window = U/V)
      bu = stencil_B_sym(U, V, F);
    } else if (MASK && pok) {  // boundary pressure node: its B rows from the class table (B = -h PB)
      const int cls = (nrow == 0 ? 0 : (nrow == N ? 2 : 1)) * 3 + (na == 0 ? 0 : (na == N ? 2 : 1));
      const double* pbx = c_st.PB[0][cls];
      const double* pby = c_st.PB[1][cls];
      double sacc = 0.0;
#pragma unroll
      for (int r = 0; r < 5; ++r)
#pragma unroll
        for (int ox = 0; ox < 5; ++ox) sacc = fma(pby[r * 5 + ox], V[r][ox], fma(pbx[r * 5 + ox], U[r][ox], sacc));
      bu = -g.h * sacc;
    }
    ax[0] += F.GX[1][0][0][0] * Pm[0][0] + F.GX[1][0][0][2] * Pm[0][2] + F.GX[1][0][1][0] * Pm[1][0] +
             F.GX[1][0][1][2] * Pm[1][2];
    ax[1] += F.GX[1][1][0][0] * Pm[0][1] + F.GX[1][1][0][1] * Pm[0][2] + F.GX[1][1][1][0] * Pm[1][1] +
             F.GX[1][1][1][1] * Pm[1][2];
    ax[2] += F.GX[0][0][1][0] * Pm[1][0] + F.GX[0][0][1][2] * Pm[1][2];
    ax[3] += F.GX[0][1][1][0] * Pm[1][1] + F.GX[0][1][1][1] * Pm[1][2];
    ax[4] += F.GY[1][0][0][1] * Pm[0][1] + F.GY[1][0][1][1] * Pm[1][1];
    ax[5] += F.GY[1][1][0][0] * Pm[0][1] + F.GY[1][1][0][1] * Pm[0][2] + F.GY[1][1][1][0] * Pm[1][1] +
             F.GY[1][1][1][1] * Pm[1][2];
    ax[6] += F.GY[0][0][0][1] * Pm[0][1] + F.GY[0][0][2][1] * Pm[2][1];
    ax[7] += F.GY[0][1][0][0] * Pm[0][1] + F.GY[0][1][0][1] * Pm[0][2] + F.GY[0][1][2][0] * Pm[2][1] +
             F.GY[0][1][2][1] * Pm[2][2];
  }
  // r = b - A x on non-Dirichlet points (b columns rc0.. = 2t, 2t+1 of the b ring); NOB: b = 0
  ResVals R;
#pragma unroll
  for (int comp = 0; comp < 2; ++comp) {
    const double2 b0 = NOB ? make_double2(0.0, 0.0) : rg.b2(sm, j0, comp, t);
    const double2 b1 = NOB ? make_double2(0.0, 0.0) : rg.b2(sm, j1, comp, t);
    R.u[comp][0] = (!MASK || (j0ok && c0ok)) ? b0.x - ax[4 * comp + 0] : 0.0;
    R.u[comp][1] = (!MASK || (j0ok && c1ok)) ? b0.y - ax[4 * comp + 1] : 0.0;
    R.u[comp][2] = (!MASK || (j1ok && c0ok)) ? b1.x - ax[4 * comp + 2] : 0.0;
    R.u[comp][3] = (!MASK || (j1ok && c1ok)) ? b1.y - ax[4 * comp + 3] : 0.0;
  }
  R.p = (!MASK || pok) ? (NOB ? 0.0 : rg.bp1(sm, nrow, t)) - bu : 0.0;
  return R;
}

template <bool XZERO, bool NOB = false, class RG = RingFz, bool MASK = true>
__device__ __forceinline__ ResVals fused_residual_vals(const double* sm, const LevelGeom& g, const FusedFactors& F,
                                                       int sp, int kx0, const RG& rg = RG{}) {
  ResWin w;
  if (!XZERO) load_res_win<0, 4, 0, 2>(sm, rg, sp, w);
  return residual_from_win<XZERO, NOB, RG, MASK>(sm, g, F, sp, kx0, rg, w);
}
// the same, stored into the residual rings (rows j0, j1 and pressure row sp+1)
// Ring slots of one sweep step sp, maintained incrementally by the kernel (no
// division by the non-power-of-two ring depths inside the step): xq = slot of x
// pair sp-1, rq = residual-ring slot of lattice row 2sp-2.
template <int NXP, int OX>  // x ring: NXP pairs of width fz::WX at offset OX
struct RingSlots {
  int xq, rq;
  __device__ __forceinline__ static RingSlots at(int sp) { return RingSlots{pmod(sp - 1, NXP), pmod(2 * sp - 2, fz::RR)}; }
  __device__ __forceinline__ void advance() {
    xq = xq == NXP - 1 ? 0 : xq + 1;
    rq = rq + 2 >= fz::RR ? rq + 2 - fz::RR : rq + 2;
  }
  // x pair sp-1+d (d in -1..2)
  __device__ __forceinline__ int xpair_d(int d) const {
    int q = xq + d;
    q = q >= NXP ? q - NXP : (q < 0 ? q + NXP : q);
    return OX + q * 4 * fz::WX;
  }
  // lattice row j = 2sp+r (r in -3..4): pair sp + ((r-1)>>1) = sp-1 + d
  __device__ __forceinline__ int xr(int r, int c) const { return xpair_d(((r - 1) >> 1) + 1) + c * 2 * fz::WX + ((r - 1) & 1) * fz::WX; }
  // residual ring row 2sp-2+o (o in 0..6)
  __device__ __forceinline__ int rr(int o, int c) const {
    int q = rq + o;
    q = q >= fz::RR ? q - fz::RR : q;
    return fz::ORS + q * 2 * fz::W + c * fz::W;
  }
};
using RingFzS = RingSlots<fz::XPR, fz::OXS>;
// adapter for fused_residual_vals: rows addressed through the step's slots
struct RingFzStep {
  RingFzS S;
  int sp;
  __device__ __forceinline__ int x(int j, int c) const { return S.xr(j - 2 * sp, c); }
  __device__ __forceinline__ int p(int r) const { return prow(r); }
  __device__ __forceinline__ int b(int j, int c) const { return brow(j, c); }
  __device__ __forceinline__ int bp(int r) const { return bprow(r); }
  SVK_RING_B_FROM_SMEM
};
template <bool XZERO, bool NOB = false, int RRN = fz::RR, int ORSB = fz::ORS, int ORPB = fz::ORP>
__device__ __forceinline__ void fused_residual(double* sm, const LevelGeom& g, const FusedFactors& F, int sp,
                                               int kx0) {
  const RingFzStep rg{RingFzS::at(sp), sp};
  const ResVals R = fused_residual_vals<XZERO, NOB, RingFzStep, false>(sm, g, F, sp, kx0, rg);
  const int t = threadIdx.x;
#pragma unroll
  for (int comp = 0; comp < 2; ++comp) {
    sts2(sm + rg.S.rr(3, comp) + 2 * t, R.u[comp][0], R.u[comp][1]);
    sts2(sm + rg.S.rr(4, comp) + 2 * t, R.u[comp][2], R.u[comp][3]);
  }
  sm[ORPB + ((sp + 1) & 3) * fz::PWID + t] = R.p;
}
// the same with the step's slots supplied by the caller
__device__ __forceinline__ void fused_residual_step(double* sm, const LevelGeom& g, const FusedFactors& F, int sp,
                                                    int kx0, const RingFzS& S, double (&pm)[3][3], bool first) {
  const RingFzStep rg{S, sp};
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
  const ResVals R = residual_from_win<false, false, RingFzStep, false>(sm, g, F, sp, kx0, rg, win);
  const int t = threadIdx.x;
#pragma unroll
  for (int comp = 0; comp < 2; ++comp) {
    sts2(sm + S.rr(3, comp) + 2 * t, R.u[comp][0], R.u[comp][1]);
    sts2(sm + S.rr(4, comp) + 2 * t, R.u[comp][2], R.u[comp][3]);
  }
  sm[fz::ORP + ((sp + 1) & 3) * fz::PWID + t] = R.p;
}

// forward even/odd transform of one 5-vector with stride st (in place)
#define SVK_SPLIT5(v, o, st)                                          \
  {                                                                   \
    const double a_ = v[o], b_ = v[o + st], c_ = v[o + 2 * st], d_ = v[o + 3 * st], e_ = v[o + 4 * st]; \
    v[o] = a_ + e_;                                                   \
    v[o + st] = b_ + d_;                                              \
    v[o + 2 * st] = c_;                                               \
    v[o + 3 * st] = a_ - e_;                                          \
    v[o + 4 * st] = b_ - d_;                                          \
  }
// inverse (row scaling already folded into the blocks): v0=E0+D0 v1=E1+D1 v2=E2 v3=E1-D1 v4=E0-D0
#define SVK_UNSPLIT5(v, o, st)                                        \
  {                                                                   \
    const double e0_ = v[o], e1_ = v[o + st], e2_ = v[o + 2 * st], d0_ = v[o + 3 * st], d1_ = v[o + 4 * st]; \
    v[o] = e0_ + d0_;                                                 \
    v[o + st] = e1_ + d1_;                                            \
    v[o + 2 * st] = e2_;                                              \
    v[o + 3 * st] = e1_ - d1_;                                        \
    v[o + 4 * st] = e0_ - d0_;                                        \
  }

__device__ __forceinline__ void fwd_transform(double (&v)[25]) {
#pragma unroll
  for (int r = 0; r < 5; ++r) SVK_SPLIT5(v, r * 5, 1);
#pragma unroll
  for (int c = 0; c < 5; ++c) SVK_SPLIT5(v, c, 5);
}
__device__ __forceinline__ void inv_transform(double (&v)[25]) {
#pragma unroll
  for (int c = 0; c < 5; ++c) SVK_UNSPLIT5(v, c, 5);
#pragma unroll
  for (int r = 0; r < 5; ++r) SVK_UNSPLIT5(v, r * 5, 1);
}
}  // namespace svk
#include "solve_gen.cuh"
namespace svk {

template <bool XZERO>
__global__ void __launch_bounds__(fz::kNT, fz::kMinB) k_vanka_fused(const FusedArgs A, const FusedFactors F,
                                                            const __grid_constant__ FusedMaps M) {
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
  uint64_t* bars = reinterpret_cast<uint64_t*>(sm + fz::OMB);
  unsigned phases = 0u;  // bit b: parity of mbarrier b (a register, not a local array)

  if (t == 0) {
    mbar_init(&bars[0], 1);
    mbar_init(&bars[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  pdl_wait();
  // prologue: x pairs sB-3 .. sB+1 (rows 2sB-5 .. 2sB+4), p rows sB-2 .. sB+1,
  // b pairs sB-2, sB-1 (rows 2sB-3 .. 2sB), b_p rows sB-1, sB  -> barrier 0
  if (t == 0) {
    unsigned bytes = 2 * fz::kBBytes + 2 * fz::kBPBytes + (XZERO ? 0u : 5 * fz::kXBytes + 4 * fz::kPBytes);
    mbar_expect_tx(&bars[0], bytes);
    if (!XZERO) {
      for (int p = sB - 3; p <= sB + 1; ++p) tma_load_3d(sm + xpair(p), &M.xv, xc0, 2 * p + 1, 0, &bars[0]);
      for (int r = sB - 2; r <= sB + 1; ++r) tma_load_2d(sm + prow(r), &M.xp, pc0, r, &bars[0]);
    }
    for (int p = sB - 2; p <= sB - 1; ++p) tma_load_3d(sm + bpair(p), &M.bv, xc0 + 2, 2 * p + 1, 0, &bars[0]);
    for (int r = sB - 1; r <= sB; ++r) tma_load_2d(sm + bprow(r), &M.bp, kx0 - 2, r, &bars[0]);
  }
  mbar_wait(&bars[0], 0u);
  phases ^= 1u;
  fused_residual<XZERO>(sm, A.g, F, sB - 2, kx0);
  fused_residual<XZERO>(sm, A.g, F, sB - 1, kx0);
  __syncthreads();
  // data of step sB: p row sB+2, b pair sB, b_p row sB+1 -> barrier 1
  if (t == 0) {
    unsigned bytes = fz::kBBytes + fz::kBPBytes + (XZERO ? 0u : fz::kPBytes);
    mbar_expect_tx(&bars[1], bytes);
    if (!XZERO) tma_load_2d(sm + prow(sB + 2), &M.xp, pc0, sB + 2, &bars[1]);
    tma_load_3d(sm + bpair(sB), &M.bv, xc0 + 2, 2 * sB + 1, 0, &bars[1]);
    tma_load_2d(sm + bprow(sB + 1), &M.bp, kx0 - 2, sB + 1, &bars[1]);
  }

  // lane l of warp w solves strip patch pi = 30w + l (node column kxp) and, for
  // lanes 1..30, owns lattice columns 2kxp, 2kxp+1 (ring columns 2pi+2, 2pi+3)
  const int pi = fz::kOWN * warp + lane;
  const int kxp = kx0 - 1 + pi;
  const bool owner = lane >= 1 && lane <= fz::kOWN;
  // Owner-computes accumulation in registers: carry[r][comp][col] holds the
  // partial sums of this lane's two lattice columns on rows 2s-2+r (r = 0,1,2)
  // entering step s; neighbour patch columns contribute through warp shuffles.
  // Summation order is fixed (deterministic).
  double carry[3][2][2];
#pragma unroll
  for (int r = 0; r < 3; ++r)
#pragma unroll
    for (int c = 0; c < 2; ++c) carry[r][c][0] = carry[r][c][1] = 0.0;
  // per-thread output constants: column flags and multiplicity weights
  // W_i = omega / (patches holding the point): 3 per axis at even, 2 at odd lattice indices
  const int i0 = 2 * kxp;
  const bool cin0 = i0 >= 1 && i0 <= lat - 2, cin1 = i0 + 1 <= lat - 2;
  // Output weights with the column mask folded in (hoisted out of the step
  // loop): 0 on Dirichlet and padding columns, where x_out = x_in + 0 keeps the
  // boundary value (padding columns arrive as TMA zero fill and stay 0).
  double wgt[2][2];  // [row parity][column parity]
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int b = 0; b < 2; ++b)
      wgt[a][b] = (b ? cin1 : cin0)
                      ? (A.scalar_w ? A.omega : A.omega * (a ? 0.5 : 1.0 / 3.0) * (b ? 0.5 : 1.0 / 3.0))
                      : 0.0;
  const bool colout = owner && 2 * kxp < g.pu;
  double* const out_u = A.xout + g.oux + i0;  // dereferenced only when colout
  double* const out_v = A.xout + g.ouy + i0;
  RingFzS S = RingFzS::at(sB);
  double pmw[3][3];  // pressure window rolled across steps
  for (int s = sB; s <= sE; ++s) {
    // Data of step s (x pairs up to s+1, p rows up to s+2, b pair s, b_p row s+1)
    // arrived on barrier (s-sB+1)&1; prefetch step s+1 into the other one.
    // WAR safety with one CTA barrier per step (every thread has passed the
    // barrier of step s-1, so has finished step s-1's residual; it may still
    // be in step s-1's solve/output):
    //   x pair s+2 -> slot of pair s-4 (read last at step s-2's output)
    //   p row  s+3 -> slot of row  s-5;  b pair s+1 -> slot of pair s-1 (step s-1 residual)
    //   b_p row s+2 -> slot of row s (step s-1 residual)
    //   residual rows 2s+1, 2s+2 -> slots of rows 2s-6, 2s-5 (step s-2's solve)
    //   pressure residual row s+1 -> slot of row s-3 (step s-3's solve)
    const int bi = (s - sB + 1) & 1;
    mbar_wait(&bars[bi], (phases >> bi) & 1u);
    phases ^= 1u << bi;
    uint64_t* nbar = &bars[(s - sB) & 1];
    if (t == (((s - sB) & 1) << 5) % fz::kNT) {  // the issuing lane alternates between warps
      unsigned bytes = fz::kBBytes + fz::kBPBytes + (XZERO ? 0u : fz::kXBytes + fz::kPBytes);
      mbar_expect_tx(nbar, bytes);
      if (!XZERO) {
        tma_load_3d(sm + xpair(s + 2), &M.xv, xc0, 2 * s + 5, 0, nbar);
        tma_load_2d(sm + prow(s + 3), &M.xp, pc0, s + 3, nbar);
      }
      tma_load_3d(sm + bpair(s + 1), &M.bv, xc0 + 2, 2 * s + 3, 0, nbar);
      tma_load_2d(sm + bprow(s + 2), &M.bp, kx0 - 2, s + 2, nbar);
    }
    fused_residual_step(sm, A.g, F, s, kx0, S, pmw, s == sB);
    __syncthreads();

    // ---- patch solve (alg:vk line 2: A_i delta_i = V_i r, exactly) ----
    double vx[25], vy[25];
    double dp = 0.0;
    const bool valid = kxp >= 0 && kxp <= N && s >= 0 && s <= N;
    const bool generic = kxp >= 2 && kxp <= N - 2 && s >= 2 && s <= N - 2;
    if (valid && generic) {
#pragma unroll
      for (int oy = 0; oy < 5; ++oy) {  // window columns 2kxp-2.. = ring columns 2pi .. 2pi+4
        const double* ru = sm + S.rr(oy, 0) + 2 * pi;
        const double* rv = sm + S.rr(oy, 1) + 2 * pi;
        const double2 u01 = lds2(ru), u23 = lds2(ru + 2), v01 = lds2(rv), v23 = lds2(rv + 2);
        vx[oy * 5 + 0] = u01.x; vx[oy * 5 + 1] = u01.y; vx[oy * 5 + 2] = u23.x; vx[oy * 5 + 3] = u23.y;
        vx[oy * 5 + 4] = ru[4];
        vy[oy * 5 + 0] = v01.x; vy[oy * 5 + 1] = v01.y; vy[oy * 5 + 2] = v23.x; vy[oy * 5 + 3] = v23.y;
        vy[oy * 5 + 4] = rv[4];
      }
      dp = solve_generic_sym(vx, vy, sm[rprow(s) + pi + 1], F);
    } else if (valid) {  // precomputed by k_boundary_patches
      const int64_t nb = bd_count(N), bi = bd_index(kxp, s, N);
#pragma unroll
      for (int q = 0; q < 25; ++q) {
        vx[q] = A.bd[q * nb + bi];
        vy[q] = A.bd[(25 + q) * nb + bi];
      }
      dp = A.bd[50 * nb + bi];
    } else {
#pragma unroll
      for (int q = 0; q < 25; ++q) {
        vx[q] = 0.0;
        vy[q] = 0.0;
      }
    }
    // pressure: only patch k holds p_k (multiplicity 1) -> output now
    if (owner && s >= y0 && s < y1 && kxp < g.pp) {
      const double xp = XZERO ? 0.0 : sm[prow(s) + pi + 3];
      A.xout[g.op + (int64_t)s * g.pp + kxp] = kxp <= N ? fma(A.omega, dp, xp) : 0.0;
    }
    // ---- sum_i V_i^T delta_i on this lane's columns, lattice rows 2s-2 .. 2s+2,
    //      and x_out on rows 2s-2, 2s-1 (node row s-1), which are now complete ----
    const int ny = s - 1;
    const bool rowout = colout && ny >= y0 && ny < y1;  // the row test is uniform over the CTA
    // x_in of the output rows, loaded ahead of the shuffles (hides the shared-memory latency)
    double2 xin_o[2][2];  // [component][row parity]
    if (rowout) {
#pragma unroll
      for (int c = 0; c < 2; ++c)
#pragma unroll
        for (int rr = 0; rr < 2; ++rr) xin_o[c][rr] = lds2(sm + S.xr(rr - 2, c) + 2 * pi + 4);
    }
    double* const ou_row = out_u + (int64_t)(2 * ny) * g.pu;  // dereferenced only when rowout
#pragma unroll
    for (int c = 0; c < 2; ++c) {
      const double* v = c ? vy : vx;
      double S0[5], S1[5];
#pragma unroll
      for (int oy = 0; oy < 5; ++oy) {
        const double r0 = __shfl_down_sync(0xffffffffu, v[oy * 5 + 0], 1);  // patch pi+1, window column 0
        const double r1 = __shfl_down_sync(0xffffffffu, v[oy * 5 + 1], 1);  // patch pi+1, window column 1
        const double l4 = __shfl_up_sync(0xffffffffu, v[oy * 5 + 4], 1);    // patch pi-1, window column 4
        S0[oy] = oy < 3 ? carry[oy][c][0] + v[oy * 5 + 2] + l4 + r0 : v[oy * 5 + 2] + l4 + r0;
        S1[oy] = oy < 3 ? carry[oy][c][1] + v[oy * 5 + 3] + r1 : v[oy * 5 + 3] + r1;
      }
#pragma unroll
      for (int r = 0; r < 3; ++r) {
        carry[r][c][0] = S0[r + 2];
        carry[r][c][1] = S1[r + 2];
      }
      if (rowout) {
        double* const oc = ou_row + (c ? g.ouy - g.oux : 0);
#pragma unroll
        for (int rr = 0; rr < 2; ++rr) {
          const int j = 2 * ny + rr;  // rr = row parity
          if (j > lat - 1) continue;  // uniform: the row past the last lattice row
          const bool jin = j >= 1 && j <= lat - 2;  // uniform: Dirichlet rows keep x_in
          const double2 x = xin_o[c][rr];
          const double w0 = jin ? wgt[rr][0] : 0.0, w1 = jin ? wgt[rr][1] : 0.0;
          *reinterpret_cast<double2*>(oc + rr * g.pu) = make_double2(fma(w0, S0[rr], x.x), fma(w1, S1[rr], x.y));
        }
      }
    }
    S.advance();
  }
  // the last prefetch (for step sE+1) must land before the CTA's shared memory is released
  mbar_wait(&bars[(sE - sB) & 1], (phases >> ((sE - sB) & 1)) & 1u);
}

// -----------------------------------------------------------------------------
// Pre-smoothing from zero (alg:mg line 2 on a V-cycle level entered with x = 0,
// P:146): the residual IS b, and every generic patch window lies in the interior
// (no Dirichlet point to mask), so this specialised kernel reads the patch
// windows straight from a 4-pair b ring -- no residual phase, no residual ring,
// no x loads: x_out = W sum_i V_i^T A_i^{-1} V_i b.  Same strip / warp layout and
// owner-computes accumulation as k_vanka_fused; boundary patches from `bd`.
// -----------------------------------------------------------------------------
namespace fz0 {
constexpr int BPR = 4, BPP = 4;  // b row pairs, b_p rows (slots = index & 3)
constexpr int OBS = 0;
constexpr int OBP = OBS + BPR * 4 * fz::W;
constexpr int OMB = OBP + BPP * fz::PWID;
constexpr int kSmemBytes = (OMB + 2) * 8;
}  // namespace fz0
__device__ __forceinline__ int z0_brow(int j, int c) {
  return fz0::OBS + (((j - 1) >> 1) & 3) * 4 * fz::W + c * 2 * fz::W + ((j - 1) & 1) * fz::W;
}
__device__ __forceinline__ int z0_bprow(int r) { return fz0::OBP + (r & 3) * fz::PWID; }

__global__ void __launch_bounds__(fz::kNT, fz::kMinB) k_vanka_zero(const FusedArgs A, const FusedFactors F,
                                                            const __grid_constant__ FusedMaps M) {
  extern __shared__ __align__(1024) double sm[];
  const LevelGeom& g = A.g;
  const int N = g.N, lat = g.lat;
  const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
  const int kx0 = blockIdx.x * fz::kNOUT;
  const int y0 = g.r0 + blockIdx.y * A.chunk;
  const int y1 = min(y0 + A.chunk, g.r1);
  if (y0 >= y1) return;
  const int xc0 = 2 * kx0 - 6;
  const int sB = y0 - 1, sE = y1;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sm + fz0::OMB);
  unsigned phases = 0u;
  if (t == 0) {
    mbar_init(&bars[0], 1);
    mbar_init(&bars[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  pdl_wait();
  // data of step sB: b pairs sB-2 .. sB (rows 2sB-3 .. 2sB+2), b_p row sB -> barrier 0
  if (t == 0) {
    mbar_expect_tx(&bars[0], 3 * fz::kBBytes + fz::kBPBytes);
    for (int p = sB - 2; p <= sB; ++p)
      tma_load_3d(sm + z0_brow(2 * p + 1, 0), &M.bv, xc0 + 2, 2 * p + 1, 0, &bars[0]);
    tma_load_2d(sm + z0_bprow(sB), &M.bp, kx0 - 2, sB, &bars[0]);
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
  double wgt[2][2];  // [row parity][column parity], column mask folded in (as k_vanka_fused)
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int b = 0; b < 2; ++b)
      wgt[a][b] = (b ? cin1 : cin0)
                      ? (A.scalar_w ? A.omega : A.omega * (a ? 0.5 : 1.0 / 3.0) * (b ? 0.5 : 1.0 / 3.0))
                      : 0.0;
  const bool colout = owner && 2 * kxp < g.pu;
  double* const out_u = A.xout + g.oux + i0;  // dereferenced only when colout
  for (int s = sB; s <= sE; ++s) {
    // step s: b pair s and b_p row s arrived on barrier (s-sB)&1.  After the CTA
    // barrier every thread has finished step s-1 (windows of pairs s-3 .. s-1),
    // so pair s+1 may replace the slot of pair s-3 and b_p row s+1 that of s-3.
    const int bi = (s - sB) & 1;
    mbar_wait(&bars[bi], (phases >> bi) & 1u);
    phases ^= 1u << bi;
    __syncthreads();
    if (t == (bi << 5) % fz::kNT) {  // the issuing lane alternates between warps
      uint64_t* nbar = &bars[bi ^ 1];
      mbar_expect_tx(nbar, fz::kBBytes + fz::kBPBytes);
      tma_load_3d(sm + z0_brow(2 * s + 3, 0), &M.bv, xc0 + 2, 2 * s + 3, 0, nbar);
      tma_load_2d(sm + z0_bprow(s + 1), &M.bp, kx0 - 2, s + 1, nbar);
    }
    double vx[25], vy[25];
    double dp = 0.0;
    const bool valid = kxp >= 0 && kxp <= N && s >= 0 && s <= N;
    const bool generic = kxp >= 2 && kxp <= N - 2 && s >= 2 && s <= N - 2;
    if (valid && generic) {  // window rows 2s-2 .. 2s+2, columns 2kxp-2 .. = b ring columns 2pi ..
#pragma unroll
      for (int oy = 0; oy < 5; ++oy) {
        const double* ru = sm + z0_brow(2 * s - 2 + oy, 0) + 2 * pi;
        const double* rv = sm + z0_brow(2 * s - 2 + oy, 1) + 2 * pi;
        const double2 u01 = lds2(ru), u23 = lds2(ru + 2), v01 = lds2(rv), v23 = lds2(rv + 2);
        vx[oy * 5 + 0] = u01.x; vx[oy * 5 + 1] = u01.y; vx[oy * 5 + 2] = u23.x; vx[oy * 5 + 3] = u23.y;
        vx[oy * 5 + 4] = ru[4];
        vy[oy * 5 + 0] = v01.x; vy[oy * 5 + 1] = v01.y; vy[oy * 5 + 2] = v23.x; vy[oy * 5 + 3] = v23.y;
        vy[oy * 5 + 4] = rv[4];
      }
      dp = solve_generic_sym(vx, vy, sm[z0_bprow(s) + pi + 1], F);
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
    if (owner && s >= y0 && s < y1 && kxp < g.pp)
      A.xout[g.op + (int64_t)s * g.pp + kxp] = kxp <= N ? A.omega * dp : 0.0;
    const int ny = s - 1;
    const bool rowout = colout && ny >= y0 && ny < y1;  // the row test is uniform over the CTA
    double* const ou_row = out_u + (int64_t)(2 * ny) * g.pu;
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
        double* const oc = ou_row + (c ? g.ouy - g.oux : 0);
#pragma unroll
        for (int rr = 0; rr < 2; ++rr) {
          const int j = 2 * ny + rr;
          if (j > lat - 1) continue;                // uniform
          const bool jin = j >= 1 && j <= lat - 2;  // uniform: Dirichlet rows are 0
          const double w0 = jin ? wgt[rr][0] : 0.0, w1 = jin ? wgt[rr][1] : 0.0;
          *reinterpret_cast<double2*>(oc + rr * g.pu) = make_double2(w0 * S0[rr], w1 * S1[rr]);
        }
      }
    }
  }
  const int bl = (sE + 1 - sB) & 1;
  mbar_wait(&bars[bl], (phases >> bl) & 1u);
}

// -----------------------------------------------------------------------------
// Validation mode ("only 25 different patch matrices",
// S:391).  Tuned Vanka stores one inverse per group (category pair) and, for
// the generic group, the reflection-basis Schur factors; validation rebuilds
// every patch's own inverse (k_patch_setup_simple, in batches) and compares it
// with the stored inverse of its group, and applies the generic factors to the
// 51 unit vectors and compares the result with the generic group's inverse.
// Deviations are |a - b| / max|group inverse|, maximised with an atomicMax on
// the bit pattern (monotone for non-negative doubles).
// -----------------------------------------------------------------------------
__device__ __forceinline__ void atomic_max_nonneg(double* addr, double v) {
  atomicMax(reinterpret_cast<unsigned long long*>(addr), (unsigned long long)__double_as_longlong(v));
}
// batch entry (q, i): patch p0 + i, slot pair q = r * 51 + c
__global__ void k_validate_batch(LevelGeom g, int64_t p0, int64_t nb, const double* __restrict__ batch,
                                 const double* __restrict__ ginv, const double* __restrict__ gscale,
                                 double* __restrict__ maxdev) {
  const int N = g.N;
  const int64_t np = (int64_t)(N + 1) * (N + 1);
  double dev = 0.0;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < nb * kGroupStride;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e % nb, q = e / nb, p = p0 + i;
    if (p >= np) continue;
    const int kx = (int)(p % (N + 1)), ky = (int)(p / (N + 1));
    const int grp = pcat(ky, N) * 5 + pcat(kx, N);
    const double d = fabs(batch[q * nb + i] - ginv[(int64_t)grp * kGroupStride + q]) / gscale[grp];
    dev = d > dev ? d : dev;  // NaN-safe below: a NaN difference is reported as +inf
    if (d != d) dev = INFINITY;
  }
  for (int o = 16; o > 0; o >>= 1) dev = fmax(dev, __shfl_xor_sync(0xffffffffu, dev, o));
  if ((threadIdx.x & 31) == 0) atomic_max_nonneg(maxdev, dev);
}
// column q of the generic patch's inverse through the structured solve
// (solve_generic_sym) vs the generic group's stored dense inverse
__global__ void k_validate_factors(const FusedFactors F, const double* __restrict__ ginv12, double gscale,
                                   double* __restrict__ maxdev) {
  const int q = threadIdx.x;
  if (q >= kSlots) return;
  double vx[25], vy[25];
#pragma unroll
  for (int k = 0; k < 25; ++k) {
    vx[k] = (q == k) ? 1.0 : 0.0;
    vy[k] = (q == 25 + k) ? 1.0 : 0.0;
  }
  const double dp = solve_generic_sym(vx, vy, q == 50 ? 1.0 : 0.0, F);
  double dev = 0.0;
  for (int r = 0; r < kSlots; ++r) {
    const double v = r < 25 ? vx[r] : (r < 50 ? vy[r - 25] : dp);
    const double d = fabs(v - ginv12[r * kSlots + q]) / gscale;
    dev = (d > dev || d != d) ? (d != d ? INFINITY : d) : dev;
  }
  atomic_max_nonneg(maxdev, dev);
}

inline int launch_factor_setup(const int* d_Ns, int nlev, double nu, const double* /*d_inv*/, double* d_fac,
                               int* d_status) {
  k_factor_setup<<<nlev, 256>>>(d_Ns, nu, d_fac, d_status);
  return 0;
}

// chunk height: about `waves` full waves of 2 CTAs per SM over the strips
inline int fused_chunk(const LevelGeom& g, int nstrips, int nsm) {
  const int rows = g.r1 - g.r0;
  const int resident = fz::kMinB * nsm;
  static const double target = [] {  // node rows per CTA the wave count aims at (SVK_CHUNK_ROWS: tuning aid)
    const char* e = std::getenv("SVK_CHUNK_ROWS");
    return e ? std::atof(e) : 64.0;
  }();
  const double work = (double)nstrips * rows / target;
  int waves = (int)(work / resident + 0.5);
  if (waves < 1) waves = 1;
  int chunks = (resident * waves) / nstrips;
  if (chunks < 1) chunks = 1;
  if (chunks > rows) chunks = rows;
  return (rows + chunks - 1) / chunks;
}

// ---- host: TMA descriptors --------------------------------------------------
typedef CUresult (*PFN_encodeTiled)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                    const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                    CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
inline PFN_encodeTiled get_encode() {
  static const PFN_encodeTiled fn = [] {  // thread-safe one-time lookup
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      return (PFN_encodeTiled)p;
    return (PFN_encodeTiled) nullptr;
  }();
  return fn;
}
// the last TMA descriptor encoding failure of this thread (for error messages)
inline std::string& tma_error() {
  static thread_local std::string e;
  return e;
}
inline bool tma_encoded(CUresult r, const char* what, const void* base) {
  if (r == CUDA_SUCCESS) return true;
  char buf[160];
  std::snprintf(buf, sizeof buf, "cuTensorMapEncodeTiled(%s, base %p) failed: CUresult %d", what, base, (int)r);
  tma_error() = buf;
  return false;
}
// velocity planes of a vector: dims {lat cols, lat rows, 2 comps}; box {256, 2, 2}
inline bool make_vel_map(CUtensorMap* m, const LevelGeom& g, const double* v, unsigned boxw = fz::W) {
  PFN_encodeTiled enc = get_encode();
  if (!enc) return tma_encoded(CUDA_ERROR_NOT_FOUND, "entry point", v);
  const cuuint64_t dims[3] = {(cuuint64_t)g.lat, (cuuint64_t)g.lat, 2};
  const cuuint64_t strides[2] = {(cuuint64_t)g.pu * 8, (cuuint64_t)(g.ouy - g.oux) * 8};
  const cuuint32_t box[3] = {boxw, 2, 2};
  const cuuint32_t es[3] = {1, 1, 1};
  return tma_encoded(enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, (void*)(v + g.oux), dims, strides, box, es,
                         CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                         CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE),
                     "velocity", v);
}
// pressure plane: dims {N+1, N+1}; box {boxw, 1}
inline bool make_p_map(CUtensorMap* m, const LevelGeom& g, const double* v, unsigned boxw) {
  PFN_encodeTiled enc = get_encode();
  if (!enc) return false;
  const cuuint64_t dims[2] = {(cuuint64_t)(g.N + 1), (cuuint64_t)(g.N + 1)};
  const cuuint64_t strides[1] = {(cuuint64_t)g.pp * 8};
  const cuuint32_t box[2] = {boxw, 1};
  const cuuint32_t es[2] = {1, 1};
  return tma_encoded(enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, (void*)(v + g.op), dims, strides, box, es,
                         CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                         CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE),
                     "pressure", v);
}

inline int launch_fused_sweep(const LevelGeom& g, double nu, double omega, int scalar_w, const FusedFactors& F,
                              const double* dinv, const BdTile* tiles, int ntiles, double* bd, const double* xin,
                              const double* b, double* xout, int nsm, cudaStream_t s, cudaEvent_t ev0 = nullptr,
                              unsigned ev0_flags = 0) {
  launch_pdl(k_boundary_patches, dim3((unsigned)ntiles), dim3(kBdThreads), 0, s, g, nu, dinv, tiles, xin, b, bd);
  // profiling: the caller's start event between the two kernels times the sweep kernel alone
  if (ev0 && cudaEventRecordWithFlags(ev0, s, ev0_flags) != cudaSuccess) return -3;
  static bool attr_done[64] = {false};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev >= 0 && dev < 64 && !attr_done[dev]) {
    cudaFuncSetAttribute(k_vanka_fused<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, fz::kSmemBytes);
    cudaFuncSetAttribute(k_vanka_zero, cudaFuncAttributeMaxDynamicSharedMemorySize, fz0::kSmemBytes);
    attr_done[dev] = true;
  }
  const int ncover = (int)std::max<int64_t>(g.pu / 2, g.pp);
  const int nstrips = (ncover + fz::kNOUT - 1) / fz::kNOUT;
  FusedArgs A{g, omega, scalar_w, 0, bd, xout};
  A.chunk = fused_chunk(g, nstrips, nsm);
  FusedMaps M;
  std::memset(&M, 0, sizeof(M));
  if (!make_vel_map(&M.bv, g, b) || !make_p_map(&M.bp, g, b, fz::PWID)) return -2;
  if (xin && (!make_vel_map(&M.xv, g, xin, fz::WX) || !make_p_map(&M.xp, g, xin, fz::PXW))) return -2;
  const dim3 grid(nstrips, (g.r1 - g.r0 + A.chunk - 1) / A.chunk);
  if (xin) launch_pdl(k_vanka_fused<false>, grid, dim3(fz::kNT), fz::kSmemBytes, s, A, F, M);
  else launch_pdl(k_vanka_zero, grid, dim3(fz::kNT), fz0::kSmemBytes, s, A, F, M);
  return 0;
}

}  // namespace svk
