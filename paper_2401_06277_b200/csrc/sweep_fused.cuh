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
// kernel -- one CTA of 64 threads per patch: the 51 window residuals
// (stencil from global memory), then one row of the dense padded group
// inverse per thread -- and their corrections are stored slot-major in `bd`.
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

__global__ void __launch_bounds__(64) k_boundary_patches(LevelGeom g, double nu, const double* __restrict__ dinv,
                                                        const double* __restrict__ x, const double* __restrict__ b,
                                                        double* __restrict__ bd) {
  const int N = g.N, lat = g.lat;
  const int64_t nb = bd_count(N);
  const int64_t id = blockIdx.x;
  int kx, ky;
  if (id < 4 * (int64_t)(N + 1)) {
    const int r = (int)(id / (N + 1));
    ky = r <= 1 ? r : r + N - 3;
    kx = (int)(id % (N + 1));
  } else {
    const int64_t q = id - 4 * (int64_t)(N + 1);
    const int c = (int)(q / (N - 3));
    kx = c <= 1 ? c : c + N - 3;
    ky = 2 + (int)(q % (N - 3));
  }
  __shared__ double rv[kSlots];
  const int s = threadIdx.x;
  if (s < kSlots) {
    double r = 0.0;
    if (s < 50) {
      const int comp = s / 25, oy = (s % 25) / 5, ox = s % 5;
      const int i = 2 * kx - 2 + ox, j = 2 * ky - 2 + oy;
      if (i >= 1 && j >= 1 && i <= lat - 2 && j <= lat - 2) {
        const int64_t o = (comp ? g.ouy : g.oux) + (int64_t)j * g.pu + i;
        double ax = 0.0;
        if (x) ax = nu * lap_at(x + (comp ? g.ouy : g.oux), g.pu, i, j) + gradp_at(x + g.op, g.pp, i, j, comp, g.h);
        r = b[o] - ax;
      }
    } else {
      const double ax = x ? div_at(x + g.oux, x + g.ouy, g.pu, N, kx, ky, g.h) : 0.0;
      r = b[p_at(g, kx, ky)] - ax;
    }
    rv[s] = r;
  }
  __syncthreads();
  if (s < kSlots) {
    const double* A = dinv + (size_t)(pcat(ky, N) * 5 + pcat(kx, N)) * kGroupStride + s * kSlots;
    double d = 0.0;
    for (int q = 0; q < kSlots; ++q) d = fma(A[q], rv[q], d);
    bd[(int64_t)s * nb + bd_index(kx, ky, N)] = d;
  }
}

// =============================================================================
// Fused additive Vanka sweep (alg:vk) -- one kernel per sweep:
//   x_out = x_in + W sum_i V_i^T A_i^{-1} V_i (b - A x_in)
//
// Layout of the work ("owner computes", no atomics, deterministic):
//  * a CTA of kNT = 128 threads owns a STRIP of kNOUT = 124 node columns
//    [kx0, kx0+124) and a CHUNK of node rows [y0, y1); it streams upward
//    through the chunk one node row (= one patch row = two lattice rows) per
//    step, keeping rings of rows in shared memory:
//      x ring (9 lattice rows, both components), p ring (4 node rows),
//      residual ring (6 lattice rows), pressure-residual ring (2 rows),
//      accumulator ring (6 lattice rows);
//    every ring row is split by column parity, so thread t touches
//    consecutive doubles (no bank conflicts).
//  * step s: (1) prefetch the x / p rows of step s+1 (cp.async, zero-filled
//    outside the domain); (2) residual r = b - A x on lattice rows 2s+1, 2s+2
//    (thread t: lattice columns rc0+2t, rc0+2t+1) and the pressure residual on
//    node row s+1; (3) thread t solves patch (kx0-1+t, s) exactly -- generic
//    patches with the parity-blocked Schur form, boundary patches with their
//    dense 51x51 group inverse -- and adds W-less contributions into the
//    accumulator in three conflict-free phases (own columns, left neighbour's,
//    right neighbour's); (4) lattice rows 2s-2, 2s-1 are now complete: write
//    x_out = x_in + w * acc for the owned columns.
//  * patches and residuals are recomputed by both neighbouring strips at a
//    strip edge (2 patch columns and 7 lattice columns per 124 node columns).
// =============================================================================
namespace fz {
constexpr int kNT = 128, kNPATCH = 126, kNOUT = 124;
constexpr int XR = 9, XH = 132;   // x ring: rows, doubles per parity half (columns xc0 .. xc0+263)
constexpr int PR = 4, PW = 136;   // p ring: rows, columns pc0 .. pc0+135
constexpr int RR = 6, RH = 128;   // residual ring: rows, doubles per parity half (columns rc0 .. rc0+255)
constexpr int AR = 6;             // accumulator ring rows (same columns as the residual ring)
constexpr int kSmemDoubles = XR * 4 * XH + PR * PW + RR * 4 * RH + 2 * RH + AR * 4 * RH;
constexpr int kSmemBytes = kSmemDoubles * 8;
}  // namespace fz

struct FusedArgs {
  LevelGeom g;
  double omega;
  int scalar_w;
  int chunk;            // node rows per CTA
  const double* bd;     // boundary-patch corrections (k_boundary_patches), slot-major
  const double* xin;    // unused when the kernel is instantiated with XZERO
  const double* b;
  double* xout;
};

__device__ __forceinline__ int pmod(int a, int m) {
  const int r = a % m;
  return r < 0 ? r + m : r;
}
__device__ __forceinline__ void cp_async8(void* smem, const void* gmem, bool valid) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  const int sz = valid ? 8 : 0;
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(s), "l"(gmem), "r"(sz) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
__device__ __forceinline__ void cp_wait_all() { asm volatile("cp.async.wait_group 0;\n" ::: "memory"); }

struct FusedSmem {
  double* xs;   // [XR][comp][par][XH]
  double* ps;   // [PR][PW]
  double* rs;   // [RR][comp][par][RH]
  double* rps;  // [2][RH]
  double* as;   // [AR][comp][par][RH]
  __device__ __forceinline__ double& X(int j, int comp, int par, int q) const {
    return xs[((pmod(j, fz::XR) * 2 + comp) * 2 + par) * fz::XH + q];
  }
  __device__ __forceinline__ double& Pp(int row, int q) const { return ps[(row & 3) * fz::PW + q]; }
  __device__ __forceinline__ double& R(int j, int comp, int par, int q) const {
    return rs[((pmod(j, fz::RR) * 2 + comp) * 2 + par) * fz::RH + q];
  }
  __device__ __forceinline__ double& RP(int row, int q) const { return rps[(row & 1) * fz::RH + q]; }
  __device__ __forceinline__ double& Acc(int j, int comp, int par, int q) const {
    return as[((pmod(j, fz::AR) * 2 + comp) * 2 + par) * fz::RH + q];
  }
};

// x lattice row j (both components), columns xc0 .. xc0+263, zero outside the domain
__device__ __forceinline__ void load_x_row(const FusedSmem& S, const LevelGeom& g, const double* __restrict__ x, int j,
                                           int xc0) {
  const bool rowok = j >= 0 && j < g.lat;
  for (int comp = 0; comp < 2; ++comp) {
    const double* base = x + (comp ? g.ouy : g.oux);
    for (int q = threadIdx.x; q < 2 * fz::XH; q += fz::kNT) {
      const int c = xc0 + q;
      const bool ok = rowok && c >= 0 && c < g.lat;
      cp_async8(&S.X(j, comp, q & 1, q >> 1), ok ? base + (int64_t)j * g.pu + c : base, ok);
    }
  }
}
__device__ __forceinline__ void load_p_row(const FusedSmem& S, const LevelGeom& g, const double* __restrict__ x,
                                           int row, int pc0) {
  const bool rowok = row >= 0 && row <= g.N;
  const double* base = x + g.op;
  for (int q = threadIdx.x; q < fz::PW; q += fz::kNT) {
    const int c = pc0 + q;
    const bool ok = rowok && c >= 0 && c <= g.N;
    cp_async8(&S.Pp(row & 3, q), ok ? base + (int64_t)row * g.pp + c : base, ok);
  }
}

// Residual on lattice rows 2sp+1 (odd) and 2sp+2 (even), lattice columns
// c0 = rc0 + 2t (even) and c0+1, both components; pressure residual at node
// (kx0-2+t, sp+1).  Uses x rows 2sp..2sp+4 and p rows sp..sp+2.
template <bool XZERO>
__device__ __forceinline__ void fused_residual(const FusedSmem& S, const FusedArgs& A, const FusedFactors& F, int sp,
                                               int kx0) {
  const LevelGeom& g = A.g;
  const int N = g.N, lat = g.lat, t = threadIdx.x;
  const int rc0 = 2 * kx0 - 4;
  const int c0 = rc0 + 2 * t;
  const int j0 = 2 * sp + 1, j1 = 2 * sp + 2;
  const bool c0ok = c0 >= 1 && c0 <= lat - 2, c1ok = c0 + 1 >= 1 && c0 + 1 <= lat - 2;
  const bool j0ok = j0 >= 1 && j0 <= lat - 2, j1ok = j1 >= 1 && j1 <= lat - 2;
  double ax[2][4];  // [comp][(j0,c0) (j0,c0+1) (j1,c0) (j1,c0+1)]
  double bu = 0.0;  // B u at the pressure node
  const int na = kx0 - 2 + t, nrow = sp + 1;
  const bool pok = na >= 0 && na <= N && nrow >= 0 && nrow <= N;
  const bool pint = na >= 1 && na <= N - 1 && nrow >= 1 && nrow <= N - 1;
  if (!XZERO) {
#pragma unroll
    for (int comp = 0; comp < 2; ++comp) {
      double V[5][5];
#pragma unroll
      for (int r = 0; r < 5; ++r) {
        const int j = 2 * sp + r;
        V[r][0] = S.X(j, comp, 0, t);
        V[r][1] = S.X(j, comp, 1, t);
        V[r][2] = S.X(j, comp, 0, t + 1);
        V[r][3] = S.X(j, comp, 1, t + 1);
        V[r][4] = S.X(j, comp, 0, t + 2);
      }
      double l00 = 0, l01 = 0, l10 = 0, l11 = 0;
#pragma unroll
      for (int b = -1; b <= 1; ++b) {
#pragma unroll
        for (int a = -2; a <= 2; ++a) l00 = fma(F.L2D[1][0][b + 2][a + 2], V[1 + b][2 + a], l00);
#pragma unroll
        for (int a = -1; a <= 1; ++a) l01 = fma(F.L2D[1][1][b + 2][a + 2], V[1 + b][3 + a], l01);
      }
#pragma unroll
      for (int b = -2; b <= 2; ++b) {
#pragma unroll
        for (int a = -2; a <= 2; ++a) l10 = fma(F.L2D[0][0][b + 2][a + 2], V[2 + b][2 + a], l10);
#pragma unroll
        for (int a = -1; a <= 1; ++a) l11 = fma(F.L2D[0][1][b + 2][a + 2], V[2 + b][3 + a], l11);
      }
      ax[comp][0] = l00;
      ax[comp][1] = l01;
      ax[comp][2] = l10;
      ax[comp][3] = l11;
      // B u at node (na, nrow): window rows 2sp..2sp+4 = V rows, columns 2na-2.. = V columns
      if (pint) {
        if (comp == 0) {
#pragma unroll
          for (int oy = 1; oy <= 3; ++oy) {
            bu = fma(F.PBX[oy][0], V[oy][0], bu);
            bu = fma(F.PBX[oy][1], V[oy][1], bu);
            bu = fma(F.PBX[oy][3], V[oy][3], bu);
            bu = fma(F.PBX[oy][4], V[oy][4], bu);
          }
        } else {
#pragma unroll
          for (int oy = 0; oy < 5; ++oy) {
            if (oy == 2) continue;
            bu = fma(F.PBY[oy][1], V[oy][1], bu);
            bu = fma(F.PBY[oy][2], V[oy][2], bu);
            bu = fma(F.PBY[oy][3], V[oy][3], bu);
          }
        }
      } else if (pok) {  // boundary pressure node: general rows from the class tables
        const int cx = na == 0 ? 0 : (na == N ? 2 : 1), cy = nrow == 0 ? 0 : (nrow == N ? 2 : 1);
        double s = 0.0;
#pragma unroll
        for (int oy = 0; oy < 5; ++oy)
#pragma unroll
          for (int ox = 0; ox < 5; ++ox)
            s += (comp == 0 ? c_st.CR[cy][oy] * c_st.GR[cx][ox] : c_st.GR[cy][oy] * c_st.CR[cx][ox]) * V[oy][ox];
        bu = fma(-g.h, s, bu);
      }
    }
    // B^T p: p rows sp..sp+2, node columns kx0-3+t .. (p-array q = t .. t+2)
    double Pm[3][3];
#pragma unroll
    for (int r = 0; r < 3; ++r)
#pragma unroll
      for (int q = 0; q < 3; ++q) Pm[r][q] = S.Pp(sp + r, t + q);
    // odd row j0 = 2sp+1: nodes ky = sp, sp+1 (ty 0,1); even row j1: ky = sp..sp+2 (ty 0..2)
    // even column c0: kx = q 0..2 (G col nonzero at 0,2; C^ col nonzero at 1); odd column: q 1..2
    ax[0][0] += F.GX[1][0][0][0] * Pm[0][0] + F.GX[1][0][0][2] * Pm[0][2] + F.GX[1][0][1][0] * Pm[1][0] +
                F.GX[1][0][1][2] * Pm[1][2];
    ax[0][1] += F.GX[1][1][0][0] * Pm[0][1] + F.GX[1][1][0][1] * Pm[0][2] + F.GX[1][1][1][0] * Pm[1][1] +
                F.GX[1][1][1][1] * Pm[1][2];
    ax[0][2] += F.GX[0][0][1][0] * Pm[1][0] + F.GX[0][0][1][2] * Pm[1][2];
    ax[0][3] += F.GX[0][1][1][0] * Pm[1][1] + F.GX[0][1][1][1] * Pm[1][2];
    ax[1][0] += F.GY[1][0][0][1] * Pm[0][1] + F.GY[1][0][1][1] * Pm[1][1];
    ax[1][1] += F.GY[1][1][0][0] * Pm[0][1] + F.GY[1][1][0][1] * Pm[0][2] + F.GY[1][1][1][0] * Pm[1][1] +
                F.GY[1][1][1][1] * Pm[1][2];
    ax[1][2] += F.GY[0][0][0][1] * Pm[0][1] + F.GY[0][0][2][1] * Pm[2][1];
    ax[1][3] += F.GY[0][1][0][0] * Pm[0][1] + F.GY[0][1][0][1] * Pm[0][2] + F.GY[0][1][2][0] * Pm[2][1] +
                F.GY[0][1][2][1] * Pm[2][2];
  } else {
#pragma unroll
    for (int comp = 0; comp < 2; ++comp)
#pragma unroll
      for (int q = 0; q < 4; ++q) ax[comp][q] = 0.0;
  }
  // r = b - A x, masked; store to the residual ring
#pragma unroll
  for (int comp = 0; comp < 2; ++comp) {
    const double* bb = A.b + (comp ? g.ouy : g.oux);
    double b00 = 0, b01 = 0, b10 = 0, b11 = 0;
    if (j0ok && (c0ok || c1ok)) {
      const double2 v = *reinterpret_cast<const double2*>(bb + (int64_t)j0 * g.pu + c0);
      b00 = v.x;
      b01 = v.y;
    }
    if (j1ok && (c0ok || c1ok)) {
      const double2 v = *reinterpret_cast<const double2*>(bb + (int64_t)j1 * g.pu + c0);
      b10 = v.x;
      b11 = v.y;
    }
    S.R(j0, comp, 0, t) = (j0ok && c0ok) ? b00 - ax[comp][0] : 0.0;
    S.R(j0, comp, 1, t) = (j0ok && c1ok) ? b01 - ax[comp][1] : 0.0;
    S.R(j1, comp, 0, t) = (j1ok && c0ok) ? b10 - ax[comp][2] : 0.0;
    S.R(j1, comp, 1, t) = (j1ok && c1ok) ? b11 - ax[comp][3] : 0.0;
  }
  S.RP(nrow, t) = pok ? A.b[g.op + (int64_t)nrow * g.pp + na] - bu : 0.0;
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
// yhat = B rhat, block by block, in place (transformed index ty*5+tx)
__device__ __forceinline__ void apply_blocks(double (&v)[25], const FusedFactors& F) {
  {  // EE: ty,tx in {0,1,2}
    double in[9], out[9];
#pragma unroll
    for (int q = 0; q < 9; ++q) in[q] = v[(q / 3) * 5 + q % 3];
#pragma unroll
    for (int r = 0; r < 9; ++r) {
      double s = 0.0;
#pragma unroll
      for (int q = 0; q < 9; ++q) s = fma(F.bee[r][q], in[q], s);
      out[r] = s;
    }
#pragma unroll
    for (int q = 0; q < 9; ++q) v[(q / 3) * 5 + q % 3] = out[q];
  }
  {  // EO: ty in {0,1,2}, tx in {3,4}
    double in[6], out[6];
#pragma unroll
    for (int q = 0; q < 6; ++q) in[q] = v[(q / 2) * 5 + 3 + q % 2];
#pragma unroll
    for (int r = 0; r < 6; ++r) {
      double s = 0.0;
#pragma unroll
      for (int q = 0; q < 6; ++q) s = fma(F.beo[r][q], in[q], s);
      out[r] = s;
    }
#pragma unroll
    for (int q = 0; q < 6; ++q) v[(q / 2) * 5 + 3 + q % 2] = out[q];
  }
  {  // OE: ty in {3,4}, tx in {0,1,2}
    double in[6], out[6];
#pragma unroll
    for (int q = 0; q < 6; ++q) in[q] = v[(3 + q / 3) * 5 + q % 3];
#pragma unroll
    for (int r = 0; r < 6; ++r) {
      double s = 0.0;
#pragma unroll
      for (int q = 0; q < 6; ++q) s = fma(F.boe[r][q], in[q], s);
      out[r] = s;
    }
#pragma unroll
    for (int q = 0; q < 6; ++q) v[(3 + q / 3) * 5 + q % 3] = out[q];
  }
  {  // OO
    double in[4], out[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) in[q] = v[(3 + q / 2) * 5 + 3 + q % 2];
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      double s = 0.0;
#pragma unroll
      for (int q = 0; q < 4; ++q) s = fma(F.boo[r][q], in[q], s);
      out[r] = s;
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) v[(3 + q / 2) * 5 + 3 + q % 2] = out[q];
  }
}

// Generic patch: (vx, vy, rp) = patch residual in; (vx, vy) = (du, dv) out; returns dp.
__device__ __forceinline__ double solve_generic(double (&vx)[25], double (&vy)[25], double rp, const FusedFactors& F) {
  fwd_transform(vx);
  fwd_transform(vy);
  double sx = 0.0, sy = 0.0;
#pragma unroll
  for (int q = 0; q < 6; ++q) {
    sx = fma(F.chx[q], vx[(q / 2) * 5 + 3 + q % 2], sx);
    sy = fma(F.chy[q], vy[(3 + q / 3) * 5 + q % 3], sy);
  }
  const double dp = (sx + sy - rp) * F.inv_sigma;
  apply_blocks(vx, F);
  apply_blocks(vy, F);
#pragma unroll
  for (int q = 0; q < 6; ++q) {
    vx[(q / 2) * 5 + 3 + q % 2] = fma(-F.cpx[q], dp, vx[(q / 2) * 5 + 3 + q % 2]);
    vy[(3 + q / 3) * 5 + q % 3] = fma(-F.cpy[q], dp, vy[(3 + q / 3) * 5 + q % 3]);
  }
  inv_transform(vx);
  inv_transform(vy);
  return dp;
}

template <bool XZERO>
__global__ void __launch_bounds__(fz::kNT, 2) k_vanka_fused(const FusedArgs A, const FusedFactors F) {
  extern __shared__ double smem[];
  FusedSmem S;
  S.xs = smem;
  S.ps = S.xs + fz::XR * 4 * fz::XH;
  S.rs = S.ps + fz::PR * fz::PW;
  S.rps = S.rs + fz::RR * 4 * fz::RH;
  S.as = S.rps + 2 * fz::RH;
  const LevelGeom& g = A.g;
  const int N = g.N, lat = g.lat;
  const int t = threadIdx.x;
  const int kx0 = blockIdx.x * fz::kNOUT;
  const int y0 = blockIdx.y * A.chunk;
  const int y1 = min(y0 + A.chunk, N + 1);
  if (y0 >= y1) return;
  const int xc0 = 2 * kx0 - 6, pc0 = kx0 - 3;
  const int sB = y0 - 1, sE = y1;
  const double* xin = A.xin;

  for (int q = t; q < fz::AR * 4 * fz::RH; q += fz::kNT) S.as[q] = 0.0;
  if (!XZERO) {
    for (int j = 2 * sB - 4; j <= 2 * sB + 4; ++j) load_x_row(S, g, xin, j, xc0);
    for (int r = sB - 2; r <= sB + 1; ++r) load_p_row(S, g, xin, r, pc0);
    cp_commit();
    cp_wait_all();
  }
  __syncthreads();
  fused_residual<XZERO>(S, A, F, sB - 2, kx0);
  fused_residual<XZERO>(S, A, F, sB - 1, kx0);
  __syncthreads();
  if (!XZERO) {
    load_p_row(S, g, xin, sB + 2, pc0);
    cp_commit();
    cp_wait_all();
  }
  __syncthreads();

  const int kxp = kx0 - 1 + t;  // this thread's patch column
  for (int s = sB; s <= sE; ++s) {
    if (!XZERO) {
      load_x_row(S, g, xin, 2 * s + 5, xc0);
      load_x_row(S, g, xin, 2 * s + 6, xc0);
      load_p_row(S, g, xin, s + 3, pc0);
      cp_commit();
    }
    fused_residual<XZERO>(S, A, F, s, kx0);
    __syncthreads();

    // ---- patch solve (alg:vk line 2: A_i delta_i = V_i r, exactly) ----
    double vx[25], vy[25];
    double dp = 0.0;
    const bool valid = t < fz::kNPATCH && kxp >= 0 && kxp <= N && s >= 0 && s <= N;
    if (valid) {
#pragma unroll
      for (int oy = 0; oy < 5; ++oy) {
        const int j = 2 * s - 2 + oy;
        vx[oy * 5 + 0] = S.R(j, 0, 0, t);
        vx[oy * 5 + 1] = S.R(j, 0, 1, t);
        vx[oy * 5 + 2] = S.R(j, 0, 0, t + 1);
        vx[oy * 5 + 3] = S.R(j, 0, 1, t + 1);
        vx[oy * 5 + 4] = S.R(j, 0, 0, t + 2);
        vy[oy * 5 + 0] = S.R(j, 1, 0, t);
        vy[oy * 5 + 1] = S.R(j, 1, 1, t);
        vy[oy * 5 + 2] = S.R(j, 1, 0, t + 1);
        vy[oy * 5 + 3] = S.R(j, 1, 1, t + 1);
        vy[oy * 5 + 4] = S.R(j, 1, 0, t + 2);
      }
      const double rp = S.RP(s, t + 1);
      if (kxp >= 2 && kxp <= N - 2 && s >= 2 && s <= N - 2) {
        dp = solve_generic(vx, vy, rp, F);
      } else {  // precomputed by k_boundary_patches
        const int64_t nb = bd_count(N), bi = bd_index(kxp, s, N);
#pragma unroll
        for (int q = 0; q < 25; ++q) {
          vx[q] = A.bd[q * nb + bi];
          vy[q] = A.bd[(25 + q) * nb + bi];
        }
        dp = A.bd[50 * nb + bi];
      }
      // pressure: only patch k holds p_k (multiplicity 1) -> output now
      if (t >= 1 && t <= fz::kNOUT && s >= y0 && s < y1) {
        const double xp = XZERO ? 0.0 : S.Pp(s, t + 2);
        A.xout[g.op + (int64_t)s * g.pp + kxp] = fma(A.omega, dp, xp);
      }
    } else if (t >= 1 && t <= fz::kNOUT && s >= y0 && s < y1 && kxp > N && kxp < g.pp) {
      A.xout[g.op + (int64_t)s * g.pp + kxp] = 0.0;  // pitch padding
    }
    // ---- accumulate sum_i V_i^T delta_i: three conflict-free phases ----
    if (valid) {
#pragma unroll
      for (int oy = 0; oy < 5; ++oy) {
        const int j = 2 * s - 2 + oy;
        S.Acc(j, 0, 0, t + 1) += vx[oy * 5 + 2];
        S.Acc(j, 0, 1, t + 1) += vx[oy * 5 + 3];
        S.Acc(j, 1, 0, t + 1) += vy[oy * 5 + 2];
        S.Acc(j, 1, 1, t + 1) += vy[oy * 5 + 3];
      }
    }
    __syncthreads();
    if (valid) {
#pragma unroll
      for (int oy = 0; oy < 5; ++oy) {
        const int j = 2 * s - 2 + oy;
        S.Acc(j, 0, 0, t) += vx[oy * 5 + 0];
        S.Acc(j, 0, 1, t) += vx[oy * 5 + 1];
        S.Acc(j, 1, 0, t) += vy[oy * 5 + 0];
        S.Acc(j, 1, 1, t) += vy[oy * 5 + 1];
      }
    }
    __syncthreads();
    if (valid) {
#pragma unroll
      for (int oy = 0; oy < 5; ++oy) {
        const int j = 2 * s - 2 + oy;
        S.Acc(j, 0, 0, t + 2) += vx[oy * 5 + 4];
        S.Acc(j, 1, 0, t + 2) += vy[oy * 5 + 4];
      }
    }
    __syncthreads();

    // ---- lattice rows 2s-2, 2s-1 (node row s-1) are complete ----
    const int ny = s - 1;
    if (t < fz::kNOUT) {
      const int kx = kx0 + t;
      const bool rowout = ny >= y0 && ny < y1 && 2 * kx < g.pu;
#pragma unroll
      for (int rr = 0; rr < 2; ++rr) {
        const int j = 2 * ny + rr;
#pragma unroll
        for (int comp = 0; comp < 2; ++comp) {
          const double a0 = S.Acc(j, comp, 0, t + 2), a1 = S.Acc(j, comp, 1, t + 2);
          S.Acc(j, comp, 0, t + 2) = 0.0;
          S.Acc(j, comp, 1, t + 2) = 0.0;
          if (!rowout || j > lat - 1) continue;
          const int i0 = 2 * kx;
          const double x0 = XZERO ? 0.0 : S.X(j, comp, 0, t + 3), x1 = XZERO ? 0.0 : S.X(j, comp, 1, t + 3);
          const bool jin = j >= 1 && j <= lat - 2;
          double o0, o1;
          if (A.scalar_w) {
            o0 = (jin && i0 >= 1 && i0 <= lat - 2) ? fma(A.omega, a0, x0) : (i0 <= lat - 1 ? x0 : 0.0);
            o1 = (jin && i0 + 1 <= lat - 2) ? fma(A.omega, a1, x1) : (i0 + 1 <= lat - 1 ? x1 : 0.0);
          } else {
            const double wy = (j & 1) ? 0.5 : (1.0 / 3.0);  // 1 / (patches per axis holding the point)
            o0 = (jin && i0 >= 1 && i0 <= lat - 2) ? fma(A.omega * wy * (1.0 / 3.0), a0, x0) : (i0 <= lat - 1 ? x0 : 0.0);
            o1 = (jin && i0 + 1 <= lat - 2) ? fma(A.omega * wy * 0.5, a1, x1) : (i0 + 1 <= lat - 1 ? x1 : 0.0);
          }
          *reinterpret_cast<double2*>(A.xout + (comp ? g.ouy : g.oux) + (int64_t)j * g.pu + i0) = make_double2(o0, o1);
        }
      }
    } else {  // ghost accumulator columns nobody outputs: keep them clean
      const int q = t - fz::kNOUT;  // 0..3 -> columns 0,1 and 126,127 of the ring
      const int col = q < 2 ? q : fz::kNPATCH + (q - 2);
#pragma unroll
      for (int rr = 0; rr < 2; ++rr)
#pragma unroll
        for (int comp = 0; comp < 2; ++comp) {
          S.Acc(2 * ny + rr, comp, 0, col) = 0.0;
          S.Acc(2 * ny + rr, comp, 1, col) = 0.0;
        }
    }
    if (!XZERO) cp_wait_all();
    __syncthreads();
  }
}

inline int launch_factor_setup(const int* d_Ns, int nlev, double nu, const double* /*d_inv*/, double* d_fac,
                               int* d_status) {
  k_factor_setup<<<nlev, 256>>>(d_Ns, nu, d_fac, d_status);
  return 0;
}

// chunk height: about `waves` full waves of 2 CTAs per SM over the strips
inline int fused_chunk(const LevelGeom& g, int nstrips, int nsm) {
  const int resident = 2 * nsm;
  const double work = (double)nstrips * (g.N + 1) / 128.0;
  int waves = (int)(work / resident + 0.5);
  if (waves < 1) waves = 1;
  int chunks = (resident * waves) / nstrips;
  if (chunks < 1) chunks = 1;
  if (chunks > g.N + 1) chunks = g.N + 1;
  return (g.N + 1 + chunks - 1) / chunks;
}

inline int launch_fused_sweep(const LevelGeom& g, double nu, double omega, int scalar_w, const FusedFactors& F,
                              const double* dinv, double* bd, const double* xin, const double* b, double* xout,
                              int nsm, cudaStream_t s) {
  k_boundary_patches<<<(unsigned)bd_count(g.N), 64, 0, s>>>(g, nu, dinv, xin, b, bd);
  static bool attr_done[64] = {false};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev >= 0 && dev < 64 && !attr_done[dev]) {
    cudaFuncSetAttribute(k_vanka_fused<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, fz::kSmemBytes);
    cudaFuncSetAttribute(k_vanka_fused<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, fz::kSmemBytes);
    attr_done[dev] = true;
  }
  const int ncover = (int)std::max<int64_t>(g.pu / 2, g.pp);
  const int nstrips = (ncover + fz::kNOUT - 1) / fz::kNOUT;
  FusedArgs A{g, omega, scalar_w, 0, bd, xin, b, xout};
  A.chunk = fused_chunk(g, nstrips, nsm);
  const dim3 grid(nstrips, (g.N + 1 + A.chunk - 1) / A.chunk);
  if (xin) k_vanka_fused<false><<<grid, fz::kNT, fz::kSmemBytes, s>>>(A, F);
  else k_vanka_fused<true><<<grid, fz::kNT, fz::kSmemBytes, s>>>(A, F);
  return 0;
}

}  // namespace svk
