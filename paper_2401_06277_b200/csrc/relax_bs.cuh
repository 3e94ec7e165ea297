// relax_bs.cuh -- the paper's same-run comparator relaxations:
// inexact Braess-Sarazin (alg:bs) and Schur-Uzawa (alg:uz).
//
// With r = b - A x (masked), D = diag(L) on the non-Dirichlet velocity DOFs and
// S = -(1/t) B D^{-1} B^T:
//   Braess-Sarazin:  S dp ~= r_p - (1/t) B D^{-1} r_u        (eq:bseq1, nj Jacobi sweeps)
//                    du   = (1/t) D^{-1} (r_u - B^T dp)      (eq:bseq2)
//                    x   += omega_BS (du, dp)
//   Schur-Uzawa:     du   = (1/t) D^{-1} r_u
//                    S dp ~= r_p - B du                       (eq:uzblock; DESIGN reading 19)
//                    x   += (du, dp)
// Both right-hand sides are the same vector r_p - (1/t) B D^{-1} r_u.
//
// Structure instead of matrices: D^{-1} is one constant per lattice
// parity class; B / B^T rows come from the stencil tables; S is a 5x5 pressure
// stencil whose coefficients depend only on the per-axis distance class of the
// node to the boundary (0, 1, 2, interior, N-2, N-1, N -> 7 x 7 classes), built
// once per level on the host from the exact 1D element matrices.
// Kernels: residual (k_residual_strip) -> k_bs_rhs -> nj x k_schur_jacobi ->
// k_bs_update2.  Plane kernels; the comparators are not the hot path.
#pragma once
#include "kernels_common.cuh"

namespace svk {

constexpr int kSchurCls = 7;                             // classes per axis
constexpr int kSchurStride = kSchurCls * kSchurCls * 25;  // doubles per level

struct BsArgs {
  LevelGeom g;
  double inv_t;        // 1/t
  double omega_r;      // omega_BS (Braess-Sarazin) or 1 (Schur-Uzawa)
  double dinv[2][2];   // 1 / L_jj by lattice parity [j & 1][i & 1]
  int su;              // 1: Schur-Uzawa (no B^T dp term in du)
};

__host__ __device__ __forceinline__ int schur_cls(int k, int N) {
  if (N < 6) return k;  // tiny level: every node is its own class (N + 1 <= 7)
  return k <= 2 ? k : (k >= N - 2 ? 6 - (N - k) : 3);
}

// rhs_k = r_p,k - (1/t) sum_j B_kj D^{-1}_j r_u,j   (pressure nodes; pitch pp, rows N+1)
__global__ void k_bs_rhs(const BsArgs a, const double* __restrict__ r, double* __restrict__ rhs) {
  const LevelGeom& g = a.g;
  const int kx = blockIdx.x * blockDim.x + threadIdx.x, ky = blockIdx.y * blockDim.y + threadIdx.y;
  const int N = g.N, lat = g.lat;
  if (ky > N || kx >= g.pp) return;
  if (kx > N) {
    rhs[(int64_t)ky * g.pp + kx] = 0.0;
    return;
  }
  const int cx = kx == 0 ? 0 : (kx == N ? 2 : 1), cy = ky == 0 ? 0 : (ky == N ? 2 : 1);
  double s = 0.0;
  for (int oy = 0; oy < 5; ++oy) {
    const int j = 2 * ky - 2 + oy;
    if (j < 1 || j > lat - 2) continue;  // Dirichlet rows: D^{-1} := 0
    const double cyc = c_st.CR[cy][oy], gyc = c_st.GR[cy][oy];
    const double* rx = r + g.oux + (int64_t)j * g.pu;
    const double* ry = r + g.ouy + (int64_t)j * g.pu;
    for (int ox = 0; ox < 5; ++ox) {
      const int i = 2 * kx - 2 + ox;
      if (i < 1 || i > lat - 2) continue;
      const double di = a.dinv[j & 1][i & 1];
      s += di * (cyc * c_st.GR[cx][ox] * rx[i] + gyc * c_st.CR[cx][ox] * ry[i]);
    }
  }
  // B = -h (C^ (x) G, G (x) C^)
  rhs[(int64_t)ky * g.pp + kx] = r[p_at(g, kx, ky)] + a.inv_t * g.h * s;
}

// one weighted-Jacobi sweep on S dp = rhs: dp_out = dp_in + omega (rhs - S dp_in) / S_kk
// (dp_in == nullptr: dp_in = 0).  st: this level's class stencils [cy][cx][5x5].
__global__ void k_schur_jacobi(LevelGeom g, const double* __restrict__ st, double omega, const double* __restrict__ rhs,
                               const double* __restrict__ dp_in, double* __restrict__ dp_out) {
  const int kx = blockIdx.x * blockDim.x + threadIdx.x, ky = blockIdx.y * blockDim.y + threadIdx.y;
  const int N = g.N;
  if (ky > N || kx >= g.pp) return;
  const int64_t o = (int64_t)ky * g.pp + kx;
  if (kx > N) {
    dp_out[o] = 0.0;
    return;
  }
  const double* c = st + (schur_cls(ky, N) * kSchurCls + schur_cls(kx, N)) * 25;
  double sdp = 0.0, d0 = 0.0;
  if (dp_in) {
    d0 = dp_in[o];
    for (int dy = -2; dy <= 2; ++dy) {
      const int m = ky + dy;
      if (m < 0 || m > N) continue;
      for (int dx = -2; dx <= 2; ++dx) {
        const int n = kx + dx;
        if (n < 0 || n > N) continue;
        sdp = fma(c[(dy + 2) * 5 + dx + 2], dp_in[(int64_t)m * g.pp + n], sdp);
      }
    }
  }
  dp_out[o] = d0 + omega * (rhs[o] - sdp) / c[12];
}

// x_out = x_in + omega_r (du, dp),  du = (1/t) D^{-1} (r_u - [B^T dp]) on non-Dirichlet DOFs
// Two lattice columns (even, odd) per thread and one row per warp, so the B^T
// stencil shape (parity) is warp-uniform: no divergence between neighbouring
// threads and unrolled pressure taps.  z = 0, 1: velocity planes;
// z = 2: the pressure plane (nodes 2p, 2p+1 of row j).  grid: (pairs / 32, rows / 8, 3).
__global__ void __launch_bounds__(256) k_bs_update2(const BsArgs a, const double* __restrict__ xin,
                                                    const double* __restrict__ r, const double* __restrict__ dp,
                                                    double* __restrict__ xout) {
  const LevelGeom& g = a.g;
  const int plane = blockIdx.z;
  const int pr = blockIdx.x * blockDim.x + threadIdx.x;  // column pair
  const int j = blockIdx.y * blockDim.y + threadIdx.y;
  const int N = g.N, lat = g.lat;
  if (plane == 2) {
    if (j > N) return;
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const int i = 2 * pr + e;
      if (i >= g.pp) continue;
      const int64_t o = p_at(g, i, j);
      xout[o] = i > N ? 0.0 : fma(a.omega_r, dp[(int64_t)j * g.pp + i], xin[o]);
    }
    return;
  }
  const int i0 = 2 * pr;
  if (j >= lat || i0 >= g.pu) return;
  const int64_t o = (plane ? g.ouy : g.oux) + (int64_t)j * g.pu + i0;
  const int pj = j & 1;
  // pressure window: node rows ky0 .. ky0 + 2 (row parity odd: 2 rows), columns pr-1 .. pr+1
  const int ky0 = pj ? (j - 1) >> 1 : (j >> 1) - 1;
  double P[3][3];
#pragma unroll
  for (int ty = 0; ty < 3; ++ty)
#pragma unroll
    for (int tx = 0; tx < 3; ++tx) {
      const int ky = ky0 + ty, kx = pr - 1 + tx;
      const bool ok = !a.su && ky >= 0 && ky <= N && kx >= 0 && kx <= N && (ty < 2 || !pj);
      P[ty][tx] = ok ? dp[(int64_t)ky * g.pp + kx] : 0.0;
    }
  double res[2];
#pragma unroll
  for (int e = 0; e < 2; ++e) {  // e = column parity of point i0 + e
    const int i = i0 + e;
    double bt = 0.0;
#pragma unroll
    for (int ty = 0; ty < 3; ++ty) {
      if (pj && ty == 2) continue;
      const double cy = plane == 0 ? c_st.CC[pj][ty] : c_st.GC[pj][ty];
      double tsum = 0.0;
#pragma unroll
      for (int tx = 0; tx < 3 - e; ++tx)  // even point: nodes pr-1 .. pr+1; odd: pr .. pr+1
        tsum += (plane == 0 ? c_st.GC[e][tx] : c_st.CC[e][tx]) * P[ty][tx + e];
      bt += cy * tsum;
    }
    bt *= -g.h;
    if (i >= lat) res[e] = 0.0;
    else if (i == 0 || j == 0 || i == lat - 1 || j == lat - 1) res[e] = xin[o + e];
    else res[e] = fma(a.omega_r * a.inv_t * (pj ? a.dinv[1][e] : a.dinv[0][e]), r[o + e] - bt, xin[o + e]);
  }
  if (i0 + 1 < g.pu) *reinterpret_cast<double2*>(xout + o) = make_double2(res[0], res[1]);
  else xout[o] = res[0];
}

// ---- host: S class stencils of one level --------------------------------------
// 1D assembled entries from the element tables (host twins of k1/m1/c1/g1 in
// stencil.cuh): h K, M / h, C / h, G.
inline double h_k1(const StencilConst& t, int i, int ip, int N) {
  double s = 0.0;
  for (int e = std::max(0, (std::max(i, ip) - 1) / 2); e <= std::min(N - 1, std::min(i, ip) / 2); ++e) {
    const int a = i - 2 * e, b = ip - 2 * e;
    if (a >= 0 && a <= 2 && b >= 0 && b <= 2) s += t.Khat[a][b];
  }
  return s;
}
inline double h_m1(const StencilConst& t, int i, int ip, int N) {
  double s = 0.0;
  for (int e = std::max(0, (std::max(i, ip) - 1) / 2); e <= std::min(N - 1, std::min(i, ip) / 2); ++e) {
    const int a = i - 2 * e, b = ip - 2 * e;
    if (a >= 0 && a <= 2 && b >= 0 && b <= 2) s += t.Mhat[a][b];
  }
  return s;
}
inline double h_c1(const StencilConst& t, int k, int i, int N) {
  double s = 0.0;
  for (int e = k - 1; e <= k; ++e) {
    if (e < 0 || e >= N) continue;
    const int c = k - e, a = i - 2 * e;
    if (a >= 0 && a <= 2) s += t.Chat[c][a];
  }
  return s;
}
inline double h_g1(const StencilConst& t, int k, int i, int N) {
  double s = 0.0;
  for (int e = k - 1; e <= k; ++e) {
    if (e < 0 || e >= N) continue;
    const int c = k - e, a = i - 2 * e;
    if (a >= 0 && a <= 2) s += t.Ge[c][a];
  }
  return s;
}

// S_{k, k+d} = -(1/t) sum_j B_kj D^{-1}_j B_{k+d, j} for a representative node of every
// (cy, cx) class; out[(cy*7 + cx)*25 + (dy+2)*5 + dx+2].
inline void build_schur_stencils(const StencilConst& t, int N, double nu, double tt, double* out) {
  const int lat = 2 * N + 1;
  const double h = 1.0 / N;
  auto rep = [&](int c) { return N < 6 ? c : (c <= 3 ? c : N - (6 - c)); };
  const int ncls = N < 6 ? N + 1 : kSchurCls;
  std::fill(out, out + kSchurStride, 0.0);
  for (int cy = 0; cy < ncls; ++cy)
    for (int cx = 0; cx < ncls; ++cx) {
      const int ky = rep(cy), kx = rep(cx);
      for (int dy = -2; dy <= 2; ++dy)
        for (int dx = -2; dx <= 2; ++dx) {
          const int my = ky + dy, mx = kx + dx;
          if (my < 0 || my > N || mx < 0 || mx > N) continue;
          double s = 0.0;
          for (int jy = std::max(1, 2 * ky - 2); jy <= std::min(lat - 2, 2 * ky + 2); ++jy)
            for (int jx = std::max(1, 2 * kx - 2); jx <= std::min(lat - 2, 2 * kx + 2); ++jx) {
              const double d = nu * (h_m1(t, jy, jy, N) * h_k1(t, jx, jx, N) + h_k1(t, jy, jy, N) * h_m1(t, jx, jx, N));
              const double bxk = -h * h_c1(t, ky, jy, N) * h_g1(t, kx, jx, N);
              const double bxm = -h * h_c1(t, my, jy, N) * h_g1(t, mx, jx, N);
              const double byk = -h * h_g1(t, ky, jy, N) * h_c1(t, kx, jx, N);
              const double bym = -h * h_g1(t, my, jy, N) * h_c1(t, mx, jx, N);
              s += (bxk * bxm + byk * bym) / d;
            }
          out[(cy * kSchurCls + cx) * 25 + (dy + 2) * 5 + dx + 2] = -s / tt;
        }
    }
}

}  // namespace svk
