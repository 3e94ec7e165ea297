// bt.cuh -- the block-triangular preconditioner of the paper's comparison
// (alg:bt):
//   [[L, B^T], [0, -M]] (du, dp) = r,   M = Q1 pressure mass matrix (Shat ~ -M)
//   1. M dp = -r_p   by bt_cycles V(bt_nu, bt_nu) cycles, weighted Jacobi (omega_p)
//   2. L du = r_u - B^T dp   likewise (both components at once, omega_u)
// (3 V(3,3) cycles per block, weights 0.6 / 1.0).  The block multigrid
// reuses the level hierarchy, the Q2 / Q1 transfer kernels and the stencil tables;
// "part" 0 = the velocity planes (interior system, corrections vanish on the
// Dirichlet lattice points), part 1 = the pressure plane.  Level 0 is solved
// exactly with dense inverses built on the host (interior L, 2 x 49 unknowns at
// N0 = 4; M, 25 unknowns).  Plane kernels: HBM-bound comparator code.
#pragma once
#include "relax_bs.cuh"

namespace svk {

struct BtArgs {
  LevelGeom g;
  double nu;
  double omega;       // Jacobi weight of this part
  double dinv[2][2];  // velocity: 1 / L_jj by lattice parity
  int part;           // 0 velocity planes, 1 pressure plane
};

// 1D Q1 mass row of node k (h/6 * (1, 4, 1); boundary diagonal 2): entry (k, k+d)
__device__ __forceinline__ double q1m(int k, int d, int N, double h) {
  if (k + d < 0 || k + d > N) return 0.0;
  if (d != 0) return h / 6.0;
  return (k == 0 || k == N ? 2.0 : 4.0) * h / 6.0;
}
__device__ __forceinline__ double mass_at(const double* __restrict__ p, int64_t pp, int N, double h, int kx, int ky,
                                          double* diag) {
  double s = 0.0;
  for (int dy = -1; dy <= 1; ++dy) {
    const double my = q1m(ky, dy, N, h);
    if (my == 0.0) continue;
    for (int dx = -1; dx <= 1; ++dx) {
      const double mx = q1m(kx, dx, N, h);
      if (mx == 0.0) continue;
      s += my * mx * p[(int64_t)(ky + dy) * pp + kx + dx];
    }
  }
  *diag = q1m(ky, 0, N, h) * q1m(kx, 0, N, h);
  return s;
}

// JAC = 1: out = x + omega D^{-1} (b - A x);  JAC = 0: out = b - A x  (part planes only;
// velocity Dirichlet points and padding -> 0).  grid: z = planes of the part.
template <int JAC>
__global__ void k_bt_smooth(const BtArgs a, const double* __restrict__ x, const double* __restrict__ b,
                            double* __restrict__ out) {
  const LevelGeom& g = a.g;
  const int i = blockIdx.x * blockDim.x + threadIdx.x, j = blockIdx.y * blockDim.y + threadIdx.y;
  const int N = g.N, lat = g.lat;
  if (a.part == 0) {
    const int comp = blockIdx.z;
    if (j >= lat || i >= g.pu) return;
    const int64_t o = (comp ? g.ouy : g.oux) + (int64_t)j * g.pu + i;
    if (i == 0 || j == 0 || i >= lat - 1 || j == lat - 1) {
      out[o] = 0.0;
      return;
    }
    const double r = b[o] - a.nu * lap_at(x + (comp ? g.ouy : g.oux), g.pu, i, j);
    out[o] = JAC ? fma(a.omega * a.dinv[j & 1][i & 1], r, x[o]) : r;
  } else {
    if (j > N || i >= g.pp) return;
    const int64_t o = p_at(g, i, j);
    if (i > N) {
      out[o] = 0.0;
      return;
    }
    double d;
    const double r = b[o] - mass_at(x + g.op, g.pp, N, g.h, i, j, &d);
    out[o] = JAC ? fma(a.omega / d, r, x[o]) : r;
  }
}

// Velocity part, two lattice columns (one even, one odd) per thread so the
// parity -- hence the stencil, taken from the level's L2D table (the fused
// sweep's, nu (M (x) K + K (x) M) by parity class) -- is warp-uniform and the
// 5 x 5 loops unroll: JAC = 1: out = x + omega D^{-1} (b - L x), JAC = 0:
// out = b - L x; Dirichlet points and padding -> 0.  grid: (pairs / 32, rows / 8, 2).
struct L2DTab {
  double c[2][2][5][5];
};
template <int JAC>
__global__ void __launch_bounds__(256) k_bt_smooth_vel(const BtArgs a, const L2DTab T, const double* __restrict__ x,
                                                       const double* __restrict__ b, double* __restrict__ out) {
  const LevelGeom& g = a.g;
  const int lat = g.lat;
  const int i0 = 2 * (blockIdx.x * blockDim.x + threadIdx.x), j = blockIdx.y * blockDim.y + threadIdx.y;
  const int comp = blockIdx.z;
  if (j >= lat || i0 >= g.pu) return;
  const double* u = x + (comp ? g.ouy : g.oux);
  const int64_t o = (comp ? g.ouy : g.oux) + (int64_t)j * g.pu + i0;
  double w[5][6];  // rows j-2 .. j+2, columns i0-2 .. i0+3 (0 outside the plane)
#pragma unroll
  for (int bb = 0; bb < 5; ++bb) {
    const int jj = j - 2 + bb;
    const bool rok = jj >= 0 && jj < lat;
#pragma unroll
    for (int aa = 0; aa < 6; ++aa) {
      const int ii = i0 - 2 + aa;
      w[bb][aa] = (rok && ii >= 0 && ii < lat) ? u[(int64_t)jj * g.pu + ii] : 0.0;
    }
  }
  const int pj = j & 1;
  double r[2];
#pragma unroll
  for (int e = 0; e < 2; ++e) {  // e = column parity of point i0 + e (row parity: warp-uniform branch)
    double s = 0.0;
    if (pj) {
#pragma unroll
      for (int bb = 0; bb < 5; ++bb)
#pragma unroll
        for (int aa = 0; aa < 5; ++aa) s = fma(T.c[1][e][bb][aa], w[bb][aa + e], s);
    } else {
#pragma unroll
      for (int bb = 0; bb < 5; ++bb)
#pragma unroll
        for (int aa = 0; aa < 5; ++aa) s = fma(T.c[0][e][bb][aa], w[bb][aa + e], s);
    }
    r[e] = s;
  }
  const bool jin = j >= 1 && j <= lat - 2;
  double res[2];
#pragma unroll
  for (int e = 0; e < 2; ++e) {
    const int i = i0 + e;
    const bool in = jin && i >= 1 && i <= lat - 2;
    const double rv = in ? b[o + e] - r[e] : 0.0;
    res[e] = JAC ? (in ? fma(a.omega * (pj ? a.dinv[1][e] : a.dinv[0][e]), rv, x[o + e]) : 0.0) : rv;
  }
  if (i0 + 1 < g.pu) *reinterpret_cast<double2*>(out + o) = make_double2(res[0], res[1]);
  else out[o] = res[0];
}

// BT right-hand sides on the finest level: MODE 0: out = (0, 0, -r_p);
// MODE 1: out_u = r_u - B^T dp (dp = the pressure plane of x), out_p = 0.
template <int MODE>
__global__ void k_bt_rhs(LevelGeom g, const double* __restrict__ r, const double* __restrict__ x,
                         double* __restrict__ out) {
  const int plane = blockIdx.z;
  const int i = blockIdx.x * blockDim.x + threadIdx.x, j = blockIdx.y * blockDim.y + threadIdx.y;
  const int N = g.N, lat = g.lat;
  if (plane < 2) {
    if (j >= lat || i >= g.pu) return;
    const int64_t o = (plane ? g.ouy : g.oux) + (int64_t)j * g.pu + i;
    if (MODE == 0 || i == 0 || j == 0 || i >= lat - 1 || j == lat - 1) {
      out[o] = 0.0;
      return;
    }
    out[o] = r[o] - gradp_at(x + g.op, g.pp, i, j, plane, g.h);
  } else {
    if (j > N || i >= g.pp) return;
    const int64_t o = p_at(g, i, j);
    out[o] = (MODE == 0 && i <= N) ? -r[o] : 0.0;
  }
}

// ---- host: level-0 dense inverses (stride ni + 1, the k_coarse_apply layout) ----------
inline bool host_gj_invert(std::vector<double>& a, int n) {
  std::vector<int> piv(n);
  for (int i = 0; i < n; ++i) piv[i] = i;
  std::vector<double> inv((size_t)n * n, 0.0);
  for (int i = 0; i < n; ++i) inv[(size_t)i * n + i] = 1.0;
  for (int c = 0; c < n; ++c) {
    int p = c;
    for (int r = c + 1; r < n; ++r)
      if (std::fabs(a[(size_t)r * n + c]) > std::fabs(a[(size_t)p * n + c])) p = r;
    if (a[(size_t)p * n + c] == 0.0) return false;
    for (int k = 0; k < n; ++k) {
      std::swap(a[(size_t)p * n + k], a[(size_t)c * n + k]);
      std::swap(inv[(size_t)p * n + k], inv[(size_t)c * n + k]);
    }
    const double d = 1.0 / a[(size_t)c * n + c];
    for (int k = 0; k < n; ++k) {
      a[(size_t)c * n + k] *= d;
      inv[(size_t)c * n + k] *= d;
    }
    for (int r = 0; r < n; ++r) {
      if (r == c) continue;
      const double f = a[(size_t)r * n + c];
      if (f == 0.0) continue;
      for (int k = 0; k < n; ++k) {
        a[(size_t)r * n + k] -= f * a[(size_t)c * n + k];
        inv[(size_t)r * n + k] -= f * inv[(size_t)c * n + k];
      }
    }
  }
  a.swap(inv);
  return true;
}
// interior L on level 0 (both components, block diagonal) and M; idx = vector offsets
inline bool build_bt_coarse(const StencilConst& t, const LevelGeom& g, double nu, std::vector<double>& invL,
                            std::vector<int>& idxL, std::vector<double>& invM, std::vector<int>& idxM) {
  const int N = g.N, lat = g.lat;
  std::vector<std::pair<int, int>> pts;
  for (int j = 1; j < lat - 1; ++j)
    for (int i = 1; i < lat - 1; ++i) pts.push_back({i, j});
  const int m = (int)pts.size(), ni = 2 * m;
  std::vector<double> a((size_t)ni * ni, 0.0);
  for (int r = 0; r < m; ++r)
    for (int c = 0; c < m; ++c) {
      const int i = pts[r].first, j = pts[r].second, ip = pts[c].first, jp = pts[c].second;
      const double v = nu * (h_m1(t, j, jp, N) * h_k1(t, i, ip, N) + h_k1(t, j, jp, N) * h_m1(t, i, ip, N));
      a[(size_t)r * ni + c] = v;
      a[(size_t)(m + r) * ni + m + c] = v;
    }
  if (!host_gj_invert(a, ni)) return false;
  invL.assign((size_t)(ni + 1) * (ni + 1), 0.0);
  for (int r = 0; r < ni; ++r)
    for (int c = 0; c < ni; ++c) invL[(size_t)r * (ni + 1) + c] = a[(size_t)r * ni + c];
  idxL.clear();
  for (int comp = 0; comp < 2; ++comp)
    for (auto& q : pts) idxL.push_back((int)((comp ? g.ouy : g.oux) + (int64_t)q.second * g.pu + q.first));
  // Q1 mass: (h/6)^2 (1D rows 1, 4, 1; boundary diagonal 2)
  const int np = (N + 1) * (N + 1);
  auto m1 = [&](int k, int kp) {
    if (std::abs(k - kp) > 1) return 0.0;
    if (k != kp) return 1.0 / (6.0 * N);
    return (k == 0 || k == N ? 2.0 : 4.0) / (6.0 * N);
  };
  std::vector<double> b((size_t)np * np, 0.0);
  for (int r = 0; r < np; ++r)
    for (int c = 0; c < np; ++c) b[(size_t)r * np + c] = m1(r / (N + 1), c / (N + 1)) * m1(r % (N + 1), c % (N + 1));
  if (!host_gj_invert(b, np)) return false;
  invM.assign((size_t)(np + 1) * (np + 1), 0.0);
  for (int r = 0; r < np; ++r)
    for (int c = 0; c < np; ++c) invM[(size_t)r * (np + 1) + c] = b[(size_t)r * np + c];
  idxM.clear();
  for (int ky = 0; ky <= N; ++ky)
    for (int kx = 0; kx <= N; ++kx) idxM.push_back((int)p_at(g, kx, ky));
  return true;
}

}  // namespace svk
