// kernels_common.cuh -- residual / matvec, problem data, transfers, patch setup,
// level-0 solve and the unfused (paper-split) Vanka sweep of libsvk.
// Single translation unit: included from svk.cu after stencil.cuh.
#pragma once
#include "stencil.cuh"

namespace svk {

// Programmatic dependent launch: the V-cycle kernels are launched with
// programmaticStreamSerialization, so a kernel's CTAs are scheduled (and run their
// dependency-free prologue) while the previous kernel drains; every such kernel
// calls pdl_wait() before touching memory the previous kernel writes.  No kernel
// triggers early, so the wait returns only when the previous grid has completed
// and its writes are visible.  SVK_PDL=0 launches them plainly (wait is a no-op).
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;\n" ::: "memory"); }
inline bool pdl_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("SVK_PDL");
    return !(e && e[0] == '0');
  }();
  return on;
}
template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*k)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s, Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, k, std::forward<Args>(args)...);
}

constexpr int kSlots = 51;             // padded patch slots: 2 x 5x5 velocity window + 1 pressure
constexpr int kGroupStride = kSlots * kSlots;

__host__ __device__ __forceinline__ int64_t ux_at(const LevelGeom& g, int i, int j) { return g.oux + (int64_t)j * g.pu + i; }
__host__ __device__ __forceinline__ int64_t uy_at(const LevelGeom& g, int i, int j) { return g.ouy + (int64_t)j * g.pu + i; }
__host__ __device__ __forceinline__ int64_t p_at(const LevelGeom& g, int kx, int ky) { return g.op + (int64_t)ky * g.pp + kx; }

// ---------------------------------------------------------------------------
// (L u)(i,j) for one velocity component at a NON-Dirichlet lattice point,
// from the 1D rows KR/MR: L = nu (M (x) K + K (x) M).
// ---------------------------------------------------------------------------
__device__ __forceinline__ double lap_at(const double* __restrict__ u, int64_t pu, int i, int j) {
  const int pi = i & 1, pj = j & 1;
  const int ra = pi ? 1 : 2, rb = pj ? 1 : 2;
  double s = 0.0;
  for (int bb = -rb; bb <= rb; ++bb) {
    const double my = c_st.MR[pj][bb + 2], ky = c_st.KR[pj][bb + 2];
    const double* row = u + (int64_t)(j + bb) * pu + i;
    for (int aa = -ra; aa <= ra; ++aa) s += (my * c_st.KR[pi][aa + 2] + ky * c_st.MR[pi][aa + 2]) * row[aa];
  }
  return s;
}

// (B^T p) at a non-Dirichlet lattice point for component comp (0: x, 1: y)
__device__ __forceinline__ double gradp_at(const double* __restrict__ p, int64_t pp, int i, int j, int comp, double h) {
  const int pi = i & 1, pj = j & 1;
  const int ky0 = pj ? (j - 1) >> 1 : (j >> 1) - 1, nky = pj ? 2 : 3;
  const int kx0 = pi ? (i - 1) >> 1 : (i >> 1) - 1, nkx = pi ? 2 : 3;
  double s = 0.0;
  for (int ty = 0; ty < nky; ++ty) {
    const double cy = comp == 0 ? c_st.CC[pj][ty] : c_st.GC[pj][ty];
    if (cy == 0.0) continue;
    const double* row = p + (int64_t)(ky0 + ty) * pp + kx0;
    double t = 0.0;
    for (int tx = 0; tx < nkx; ++tx) t += (comp == 0 ? c_st.GC[pi][tx] : c_st.CC[pi][tx]) * row[tx];
    s += cy * t;
  }
  return -h * s;
}

// (B u) at pressure node (kx,ky)
__device__ __forceinline__ double div_at(const double* __restrict__ ux, const double* __restrict__ uy, int64_t pu, int N,
                                         int kx, int ky, double h) {
  const int cx = kx == 0 ? 0 : (kx == N ? 2 : 1), cy = ky == 0 ? 0 : (ky == N ? 2 : 1);
  const int lat = 2 * N + 1;
  double s = 0.0;
  for (int oy = 0; oy < 5; ++oy) {
    const int j = 2 * ky - 2 + oy;
    if (j < 0 || j >= lat) continue;
    const double cyc = c_st.CR[cy][oy], gyc = c_st.GR[cy][oy];
    const double* rx = ux + (int64_t)j * pu;
    const double* ry = uy + (int64_t)j * pu;
    for (int ox = 0; ox < 5; ++ox) {
      const int i = 2 * kx - 2 + ox;
      if (i < 0 || i >= lat) continue;
      s += cyc * c_st.GR[cx][ox] * rx[i] + gyc * c_st.CR[cx][ox] * ry[i];
    }
  }
  return -h * s;
}

// The same three stencils with the vector read through an accessor u(i, j) /
// p(kx, ky) / u(comp, i, j) (same loops and summation order as lap_at / gradp_at /
// div_at): the boundary-patch kernel evaluates them on a band staged in shared memory.
template <class U>
__device__ __forceinline__ double lap_f(const U& u, int i, int j) {
  const int pi = i & 1, pj = j & 1;
  const int ra = pi ? 1 : 2, rb = pj ? 1 : 2;
  double s = 0.0;
  for (int bb = -rb; bb <= rb; ++bb) {
    const double my = c_st.MR[pj][bb + 2], ky = c_st.KR[pj][bb + 2];
    for (int aa = -ra; aa <= ra; ++aa) s += (my * c_st.KR[pi][aa + 2] + ky * c_st.MR[pi][aa + 2]) * u(i + aa, j + bb);
  }
  return s;
}
template <class P>
__device__ __forceinline__ double gradp_f(const P& p, int i, int j, int comp, double h) {
  const int pi = i & 1, pj = j & 1;
  const int ky0 = pj ? (j - 1) >> 1 : (j >> 1) - 1, nky = pj ? 2 : 3;
  const int kx0 = pi ? (i - 1) >> 1 : (i >> 1) - 1, nkx = pi ? 2 : 3;
  double s = 0.0;
  for (int ty = 0; ty < nky; ++ty) {
    const double cy = comp == 0 ? c_st.CC[pj][ty] : c_st.GC[pj][ty];
    if (cy == 0.0) continue;
    double t = 0.0;
    for (int tx = 0; tx < nkx; ++tx) t += (comp == 0 ? c_st.GC[pi][tx] : c_st.CC[pi][tx]) * p(kx0 + tx, ky0 + ty);
    s += cy * t;
  }
  return -h * s;
}
template <class U>
__device__ __forceinline__ double div_f(const U& u, int N, int kx, int ky, double h) {
  const int cx = kx == 0 ? 0 : (kx == N ? 2 : 1), cy = ky == 0 ? 0 : (ky == N ? 2 : 1);
  const int lat = 2 * N + 1;
  double s = 0.0;
  for (int oy = 0; oy < 5; ++oy) {
    const int j = 2 * ky - 2 + oy;
    if (j < 0 || j >= lat) continue;
    const double cyc = c_st.CR[cy][oy], gyc = c_st.GR[cy][oy];
    for (int ox = 0; ox < 5; ++ox) {
      const int i = 2 * kx - 2 + ox;
      if (i < 0 || i >= lat) continue;
      s += cyc * c_st.GR[cx][ox] * u(0, i, j) + gyc * c_st.CR[cx][ox] * u(1, i, j);
    }
  }
  return -h * s;
}

// r = b - A x (WITH_B) or r = A x, masked to 0 on Dirichlet rows; padding -> 0.
// grid: x over columns (pitch), y over rows, z = plane (0 ux, 1 uy, 2 p)
template <bool WITH_B>
__global__ void k_residual(LevelGeom g, double nu, const double* __restrict__ x, const double* __restrict__ b,
                           double* __restrict__ r) {
  const int plane = blockIdx.z;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const int j = blockIdx.y * blockDim.y + threadIdx.y;
  const int N = g.N, lat = g.lat;
  if (plane < 2) {
    if (j >= lat || i >= g.pu) return;
    const int64_t base = plane ? g.ouy : g.oux;
    const int64_t o = base + (int64_t)j * g.pu + i;
    if (i >= lat || i == 0 || j == 0 || i == lat - 1 || j == lat - 1) { r[o] = 0.0; return; }
    double ax = nu * lap_at(x + base, g.pu, i, j) + gradp_at(x + g.op, g.pp, i, j, plane, g.h);
    r[o] = WITH_B ? b[o] - ax : ax;
  } else {
    if (j > N || i >= g.pp) return;
    const int64_t o = g.op + (int64_t)j * g.pp + i;
    if (i > N) { r[o] = 0.0; return; }
    double ax = div_at(x + g.oux, x + g.ouy, g.pu, N, i, j, g.h);
    r[o] = WITH_B ? b[o] - ax : ax;
  }
}

// ---------------------------------------------------------------------------
// problem data: b = (f, psi) by 3x3 Gauss per element, x0 = boundary values
// ---------------------------------------------------------------------------
__device__ __forceinline__ void mms_u(int kind, double x, double y, double& ux, double& uy) {
  if (kind == 1) {
    ux = x * (1.0 - x) * (2.0 * x - 1.0) * (6.0 * y * y - 6.0 * y + 1.0);
    uy = y * (y - 1.0) * (2.0 * y - 1.0) * (6.0 * x * x - 6.0 * x + 1.0);
  } else if (kind == 2) {
    ux = 2.0 * x * x * y;
    uy = -2.0 * x * y * y;
  } else {
    ux = 0.0;
    uy = 0.0;
  }
}
// f = -nu Lap u + grad p (eq:stokes1)
__device__ __forceinline__ void mms_f(int kind, double nu, double x, double y, double& fx, double& fy) {
  if (kind == 1) {
    // with g(t) = t(1-t)(2t-1): u_x = -g(x) g'(y), u_y = g(y) g'(x), g''' = -12
    const double gx = x * (1.0 - x) * (2.0 * x - 1.0), gy = y * (1.0 - y) * (2.0 * y - 1.0);
    const double g1x = -6.0 * x * x + 6.0 * x - 1.0, g1y = -6.0 * y * y + 6.0 * y - 1.0;
    const double g2x = -12.0 * x + 6.0, g2y = -12.0 * y + 6.0;
    const double lap_ux = -(g2x * g1y + gx * -12.0);
    const double lap_uy = gy * -12.0 + g2y * g1x;
    fx = -nu * lap_ux + (2.0 * x + 8.0 / 3.0 * y);
    fy = -nu * lap_uy + (-6.0 * y + 8.0 / 3.0 * x);
  } else if (kind == 2) {
    fx = -nu * 4.0 * y + y;
    fy = nu * 4.0 * x + x;
  } else {
    fx = 0.0;
    fy = 0.0;
  }
}
__device__ __forceinline__ double lagr2(int a, double t) {
  return a == 0 ? 2.0 * (t - 0.5) * (t - 1.0) : a == 1 ? -4.0 * t * (t - 1.0) : 2.0 * t * (t - 0.5);
}

__global__ void k_set_problem(LevelGeom g, int kind, double nu, double* __restrict__ b, double* __restrict__ x0) {
  const int plane = blockIdx.z;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const int j = blockIdx.y * blockDim.y + threadIdx.y;
  const int N = g.N, lat = g.lat;
  if (plane == 2) {
    if (j > N || i >= g.pp) return;
    const int64_t o = p_at(g, i, j);
    if (b) b[o] = 0.0;
    if (x0) x0[o] = 0.0;
    return;
  }
  if (j >= lat || i >= g.pu) return;
  const int64_t o = (plane ? g.ouy : g.oux) + (int64_t)j * g.pu + i;
  if (i >= lat) {
    if (b) b[o] = 0.0;
    if (x0) x0[o] = 0.0;
    return;
  }
  const bool dir = i == 0 || j == 0 || i == lat - 1 || j == lat - 1;
  if (dir) {
    double ux, uy;
    if (kind == 3) {
      ux = (j == lat - 1 && i > 0 && i < lat - 1) ? 1.0 : 0.0;
      uy = 0.0;
    } else {
      mms_u(kind, 0.5 * i * g.h, 0.5 * j * g.h, ux, uy);
    }
    const double v = plane ? uy : ux;
    if (b) b[o] = v;
    if (x0) x0[o] = v;
    return;
  }
  if (x0) x0[o] = 0.0;
  if (!b) return;
  const double gp[3] = {0.5 - 0.5 * sqrt(0.6), 0.5, 0.5 + 0.5 * sqrt(0.6)};
  const double gw[3] = {5.0 / 18.0, 8.0 / 18.0, 5.0 / 18.0};
  double s = 0.0;
  for (int ey = max(0, (j - 1) / 2); ey <= min(N - 1, j / 2); ++ey)
    for (int ex = max(0, (i - 1) / 2); ex <= min(N - 1, i / 2); ++ex) {
      const int a = i - 2 * ex, bb = j - 2 * ey;
      for (int qy = 0; qy < 3; ++qy)
        for (int qx = 0; qx < 3; ++qx) {
          const double t = gp[qx], u = gp[qy];
          double fx, fy;
          mms_f(kind, nu, (ex + t) * g.h, (ey + u) * g.h, fx, fy);
          s += gw[qx] * gw[qy] * (plane ? fy : fx) * lagr2(a, t) * lagr2(bb, u);
        }
    }
  b[o] = s * g.h * g.h;
}

// ---------------------------------------------------------------------------
// Transfers (finite-element interpolation P, restriction P^T).
// 1D Q2 interpolation, fine lattice f -> coarse lattice:
//   f = 4e   : coarse 2e   (1)          f = 4e+2 : coarse 2e+1 (1)
//   f = 4e+1 : 2e, 2e+1, 2e+2  (3/8, 3/4, -1/8)
//   f = 4e+3 : 2e, 2e+1, 2e+2  (-1/8, 3/4, 3/8)
// 1D Q1: fine 2e -> coarse e (1); fine 2e+1 -> e, e+1 (1/2, 1/2)
// ---------------------------------------------------------------------------
// P^T column (coarse lattice c): fine indices 2c + off
__device__ __forceinline__ int p2col(int c, int* f, double* w) {
  if (c & 1) {
    f[0] = 2 * c - 1; f[1] = 2 * c; f[2] = 2 * c + 1;
    w[0] = 0.75; w[1] = 1.0; w[2] = 0.75;
    return 3;
  }
  f[0] = 2 * c - 3; f[1] = 2 * c - 1; f[2] = 2 * c; f[3] = 2 * c + 1; f[4] = 2 * c + 3;
  w[0] = -0.125; w[1] = 0.375; w[2] = 1.0; w[3] = 0.375; w[4] = -0.125;
  return 5;
}

// Vectorised prolongation x_f += P e_c (alg:mg "Correction"), the form
// used by the V-cycle.  Velocity (1D Q2, fine lattice 4e+m from coarse lattice
// 2e..2e+2: m=0 -> (1,0,0), 1 -> (3/8,3/4,-1/8), 2 -> (0,1,0), 3 -> (-1/8,3/4,3/8)):
// one thread per coarse element (ex, ey) and component produces the 4x4 fine
// points (4ex.., 4ey..) from its 3x3 coarse values -- 9 loads, 16 read-modify-
// writes as double2.  Only the owned fine rows [2 r0, 2 r1) are written;
// Dirichlet points (i or j = 0; 4 Nc is never produced) are left untouched.
__device__ __forceinline__ void prolong_q2_at(const LevelGeom& gf, const LevelGeom& gc, const double* __restrict__ ec,
                                              double* __restrict__ xf, int ex, int ey, int comp) {
  if (ex >= gc.N || ey >= gc.N) return;
  const int jlo = max(2 * gf.r0, 1), jhi = min(2 * gf.r1, gf.lat - 1);
  const double* e = ec + (comp ? gc.ouy : gc.oux) + (int64_t)(2 * ey) * gc.pu + 2 * ex;
  double tx[3][4];
#pragma unroll
  for (int r = 0; r < 3; ++r) {
    const double c0 = e[(int64_t)r * gc.pu], c1 = e[(int64_t)r * gc.pu + 1], c2 = e[(int64_t)r * gc.pu + 2];
    tx[r][0] = ex == 0 ? 0.0 : c0;  // fine column 0 is Dirichlet
    tx[r][1] = 0.375 * c0 + 0.75 * c1 - 0.125 * c2;
    tx[r][2] = c1;
    tx[r][3] = -0.125 * c0 + 0.75 * c1 + 0.375 * c2;
  }
  double* f = xf + (comp ? gf.ouy : gf.oux) + (int64_t)(4 * ey) * gf.pu + 4 * ex;
#pragma unroll
  for (int m = 0; m < 4; ++m) {
    const int j = 4 * ey + m;
    if (j < jlo || j >= jhi) continue;
    const double w0 = m == 0 ? 1.0 : m == 1 ? 0.375 : m == 2 ? 0.0 : -0.125;
    const double w1 = m == 0 ? 0.0 : m == 1 ? 0.75 : m == 2 ? 1.0 : 0.75;
    const double w2 = m == 0 ? 0.0 : m == 1 ? -0.125 : m == 2 ? 0.0 : 0.375;
    double2* row = reinterpret_cast<double2*>(f + (int64_t)m * gf.pu);
    double2 a = row[0], b = row[1];
    a.x += w0 * tx[0][0] + w1 * tx[1][0] + w2 * tx[2][0];
    a.y += w0 * tx[0][1] + w1 * tx[1][1] + w2 * tx[2][1];
    b.x += w0 * tx[0][2] + w1 * tx[1][2] + w2 * tx[2][2];
    b.y += w0 * tx[0][3] + w1 * tx[1][3] + w2 * tx[2][3];
    row[0] = a;
    row[1] = b;
  }
}
// pressure (1D Q1: fine node 2a <- a, 2a+1 <- (a, a+1)/2): one thread per coarse
// node (ax, ay) produces fine nodes (2ax, 2ax+1) x (2ay, 2ay+1); owned rows only.
__device__ __forceinline__ void prolong_q1_at(const LevelGeom& gf, const LevelGeom& gc, const double* __restrict__ ec,
                                              double* __restrict__ xf, int ax, int ay) {
  if (ax > gc.N || ay > gc.N) return;
  const double* e = ec + gc.op + (int64_t)ay * gc.pp + ax;
  const bool rx = ax < gc.N, ry = ay < gc.N;  // neighbours exist
  const double c00 = e[0], c10 = rx ? e[1] : 0.0, c01 = ry ? e[gc.pp] : 0.0, c11 = rx && ry ? e[gc.pp + 1] : 0.0;
#pragma unroll
  for (int dy = 0; dy < 2; ++dy) {
    const int j = 2 * ay + dy;
    if (j < gf.r0 || j >= gf.r1 || j > gf.N) continue;
    const double l = dy ? 0.5 * (c00 + c01) : c00, r = dy ? 0.5 * (c10 + c11) : c10;
    double* f = xf + gf.op + (int64_t)j * gf.pp + 2 * ax;
    if (rx) {
      double2 v = *reinterpret_cast<double2*>(f);
      v.x += l;
      v.y += 0.5 * (l + r);
      *reinterpret_cast<double2*>(f) = v;
    } else {
      f[0] += l;
    }
  }
}

// One launch for both transfers: blockIdx.z = 0, 1 -> velocity components (coarse
// element rows from ey0, ney of them), 2 -> pressure (coarse node rows from ay0, nay).
__global__ void __launch_bounds__(128) k_prolong(LevelGeom gf, LevelGeom gc, const double* __restrict__ ec,
                                                 double* __restrict__ xf, int ey0, int ney, int ay0, int nay) {
  pdl_wait();
  const int cx = blockIdx.x * blockDim.x + threadIdx.x;
  const int cy = blockIdx.y * blockDim.y + threadIdx.y;
  if (blockIdx.z < 2) {
    if (cy < ney) prolong_q2_at(gf, gc, ec, xf, cx, ey0 + cy, blockIdx.z);
  } else if (cy < nay) {
    prolong_q1_at(gf, gc, ec, xf, cx, ay0 + cy);
  }
}

// r_c = P^T r_f, coarse Dirichlet rows and padding set to 0
__global__ void k_restrict(LevelGeom gf, LevelGeom gc, const double* __restrict__ rf, double* __restrict__ rc,
                           int plane0) {
  const int plane = plane0 + blockIdx.z;  // planes plane0 .. plane0 + gridDim.z - 1
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const int j = blockIdx.y * blockDim.y + threadIdx.y;
  if (plane < 2) {
    if (j >= gc.lat || i >= gc.pu) return;
    const int64_t o = (plane ? gc.ouy : gc.oux) + (int64_t)j * gc.pu + i;
    if (i < 1 || j < 1 || i >= gc.lat - 1 || j >= gc.lat - 1) { rc[o] = 0.0; return; }
    int fx[5], fy[5];
    double wx[5], wy[5];
    const int nx = p2col(i, fx, wx), ny = p2col(j, fy, wy);
    const double* r = rf + (plane ? gf.ouy : gf.oux);
    double s = 0.0;
    for (int b = 0; b < ny; ++b) {
      double t = 0.0;
      for (int a = 0; a < nx; ++a) t += wx[a] * r[(int64_t)fy[b] * gf.pu + fx[a]];
      s += wy[b] * t;
    }
    rc[o] = s;
  } else {
    if (j > gc.N || i >= gc.pp) return;
    const int64_t o = p_at(gc, i, j);
    if (i > gc.N) { rc[o] = 0.0; return; }
    const double* r = rf + gf.op;
    double s = 0.0;
    for (int b = -1; b <= 1; ++b) {
      const int fj = 2 * j + b;
      if (fj < 0 || fj > gf.N) continue;
      const double wy = b ? 0.5 : 1.0;
      for (int a = -1; a <= 1; ++a) {
        const int fi = 2 * i + a;
        if (fi < 0 || fi > gf.N) continue;
        s += wy * (a ? 0.5 : 1.0) * r[(int64_t)fj * gf.pp + fi];
      }
    }
    rc[o] = s;
  }
}

// ---------------------------------------------------------------------------
// In-place Gauss-Jordan inversion with partial (row) pivoting of an n x n
// row-major matrix `a` (shared or global), by the whole block.
// perm: n ints of scratch in the same memory space.  Returns false if singular.
// ---------------------------------------------------------------------------
__device__ bool gj_invert(double* a, int n, int lda, int* perm, double* colk, int* flag) {
  const int tid = threadIdx.x, nt = blockDim.x;
  for (int k = 0; k < n; ++k) {
    if (tid == 0) {
      int p = k;
      double best = fabs(a[k * lda + k]);
      for (int r = k + 1; r < n; ++r) {
        const double v = fabs(a[r * lda + k]);
        if (v > best) { best = v; p = r; }
      }
      perm[k] = p;
      if (best == 0.0) *flag = 1;
    }
    __syncthreads();
    if (*flag) return false;
    const int p = perm[k];
    if (p != k)
      for (int c = tid; c < n; c += nt) {
        const double t = a[k * lda + c];
        a[k * lda + c] = a[p * lda + c];
        a[p * lda + c] = t;
      }
    __syncthreads();
    const double piv = a[k * lda + k];
    __syncthreads();
    for (int c = tid; c < n; c += nt) a[k * lda + c] = (c == k ? 1.0 : a[k * lda + c]) / piv;
    for (int r = tid; r < n; r += nt) colk[r] = a[r * lda + k];
    __syncthreads();
    for (int q = tid; q < n * n; q += nt) {
      const int r = q / n, c = q % n;
      if (r == k) continue;
      a[r * lda + c] = (c == k ? 0.0 : a[r * lda + c]) - colk[r] * a[k * lda + c];
    }
    __syncthreads();
  }
  for (int k = n - 1; k >= 0; --k) {  // undo the row swaps as column swaps
    const int p = perm[k];
    if (p != k)
      for (int r = tid; r < n; r += nt) {
        const double t = a[r * lda + k];
        a[r * lda + k] = a[r * lda + p];
        a[r * lda + p] = t;
      }
    __syncthreads();
  }
  return true;
}

__host__ __device__ __forceinline__ int cat_rep(int c, int N) { return c <= 2 ? c : (c == 3 ? N - 1 : N); }

// ---------------------------------------------------------------------------
// Patch setup: one CTA per (group, level).  Builds A_i = V_i A V_i^T
// for the representative patch of group (cat_x, cat_y) from the stencil
// (P:247), restricted to non-Dirichlet DOFs (reading 7), inverts it in fp64,
// and stores the inverse in the padded 51-slot layout:
//   slot = comp*25 + oy*5 + ox for the velocity point (2kx-2+ox, 2ky-2+oy),
//   slot 50 = pressure; rows/columns of absent slots are 0.
// ---------------------------------------------------------------------------
__global__ void k_patch_setup(const int* __restrict__ Ns, double nu, double* __restrict__ inv_out,
                              int* __restrict__ status) {
  const int grp = blockIdx.x, l = blockIdx.y;
  const int N = Ns[l];
  const double h = 1.0 / N;
  const int cx = grp % 5, cy = grp / 5;
  const int kx = cat_rep(cx, N), ky = cat_rep(cy, N);
  __shared__ double a[kSlots * kSlots];
  __shared__ double colk[kSlots];
  __shared__ int slot[kSlots], perm[kSlots];
  __shared__ Dof dof[kSlots];
  __shared__ int n, flag;
  const int lat = 2 * N + 1;
  if (threadIdx.x == 0) {
    int m = 0;
    for (int comp = 0; comp < 2; ++comp)
      for (int oy = 0; oy < 5; ++oy)
        for (int ox = 0; ox < 5; ++ox) {
          const int i = 2 * kx - 2 + ox, j = 2 * ky - 2 + oy;
          if (i < 1 || j < 1 || i > lat - 2 || j > lat - 2) continue;
          dof[m] = Dof{comp, i, j};
          slot[m] = comp * 25 + oy * 5 + ox;
          ++m;
        }
    dof[m] = Dof{2, kx, ky};
    slot[m] = 50;
    n = m + 1;
    flag = 0;
  }
  __syncthreads();
  const int nn = n;
  for (int q = threadIdx.x; q < nn * nn; q += blockDim.x) a[q] = a_entry(dof[q / nn], dof[q % nn], N, nu, h);
  __syncthreads();
  const bool ok = gj_invert(a, nn, nn, perm, colk, &flag);
  double* out = inv_out + ((int64_t)l * 25 + grp) * kGroupStride;
  for (int q = threadIdx.x; q < kGroupStride; q += blockDim.x) out[q] = 0.0;
  __syncthreads();
  if (!ok) {
    if (threadIdx.x == 0) atomicExch(status, 1);
    return;
  }
  for (int q = threadIdx.x; q < nn * nn; q += blockDim.x) out[slot[q / nn] * kSlots + slot[q % nn]] = a[q];
}

// ---------------------------------------------------------------------------
// Simple Vanka (the paper's baseline variant):
// every patch builds and inverts its own A_i and stores it, instead of the 25
// shared group inverses of tuned Vanka.  One CTA per patch (batched fp64
// Gauss-Jordan, as k_patch_setup); the inverse is stored slot-interleaved over
// the patches, inv[(r * 51 + c) * np + p], so that the apply kernel's per-patch
// reads are coalesced across the threads of a warp.
// ---------------------------------------------------------------------------
// (stride, base): entry q of patch p is stored at inv_out[q * stride + p - base]
// (the simple-Vanka store uses stride = patch count, base = 0; the validation
// mode builds batches of `stride` patches starting at base).
__global__ void k_patch_setup_simple(LevelGeom g, double nu, int64_t p0, double* __restrict__ inv_out,
                                     int* __restrict__ status, int64_t stride, int64_t base) {
  const int N = g.N, lat = g.lat;
  const int64_t np = (int64_t)(N + 1) * (N + 1);
  const int64_t p = p0 + blockIdx.x;
  if (p >= np) return;
  const int kx = (int)(p % (N + 1)), ky = (int)(p / (N + 1));
  __shared__ double a[kSlots * kSlots];
  __shared__ double colk[kSlots];
  __shared__ int slot[kSlots], perm[kSlots];
  __shared__ Dof dof[kSlots];
  __shared__ int n, flag;
  if (threadIdx.x == 0) {
    int m = 0;
    for (int comp = 0; comp < 2; ++comp)
      for (int oy = 0; oy < 5; ++oy)
        for (int ox = 0; ox < 5; ++ox) {
          const int i = 2 * kx - 2 + ox, j = 2 * ky - 2 + oy;
          if (i < 1 || j < 1 || i > lat - 2 || j > lat - 2) continue;
          dof[m] = Dof{comp, i, j};
          slot[m] = comp * 25 + oy * 5 + ox;
          ++m;
        }
    dof[m] = Dof{2, kx, ky};
    slot[m] = 50;
    n = m + 1;
    flag = 0;
  }
  __syncthreads();
  const int nn = n;
  for (int q = threadIdx.x; q < nn * nn; q += blockDim.x) a[q] = a_entry(dof[q / nn], dof[q % nn], N, nu, g.h);
  __syncthreads();
  const bool ok = gj_invert(a, nn, nn, perm, colk, &flag);
  for (int q = threadIdx.x; q < kGroupStride; q += blockDim.x) inv_out[(int64_t)q * stride + p - base] = 0.0;
  __syncthreads();
  if (!ok) {
    if (threadIdx.x == 0) atomicExch(status, 1);
    return;
  }
  for (int q = threadIdx.x; q < nn * nn; q += blockDim.x)
    inv_out[(int64_t)(slot[q / nn] * kSlots + slot[q % nn]) * stride + p - base] = a[q];
}
// delta_p = A_p^{-1} V_p r with patch p's own stored inverse (one thread per patch)
__global__ void __launch_bounds__(128) k_patch_solve_simple(LevelGeom g, const double* __restrict__ r,
                                                            const double* __restrict__ inv,
                                                            double* __restrict__ dbuf) {
  const int N = g.N, lat = g.lat;
  const int64_t np = (int64_t)(N + 1) * (N + 1);
  const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= np) return;
  const int kx = (int)(p % (N + 1)), ky = (int)(p / (N + 1));
  double rv[kSlots];
#pragma unroll
  for (int comp = 0; comp < 2; ++comp)
#pragma unroll
    for (int oy = 0; oy < 5; ++oy)
#pragma unroll
      for (int ox = 0; ox < 5; ++ox) {
        const int i = 2 * kx - 2 + ox, j = 2 * ky - 2 + oy;
        const bool ok = i >= 1 && j >= 1 && i <= lat - 2 && j <= lat - 2;
        rv[comp * 25 + oy * 5 + ox] = ok ? r[(comp ? g.ouy : g.oux) + (int64_t)j * g.pu + i] : 0.0;
      }
  rv[50] = r[p_at(g, kx, ky)];
  for (int s = 0; s < kSlots; ++s) {
    double d = 0.0;
#pragma unroll
    for (int t = 0; t < kSlots; ++t) d = fma(__ldcs(inv + (int64_t)(s * kSlots + t) * np + p), rv[t], d);
    dbuf[(int64_t)s * np + p] = d;
  }
}

// ---------------------------------------------------------------------------
// Level-0 minimum-norm solve (reading 3).  Setup builds the bordered
// matrix [[A_II, n],[n^T, 0]] (n = constant pressure / sqrt(m)) in global
// memory and inverts it with one CTA; the top-left block is pinv(A_II).
// ---------------------------------------------------------------------------
__global__ void k_coarse_build(LevelGeom g, double nu, const int* __restrict__ idx, int ni, double* __restrict__ m) {
  const int n = ni + 1;
  const int r = blockIdx.x;
  auto decode = [&](int q) {
    const int64_t o = idx[q];
    Dof d;
    if (o >= g.op) { d.kind = 2; d.j = (int)((o - g.op) / g.pp); d.i = (int)((o - g.op) % g.pp); }
    else if (o >= g.ouy) { d.kind = 1; d.j = (int)((o - g.ouy) / g.pu); d.i = (int)((o - g.ouy) % g.pu); }
    else { d.kind = 0; d.j = (int)(o / g.pu); d.i = (int)(o % g.pu); }
    return d;
  };
  const double nv = 1.0 / sqrt((double)(g.N + 1) * (g.N + 1));
  for (int c = threadIdx.x; c < n; c += blockDim.x) {
    double v;
    if (r < ni && c < ni) v = a_entry(decode(r), decode(c), g.N, nu, g.h);
    else if (r == ni && c == ni) v = 0.0;
    else {
      const int q = r == ni ? c : r;
      v = decode(q).kind == 2 ? nv : 0.0;
    }
    m[(int64_t)r * n + c] = v;
  }
}
__global__ void k_coarse_invert(double* m, int n, int* perm, double* colk, int* status) {
  __shared__ int flag;
  if (threadIdx.x == 0) flag = 0;
  __syncthreads();
  if (!gj_invert(m, n, n, perm, colk, &flag) && threadIdx.x == 0) atomicExch(status, 1);
}
// x = pinv b on level 0: x zeroed by the caller, then scatter.  One warp per row
// (coalesced row reads, fixed lane-strided partial sums + shuffle tree).
__global__ void k_coarse_apply(const double* __restrict__ m, int ni, const int* __restrict__ idx,
                               const double* __restrict__ b, double* __restrict__ x) {
  pdl_wait();
  const int n = ni + 1, lane = threadIdx.x & 31;
  const int r = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (r >= ni) return;
  double s = 0.0;
  for (int c = lane; c < ni; c += 32) s = fma(m[(int64_t)r * n + c], b[idx[c]], s);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (lane == 0) x[idx[r]] = s;
}

// ---------------------------------------------------------------------------
// Unfused Vanka sweep (the paper's kernel split, alg:vk_kernels P:443-453):
//   k_patch_solve_unfused: delta_i = A_i^{-1} V_i r into a packed slot-major buffer
//   k_vanka_update:        x_out = x_in + W sum_i V_i^T delta_i (owner gathers,
//                          fixed ascending patch order)
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(128) k_patch_solve_unfused(LevelGeom g, const double* __restrict__ r,
                                                             const double* __restrict__ inv,
                                                             double* __restrict__ dbuf) {
  const int N = g.N, lat = g.lat;
  const int64_t np = (int64_t)(N + 1) * (N + 1);
  const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= np) return;
  const int kx = (int)(p % (N + 1)), ky = (int)(p / (N + 1));
  const double* A = inv + (pcat(ky, N) * 5 + pcat(kx, N)) * kGroupStride;
  double rv[kSlots];
#pragma unroll
  for (int comp = 0; comp < 2; ++comp)
#pragma unroll
    for (int oy = 0; oy < 5; ++oy)
#pragma unroll
      for (int ox = 0; ox < 5; ++ox) {
        const int i = 2 * kx - 2 + ox, j = 2 * ky - 2 + oy;
        const bool ok = i >= 1 && j >= 1 && i <= lat - 2 && j <= lat - 2;
        rv[comp * 25 + oy * 5 + ox] = ok ? r[(comp ? g.ouy : g.oux) + (int64_t)j * g.pu + i] : 0.0;
      }
  rv[50] = r[p_at(g, kx, ky)];
  for (int s = 0; s < kSlots; ++s) {
    double d = 0.0;
#pragma unroll
    for (int t = 0; t < kSlots; ++t) d += A[s * kSlots + t] * rv[t];
    dbuf[(int64_t)s * np + p] = d;
  }
}

__global__ void k_vanka_update(LevelGeom g, double omega, int scalar_w, const double* __restrict__ xin,
                               const double* __restrict__ dbuf, double* __restrict__ xout) {
  const int plane = blockIdx.z;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const int j = blockIdx.y * blockDim.y + threadIdx.y;
  const int N = g.N, lat = g.lat;
  const int64_t np = (int64_t)(N + 1) * (N + 1);
  if (plane < 2) {
    if (j >= lat || i >= g.pu) return;
    const int64_t o = (plane ? g.ouy : g.oux) + (int64_t)j * g.pu + i;
    if (i >= lat) { xout[o] = 0.0; return; }
    if (i == 0 || j == 0 || i == lat - 1 || j == lat - 1) { xout[o] = xin[o]; return; }
    const int kx0 = max(0, (i - 1) >> 1), kx1 = min(N, (i + 2) >> 1);
    const int ky0 = max(0, (j - 1) >> 1), ky1 = min(N, (j + 2) >> 1);
    double s = 0.0;
    for (int ky = ky0; ky <= ky1; ++ky)
      for (int kx = kx0; kx <= kx1; ++kx) {
        const int slot = plane * 25 + (j - 2 * ky + 2) * 5 + (i - 2 * kx + 2);
        s += dbuf[(int64_t)slot * np + (int64_t)ky * (N + 1) + kx];
      }
    const int mult = (kx1 - kx0 + 1) * (ky1 - ky0 + 1);
    xout[o] = xin[o] + (scalar_w ? omega : omega / mult) * s;
  } else {
    if (j > N || i >= g.pp) return;
    const int64_t o = p_at(g, i, j);
    if (i > N) { xout[o] = 0.0; return; }
    xout[o] = xin[o] + omega * dbuf[50 * np + (int64_t)j * (N + 1) + i];
  }
}

}  // namespace svk
