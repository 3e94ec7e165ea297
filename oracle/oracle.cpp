// =============================================================================
// oracle/oracle.cpp -- the CPU ORACLE for the Vanka / V-cycle / FGMRES hot path
// of Spies, Olson, MacLachlan, "Exploiting mesh structure to improve multigrid
// performance for saddle point problems" (arXiv 2401.06277).
//
// THIS IS TEST INFRASTRUCTURE, NOT PRODUCT CODE.  Only tests/, the smoke() of
// __graft_entry__.py and bench.py's cpu_baseline / --impl reference leg may
// load it.  It shares no code, header, table or constant generator with the
// CUDA library under paper_2401_06277_b200/ (and never includes anything from
// there); the two agree only on the documented vector layout.
//
// Deliberately plain and slow: the operator is assembled element by element
// into an explicit CSR matrix by 3x3 Gauss quadrature of the bilinear forms;
// every Vanka patch matrix is extracted from that global CSR and solved with a
// dense LU; the interpolation P is built by evaluating coarse basis functions;
// the V-cycle and FGMRES follow the paper's algorithms line by line.
//
// Citations: P:n = /root/reference/PAPER.md line n (+ label).  Readings where
// the paper is silent or inconsistent are those of SURVEY.md section 8(c) and
// are listed in DESIGN.md ("Readings").
//
// Vector layout on level with N elements per dimension (all fp64, compact):
//   [ u_x on the (2N+1)^2 velocity lattice, index j*(2N+1)+i (x fastest),
//     u_y on the same lattice,
//     p on the (N+1)^2 pressure nodes, index ky*(N+1)+kx ]
// lattice point (i,j) sits at (i*h/2, j*h/2); pressure node (kx,ky) at (kx*h, ky*h).
// Level 0 is the coarsest (alg:mg); level L-1 the finest.
//
// parity pins (tests/test_oracle*.py): brute-force dense NumPy checker for
// N<=16 (operator, sweep, V-cycle incl. the three-sweep level-0 mode, scalar
// weighting, BS / SU with finite Jacobi sweeps, block-triangular with finite
// cycles), nodal exactness of two manufactured solutions, the closed-form
// cavity data and the cavity solution's mirror symmetry, symmetry / null
// vector, 25 patch groups and tab:rwf counts, Galerkin identity, pinv for the
// coarse solve, FGMRES against its least-squares definition, and the local
// full-size samplers against the global oracle.  Every function is pinned; the
// paper prints no V-cycle convergence factors or iteration counts, so those two
// PROPERTIES have no paper value to compare with.
// =============================================================================
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <map>
#include <string>
#include <vector>
#ifdef _OPENMP
#include <omp.h>
#endif

namespace {

struct Csr {
  int64_t nrows = 0;
  std::vector<int64_t> rowptr;
  std::vector<int32_t> col;
  std::vector<double> val;
};

struct Level {
  int N = 0;
  double h = 0;
  int64_t nlat = 0;  // 2N+1
  int64_t nv = 0;    // (2N+1)^2 velocity DOFs per component
  int64_t npn = 0;   // N+1
  int64_t np = 0;    // (N+1)^2 pressure DOFs
  int64_t ntot = 0;  // 2 nv + np
  Csr A;             // full assembled operator [[L, B^T],[B, 0]] (eq:stokesmatrix)
  std::vector<uint8_t> dir;  // Dirichlet flag per DOF
  // Vanka (alg:vk)
  std::vector<int64_t> pstart;  // patch p owns dofs pdof[pstart[p] .. pstart[p+1])
  std::vector<int64_t> pdof;
  std::vector<int32_t> pgroup;  // index of the distinct patch matrix (its LU)
  std::vector<std::vector<double>> glu;  // LU factors of each distinct A_i
  std::vector<std::vector<int>> gpiv;
  std::vector<int> gsize;
  std::vector<double> weight;  // diagonal of W_i, per global DOF (see reading 6)
  // interpolation from level-1 (coarse) into this level
  Csr P, PT;
  // Braess-Sarazin / Schur-Uzawa comparators (alg:bs P:236-241, alg:uz P:313-320):
  // Dinv = 1/diag(L) on non-Dirichlet velocity DOFs (0 elsewhere), indexed by
  // global DOF (< 2 nv); S = -(1/t) B D^{-1} B^T as an explicit pressure x pressure
  // CSR (indices relative to the pressure block) and its diagonal.
  std::vector<double> Dinv;
  Csr S;
  std::vector<double> Sdiag;
  // Block-triangular preconditioner (alg:bt): Q1 pressure mass matrix
  // M_kl = int phi_l phi_k (pressure indices), and on level 0 dense LU factors of
  // the velocity block of A (Dirichlet rows are identity rows) and of M.
  Csr Mp;
  std::vector<double> lu_u, lu_m;
  std::vector<int> piv_u, piv_m;
  // level-0 direct solve (reading 3: minimum-norm)
  std::vector<int64_t> interior;
  std::vector<double> clu;
  std::vector<int> cpiv;
  int cn = 0;
};

struct Ctx {
  double nu = 1.0, omega = 0.8;
  int weighting = 0;  // 0: W_i = omega*diag(1/mult); 1: W_i = omega*I
  int nu1 = 1, nu2 = 1;
  int coarse_mode = 0;  // 0: exact min-norm solve; 1: three Vanka sweeps
  // relaxation inside the V-cycle: 0 Vanka (alg:vk), 1 inexact Braess-Sarazin
  // (alg:bs), 2 Schur-Uzawa (alg:uz); t scales D, omega_r = omega_BS (BS only),
  // omega_j / nj = weight / sweeps of the Jacobi iteration on S
  int relax = 0;
  double t = 1.0, omega_r = 1.0, omega_j = 0.8;
  int nj = 3;
  // FGMRES preconditioner: 0 monolithic V-cycle (alg:mg), 1 block-triangular
  // (alg:bt) with bt_cycles V(bt_nu, bt_nu) cycles of weighted Jacobi per block
  int precond = 0, bt_cycles = 3, bt_nu = 3;
  double bt_omega_u = 1.0, bt_omega_p = 0.6;
  std::vector<Level> lev;
  std::string err;
};

// --------------------------------------------------------------------------
// 1D Lagrange bases on the reference interval [0,1] (Q2 = biquadratic,
// Q1 = bilinear tensor-product bases).
// Quadratic nodes t = 0, 1/2, 1; linear nodes t = 0, 1.
// --------------------------------------------------------------------------
double q2(int a, double t) {
  if (a == 0) return 2.0 * (t - 0.5) * (t - 1.0);
  if (a == 1) return -4.0 * t * (t - 1.0);
  return 2.0 * t * (t - 0.5);
}
double dq2(int a, double t) {  // d/dt
  if (a == 0) return 4.0 * t - 3.0;
  if (a == 1) return -8.0 * t + 4.0;
  return 4.0 * t - 1.0;
}
double q1(int a, double t) { return a == 0 ? 1.0 - t : t; }

// 3-point Gauss-Legendre rule on [0,1]; exact for polynomials of degree <= 5,
// which covers every integrand of the forms a(.,.), b(.,.) and (f, v) here.
const double kGP[3] = {0.5 - 0.5 * std::sqrt(0.6), 0.5, 0.5 + 0.5 * std::sqrt(0.6)};
const double kGW[3] = {5.0 / 18.0, 8.0 / 18.0, 5.0 / 18.0};

// --------------------------------------------------------------------------
// Right-hand sides / boundary data (P:76-81 manufactured solution; readings
// 2 and 15 of DESIGN.md for the boundary data and the cavity).
// kind 0 ZERO, 1 MMS_PAPER, 2 MMS_INSPACE, 3 CAVITY
// --------------------------------------------------------------------------
void exact_u(int kind, double x, double y, double* ux, double* uy) {
  if (kind == 1) {
    // u = ( x(1-x)(2x-1)(6y^2-6y+1), y(y-1)(2y-1)(6x^2-6x+1) )
    *ux = x * (1 - x) * (2 * x - 1) * (6 * y * y - 6 * y + 1);
    *uy = y * (y - 1) * (2 * y - 1) * (6 * x * x - 6 * x + 1);
  } else if (kind == 2) {
    *ux = 2 * x * x * y;
    *uy = -2 * x * y * y;
  } else {
    *ux = 0;
    *uy = 0;
  }
}
void exact_p(int kind, double x, double y, double* p) {
  if (kind == 1) *p = x * x - 3 * y * y + 8.0 / 3.0 * x * y;
  else if (kind == 2) *p = x * y - 0.25;
  else *p = 0;
}
// f = -nu Laplace(u) + grad p  (eq:stokes1; "f computed to satisfy")
void forcing(int kind, double nu, double x, double y, double* fx, double* fy) {
  if (kind == 1) {
    // u_x = x(1-x)(2x-1) * (6y^2-6y+1)
    double gx = x * (1 - x) * (2 * x - 1);        // -2x^3+3x^2-x
    double gx_xx = -12 * x + 6;                    // d2/dx2
    double hy = 6 * y * y - 6 * y + 1, hy_yy = 12;
    double lap_ux = gx_xx * hy + gx * hy_yy;
    // u_y = y(y-1)(2y-1) * (6x^2-6x+1)
    double gy = y * (y - 1) * (2 * y - 1);         // 2y^3-3y^2+y
    double gy_yy = 12 * y - 6;
    double hx = 6 * x * x - 6 * x + 1, hx_xx = 12;
    double lap_uy = gy_yy * hx + gy * hx_xx;
    double px = 2 * x + 8.0 / 3.0 * y, py = -6 * y + 8.0 / 3.0 * x;
    *fx = -nu * lap_ux + px;
    *fy = -nu * lap_uy + py;
  } else if (kind == 2) {
    // u = (2x^2 y, -2 x y^2): Laplace u = (4y, -4x); p = xy - 1/4: grad p = (y, x)
    *fx = -nu * 4 * y + y;
    *fy = nu * 4 * x + x;
  } else {
    *fx = 0;
    *fy = 0;
  }
}

// --------------------------------------------------------------------------
// Dense LU with partial pivoting (row-major n x n), and solve.
// --------------------------------------------------------------------------
bool lu_factor(std::vector<double>& a, std::vector<int>& piv, int n) {
  piv.resize(n);
  for (int k = 0; k < n; ++k) {
    int pr = k;
    double best = std::fabs(a[(size_t)k * n + k]);
    for (int r = k + 1; r < n; ++r) {
      double v = std::fabs(a[(size_t)r * n + k]);
      if (v > best) { best = v; pr = r; }
    }
    if (best == 0.0) return false;
    piv[k] = pr;
    if (pr != k)
      for (int c = 0; c < n; ++c) std::swap(a[(size_t)k * n + c], a[(size_t)pr * n + c]);
    double d = a[(size_t)k * n + k];
    for (int r = k + 1; r < n; ++r) {
      double l = a[(size_t)r * n + k] / d;
      a[(size_t)r * n + k] = l;
      for (int c = k + 1; c < n; ++c) a[(size_t)r * n + c] -= l * a[(size_t)k * n + c];
    }
  }
  return true;
}
void lu_solve(const std::vector<double>& a, const std::vector<int>& piv, int n, double* x) {
  for (int k = 0; k < n; ++k) std::swap(x[k], x[piv[k]]);
  for (int r = 0; r < n; ++r) {
    double s = x[r];
    for (int c = 0; c < r; ++c) s -= a[(size_t)r * n + c] * x[c];
    x[r] = s;
  }
  for (int r = n - 1; r >= 0; --r) {
    double s = x[r];
    for (int c = r + 1; c < n; ++c) s -= a[(size_t)r * n + c] * x[c];
    x[r] = s / a[(size_t)r * n + r];
  }
}

// --------------------------------------------------------------------------
// Element-by-element assembly of A = [[L, B^T],[B, 0]].
//   L_ij = a(psi_j, psi_i) = nu int grad psi_j : grad psi_i
//   B_kj = b(psi_j, phi_k) = - int phi_k div psi_j              (
//          sign: reading 1 -- the standard sign that makes eq:stokes1 hold)
// Triplets are generated in element order, then each row is stably sorted by
// column and duplicates summed in element order.
// --------------------------------------------------------------------------
void assemble(Level& L, double nu) {
  const int N = L.N;
  const double h = L.h;
  const int64_t nlat = L.nlat, nv = L.nv, npn = L.npn;
  auto iux = [&](int64_t i, int64_t j) { return j * nlat + i; };
  auto iuy = [&](int64_t i, int64_t j) { return nv + j * nlat + i; };
  auto ipp = [&](int64_t kx, int64_t ky) { return 2 * nv + ky * npn + kx; };

  // element matrices on the reference square mapped to [0,h]^2 (Jacobian h^2,
  // d/dx = (1/h) d/dt); identical on every element of the uniform grid.
  double Le[9][9] = {{0}}, Bxe[4][9] = {{0}}, Bye[4][9] = {{0}};
  for (int qx = 0; qx < 3; ++qx)
    for (int qy = 0; qy < 3; ++qy) {
      double t = kGP[qx], s = kGP[qy], w = kGW[qx] * kGW[qy] * h * h;
      double dx[9], dy[9];
      for (int b = 0; b < 3; ++b)
        for (int a = 0; a < 3; ++a) {
          dx[b * 3 + a] = dq2(a, t) * q2(b, s) / h;
          dy[b * 3 + a] = q2(a, t) * dq2(b, s) / h;
        }
      for (int m = 0; m < 9; ++m)
        for (int n2 = 0; n2 < 9; ++n2) Le[m][n2] += nu * w * (dx[m] * dx[n2] + dy[m] * dy[n2]);
      for (int d = 0; d < 2; ++d)
        for (int c = 0; c < 2; ++c) {
          double phi = q1(c, t) * q1(d, s);
          for (int m = 0; m < 9; ++m) {
            Bxe[d * 2 + c][m] += -w * phi * dx[m];
            Bye[d * 2 + c][m] += -w * phi * dy[m];
          }
        }
    }

  const int64_t n = L.ntot;
  std::vector<int64_t> cnt(n + 1, 0);
  auto for_each_triplet = [&](auto&& emit) {
    for (int ey = 0; ey < N; ++ey)
      for (int ex = 0; ex < N; ++ex) {
        int64_t vi[9], pi[4];
        for (int b = 0; b < 3; ++b)
          for (int a = 0; a < 3; ++a) vi[b * 3 + a] = iux(2 * ex + a, 2 * ey + b);
        for (int d = 0; d < 2; ++d)
          for (int c = 0; c < 2; ++c) pi[d * 2 + c] = ipp(ex + c, ey + d);
        for (int m = 0; m < 9; ++m)
          for (int n2 = 0; n2 < 9; ++n2) {
            emit(vi[m], vi[n2], Le[m][n2]);            // L, x component
            emit(vi[m] + nv, vi[n2] + nv, Le[m][n2]);  // L, y component
          }
        for (int k = 0; k < 4; ++k)
          for (int m = 0; m < 9; ++m) {
            emit(pi[k], vi[m], Bxe[k][m]);        // B_x
            emit(pi[k], vi[m] + nv, Bye[k][m]);   // B_y
            emit(vi[m], pi[k], Bxe[k][m]);        // B_x^T
            emit(vi[m] + nv, pi[k], Bye[k][m]);   // B_y^T
          }
      }
  };
  for_each_triplet([&](int64_t r, int64_t, double) { cnt[r + 1]++; });
  for (int64_t r = 0; r < n; ++r) cnt[r + 1] += cnt[r];
  std::vector<int32_t> tc(cnt[n]);
  std::vector<double> tv(cnt[n]);
  {
    std::vector<int64_t> pos(cnt.begin(), cnt.end() - 1);
    for_each_triplet([&](int64_t r, int64_t c, double v) {
      int64_t q = pos[r]++;
      tc[q] = (int32_t)c;
      tv[q] = v;
    });
  }
  // stable sort each row by column and sum duplicates (element order kept)
  std::vector<int64_t> newcnt(n + 1, 0);
#pragma omp parallel for schedule(dynamic, 4096)
  for (int64_t r = 0; r < n; ++r) {
    int64_t b = cnt[r], e = cnt[r + 1];
    std::vector<int64_t> idx(e - b);
    for (int64_t q = b; q < e; ++q) idx[q - b] = q;
    std::stable_sort(idx.begin(), idx.end(), [&](int64_t x, int64_t y) { return tc[x] < tc[y]; });
    std::vector<int32_t> c2;
    std::vector<double> v2;
    for (int64_t q : idx) {
      if (!c2.empty() && c2.back() == tc[q]) v2.back() += tv[q];
      else { c2.push_back(tc[q]); v2.push_back(tv[q]); }
    }
    for (size_t q = 0; q < c2.size(); ++q) { tc[b + q] = c2[q]; tv[b + q] = v2[q]; }
    newcnt[r + 1] = (int64_t)c2.size();
  }
  for (int64_t r = 0; r < n; ++r) newcnt[r + 1] += newcnt[r];
  L.A.nrows = n;
  L.A.rowptr = newcnt;
  L.A.col.resize(newcnt[n]);
  L.A.val.resize(newcnt[n]);
#pragma omp parallel for schedule(static)
  for (int64_t r = 0; r < n; ++r) {
    int64_t len = newcnt[r + 1] - newcnt[r];
    std::memcpy(&L.A.col[newcnt[r]], &tc[cnt[r]], len * sizeof(int32_t));
    std::memcpy(&L.A.val[newcnt[r]], &tv[cnt[r]], len * sizeof(double));
  }

  // Dirichlet velocity on all edges, both components (reading 2)
  L.dir.assign(n, 0);
  for (int64_t j = 0; j < nlat; ++j)
    for (int64_t i = 0; i < nlat; ++i)
      if (i == 0 || j == 0 || i == nlat - 1 || j == nlat - 1) {
        L.dir[iux(i, j)] = 1;
        L.dir[iuy(i, j)] = 1;
      }
}

// y = A x, then Dirichlet rows set to 0 (the operator of the interior system)
void matvec_masked(const Level& L, const double* x, double* y) {
#pragma omp parallel for schedule(static)
  for (int64_t r = 0; r < L.ntot; ++r) {
    double s = 0;
    for (int64_t q = L.A.rowptr[r]; q < L.A.rowptr[r + 1]; ++q) s += L.A.val[q] * x[L.A.col[q]];
    y[r] = L.dir[r] ? 0.0 : s;
  }
}

// r = b - A x on non-Dirichlet rows, 0 on Dirichlet rows (alg:mg line 3)
void residual(const Level& L, const double* x, const double* b, double* r) {
#pragma omp parallel for schedule(static)
  for (int64_t q = 0; q < L.ntot; ++q) {
    double s = b[q];
    for (int64_t k = L.A.rowptr[q]; k < L.A.rowptr[q + 1]; ++k) s -= L.A.val[k] * x[L.A.col[k]];
    r[q] = L.dir[q] ? 0.0 : s;
  }
}

// --------------------------------------------------------------------------
// Vanka patches.  Patch (kx,ky), 0<=kx,ky<=N, one per pressure node
// (reading 7: boundary nodes included, as tab:rwf's 76+124l+51l^2 requires):
// the pressure DOF at the node plus every velocity DOF (both components) of the
// <=2x2 elements around it, i.e. lattice window [2kx-2,2kx+2]x[2ky-2,2ky+2]
// clipped to the domain, minus Dirichlet DOFs (reading 7).
// A_i = V_i A V_i^T is extracted from the globally assembled A (reading 8) and
// LU-factored once ("inverting each patch matrix ahead of time");
// bitwise-identical A_i share one factorisation (tuned Vanka).
// --------------------------------------------------------------------------
// A_i = V_i A V_i^T of patch p (row-major n x n, n = the patch's DOF count):
// entry (r, c) = A[pdof[r], pdof[c]] from the global CSR.  The patch's DOF list
// is ascending (component, lattice row, lattice column, then the pressure
// node), so each CSR column is located by binary search.
std::vector<double> extract_patch(const Level& L, int64_t p) {
  const int64_t b = L.pstart[p], e = L.pstart[p + 1];
  const int n = (int)(e - b);
  const int64_t* dofs = &L.pdof[b];
  std::vector<double> Ai((size_t)n * n, 0.0);
  for (int r = 0; r < n; ++r) {
    const int64_t g = dofs[r];
    for (int64_t q = L.A.rowptr[g]; q < L.A.rowptr[g + 1]; ++q) {
      const int64_t* it = std::lower_bound(dofs, dofs + n, (int64_t)L.A.col[q]);
      if (it != dofs + n && *it == L.A.col[q]) Ai[(size_t)r * n + (it - dofs)] = L.A.val[q];
    }
  }
  return Ai;
}
// FNV-1a over the bytes of a matrix (a bucket key only; equality is bitwise)
uint64_t bytes_hash(const std::vector<double>& a) {
  uint64_t h = 1469598103934665603ull;
  const unsigned char* s = (const unsigned char*)a.data();
  for (size_t k = 0; k < a.size() * sizeof(double); ++k) h = (h ^ s[k]) * 1099511628211ull;
  return h ^ a.size();
}

bool build_patches(Level& L, double omega, int weighting, std::string& err) {
  const int N = L.N;
  const int64_t nlat = L.nlat, nv = L.nv, npn = L.npn;
  const int64_t npatch = (int64_t)(N + 1) * (N + 1);
  L.pstart.assign(npatch + 1, 0);
  L.pdof.clear();
  for (int ky = 0; ky <= N; ++ky)
    for (int kx = 0; kx <= N; ++kx) {
      for (int comp = 0; comp < 2; ++comp)
        for (int64_t j = 2 * ky - 2; j <= 2 * ky + 2; ++j)
          for (int64_t i = 2 * kx - 2; i <= 2 * kx + 2; ++i) {
            if (i < 0 || j < 0 || i >= nlat || j >= nlat) continue;
            int64_t g = comp * nv + j * nlat + i;
            if (!L.dir[g]) L.pdof.push_back(g);
          }
      L.pdof.push_back(2 * nv + (int64_t)ky * npn + kx);
      L.pstart[(int64_t)ky * (N + 1) + kx + 1] = (int64_t)L.pdof.size();
    }
  // extract every A_i, deduplicate by bitwise equality: patch p joins the group
  // of the first patch (ascending order) whose A_i is bitwise identical, else it
  // opens a new group.  Only the group representatives are stored; a 64-bit
  // hash of each A_i's bytes only narrows the candidates -- membership is
  // decided by a full bitwise comparison with the representative.
  L.pgroup.assign(npatch, -1);
  L.glu.clear();
  L.gpiv.clear();
  L.gsize.clear();
  std::vector<uint64_t> hash(npatch);
#pragma omp parallel for schedule(dynamic, 256)
  for (int64_t p = 0; p < npatch; ++p) hash[p] = bytes_hash(extract_patch(L, p));
  std::vector<std::vector<double>> rep;  // A_i of each group's first patch
  std::multimap<uint64_t, int> by_hash;   // hash -> group ids
  auto find_group = [&](uint64_t hv, const std::vector<double>& Ai) {
    auto range = by_hash.equal_range(hv);
    for (auto it = range.first; it != range.second; ++it)
      if (rep[it->second].size() == Ai.size() &&
          std::memcmp(rep[it->second].data(), Ai.data(), Ai.size() * sizeof(double)) == 0)
        return it->second;
    return -1;
  };
  // pass 1 (serial, ascending patches): a patch whose hash is new opens a group
  std::vector<uint8_t> settled(npatch, 0);
  for (int64_t p = 0; p < npatch; ++p) {
    if (by_hash.count(hash[p])) continue;
    std::vector<double> Ai = extract_patch(L, p);
    int gid = (int)rep.size();
    rep.push_back(Ai);
    by_hash.emplace(hash[p], gid);
    L.pgroup[p] = gid;
    settled[p] = 1;
  }
  // pass 2 (parallel): every other patch is compared bitwise with the
  // representatives of its hash
#pragma omp parallel for schedule(dynamic, 256)
  for (int64_t p = 0; p < npatch; ++p)
    if (!settled[p]) L.pgroup[p] = find_group(hash[p], extract_patch(L, p));
  // pass 3 (serial): hash collisions without a bitwise match open groups in
  // ascending patch order (never taken in practice; kept for exactness)
  for (int64_t p = 0; p < npatch; ++p) {
    if (L.pgroup[p] >= 0) continue;
    std::vector<double> Ai = extract_patch(L, p);
    int g = find_group(hash[p], Ai);
    if (g < 0) {
      g = (int)rep.size();
      rep.push_back(Ai);
      by_hash.emplace(hash[p], g);
    }
    L.pgroup[p] = g;
  }
  // group ids in order of the group's first patch
  std::vector<int> first(rep.size(), -1), order;
  for (int64_t p = 0; p < npatch; ++p)
    if (first[L.pgroup[p]] < 0) { first[L.pgroup[p]] = (int)order.size(); order.push_back(L.pgroup[p]); }
  for (int64_t p = 0; p < npatch; ++p) L.pgroup[p] = first[L.pgroup[p]];
  for (int g : order) {
    std::vector<double> Ai = rep[g];
    int n = (int)std::lround(std::sqrt((double)Ai.size()));
    std::vector<int> piv;
    if (!lu_factor(Ai, piv, n)) { err = "singular patch matrix"; return false; }
    L.glu.push_back(std::move(Ai));
    L.gpiv.push_back(std::move(piv));
    L.gsize.push_back(n);
  }
  // weights W_i ("the matrix with the weights"; reading 6):
  // multiplicity weighting omega/mult(j), mult(j) = number of patches holding j
  std::vector<int> mult(L.ntot, 0);
  for (int64_t q = 0; q < (int64_t)L.pdof.size(); ++q) mult[L.pdof[q]]++;
  L.weight.assign(L.ntot, 0.0);
  for (int64_t g = 0; g < L.ntot; ++g)
    if (mult[g] > 0) L.weight[g] = weighting == 0 ? omega / mult[g] : omega;
  return true;
}

// x_out = x_in + sum_i V_i^T W_i A_i^{-1} V_i (b - A x_in)   (alg:vk)
// patch solves in parallel, accumulation serial in ascending patch order
void vanka_sweep(const Level& L, const double* xin, const double* b, double* xout) {
  const int64_t npatch = (int64_t)L.pstart.size() - 1;
  std::vector<double> r(L.ntot);
  residual(L, xin, b, r.data());
  std::vector<double> delta(L.pdof.size());
#pragma omp parallel for schedule(static)
  for (int64_t p = 0; p < npatch; ++p) {
    int64_t s = L.pstart[p];
    int n = (int)(L.pstart[p + 1] - s);
    double* d = &delta[s];
    for (int q = 0; q < n; ++q) d[q] = r[L.pdof[s + q]];  // V_i r
    int g = L.pgroup[p];
    lu_solve(L.glu[g], L.gpiv[g], n, d);                   // A_i^{-1} V_i r
  }
  std::vector<double> acc(L.ntot, 0.0);
  for (int64_t q = 0; q < (int64_t)L.pdof.size(); ++q) {
    int64_t g = L.pdof[q];
    acc[g] += L.weight[g] * delta[q];
  }
#pragma omp parallel for schedule(static)
  for (int64_t q = 0; q < L.ntot; ++q) xout[q] = xin[q] + acc[q];
}

// --------------------------------------------------------------------------
// Braess-Sarazin and Schur-Uzawa, the paper's same-run
// comparators.  Everything is taken from the assembled CSR A:
//   B   = pressure rows of A restricted to velocity columns (eq:stokesmatrix),
//   B^T = velocity rows of A restricted to pressure columns (A is symmetric; the
//         Dirichlet velocity rows are identity rows, so they hold no B^T entries),
//   D   = diag(L) on the non-Dirichlet velocity DOFs (Dirichlet: D^{-1} := 0, the
//         correction there stays 0),
//   S   = -(1/t) B D^{-1} B^T, formed entry by entry as an explicit
//         sparse product  S_km = -(1/t) sum_j B_kj D^{-1}_j B_mj.
// --------------------------------------------------------------------------
void build_schur(Level& L, double t) {
  const int64_t nvel = 2 * L.nv, np = L.np;
  L.Dinv.assign(nvel, 0.0);
  for (int64_t r = 0; r < nvel; ++r) {
    if (L.dir[r]) continue;
    for (int64_t q = L.A.rowptr[r]; q < L.A.rowptr[r + 1]; ++q)
      if (L.A.col[q] == r) L.Dinv[r] = 1.0 / L.A.val[q];
  }
  L.S = Csr();
  L.S.nrows = np;
  L.S.rowptr.assign(np + 1, 0);
  L.Sdiag.assign(np, 0.0);
  std::vector<std::map<int32_t, double>> rows(np);
#pragma omp parallel for schedule(dynamic, 64)
  for (int64_t k = 0; k < np; ++k) {
    const int64_t rk = nvel + k;
    std::map<int32_t, double>& acc = rows[k];
    for (int64_t q = L.A.rowptr[rk]; q < L.A.rowptr[rk + 1]; ++q) {
      const int64_t j = L.A.col[q];
      if (j >= nvel || L.Dinv[j] == 0.0) continue;
      const double bkj = L.A.val[q] * L.Dinv[j];
      for (int64_t q2 = L.A.rowptr[j]; q2 < L.A.rowptr[j + 1]; ++q2) {  // B^T_{j m} = A_{j, nvel+m}
        const int64_t m = L.A.col[q2];
        if (m < nvel) continue;
        acc[(int32_t)(m - nvel)] += bkj * L.A.val[q2];
      }
    }
  }
  for (int64_t k = 0; k < np; ++k) {
    for (auto& kv : rows[k]) {
      L.S.col.push_back(kv.first);
      L.S.val.push_back(-kv.second / t);
      if (kv.first == k) L.Sdiag[k] = -kv.second / t;
    }
    L.S.rowptr[k + 1] = (int64_t)L.S.col.size();
  }
}

// y_p = B v_u (v_u: the velocity part of a full vector)
void apply_B(const Level& L, const double* v, double* y) {
  const int64_t nvel = 2 * L.nv;
#pragma omp parallel for schedule(static)
  for (int64_t k = 0; k < L.np; ++k) {
    double s = 0;
    for (int64_t q = L.A.rowptr[nvel + k]; q < L.A.rowptr[nvel + k + 1]; ++q)
      if (L.A.col[q] < nvel) s += L.A.val[q] * v[L.A.col[q]];
    y[k] = s;
  }
}
// y_u = B^T p (p: pressure block), 0 on Dirichlet velocity rows
void apply_BT(const Level& L, const double* p, double* y) {
  const int64_t nvel = 2 * L.nv;
#pragma omp parallel for schedule(static)
  for (int64_t j = 0; j < nvel; ++j) {
    double s = 0;
    for (int64_t q = L.A.rowptr[j]; q < L.A.rowptr[j + 1]; ++q)
      if (L.A.col[q] >= nvel) s += L.A.val[q] * p[L.A.col[q] - nvel];
    y[j] = L.dir[j] ? 0.0 : s;
  }
}
// nj sweeps of weighted Jacobi on S dp = rhs from dp = 0 ("standard weighted Jacobi")
void schur_jacobi(const Level& L, const double* rhs, double omega_j, int nj, double* dp) {
  std::vector<double> sdp(L.np);
  for (int64_t k = 0; k < L.np; ++k) dp[k] = 0.0;
  for (int it = 0; it < nj; ++it) {
#pragma omp parallel for schedule(static)
    for (int64_t k = 0; k < L.np; ++k) {
      double s = 0;
      for (int64_t q = L.S.rowptr[k]; q < L.S.rowptr[k + 1]; ++q) s += L.S.val[q] * dp[L.S.col[q]];
      sdp[k] = s;
    }
    for (int64_t k = 0; k < L.np; ++k) dp[k] += omega_j * (rhs[k] - sdp[k]) / L.Sdiag[k];
  }
}
// alg:bs: inexact Braess-Sarazin, x_out = x_in + omega_BS (du, dp)
//   S dp = r_p - (1/t) B D^{-1} r_u   (eq:bseq1, approximately by Jacobi)
//   du   = (1/t) D^{-1} (r_u - B^T dp)  (eq:bseq2)
void bs_sweep(const Ctx& c, const Level& L, const double* xin, const double* b, double* xout) {
  const int64_t nvel = 2 * L.nv;
  std::vector<double> r(L.ntot), w(nvel), rhs(L.np), dp(L.np), btdp(nvel);
  residual(L, xin, b, r.data());
  for (int64_t j = 0; j < nvel; ++j) w[j] = L.Dinv[j] * r[j] / c.t;
  apply_B(L, w.data(), rhs.data());
  for (int64_t k = 0; k < L.np; ++k) rhs[k] = r[nvel + k] - rhs[k];
  schur_jacobi(L, rhs.data(), c.omega_j, c.nj, dp.data());
  apply_BT(L, dp.data(), btdp.data());
  for (int64_t j = 0; j < nvel; ++j) xout[j] = xin[j] + c.omega_r * (L.Dinv[j] * (r[j] - btdp[j]) / c.t);
  for (int64_t k = 0; k < L.np; ++k) xout[nvel + k] = xin[nvel + k] + c.omega_r * dp[k];
}
// alg:uz: Schur-Uzawa, the block lower-triangular system eq:uzblock
//   t D du = r_u ;  S dp = r_p - B du  (reading 19: alg:uz's
//   "S dp = B du - r_p" contradicts eq:uzblock by a sign; eq:uzblock is followed)
void su_sweep(const Ctx& c, const Level& L, const double* xin, const double* b, double* xout) {
  const int64_t nvel = 2 * L.nv;
  std::vector<double> r(L.ntot), du(nvel), rhs(L.np), dp(L.np);
  residual(L, xin, b, r.data());
  for (int64_t j = 0; j < nvel; ++j) du[j] = L.Dinv[j] * r[j] / c.t;
  apply_B(L, du.data(), rhs.data());
  for (int64_t k = 0; k < L.np; ++k) rhs[k] = r[nvel + k] - rhs[k];
  schur_jacobi(L, rhs.data(), c.omega_j, c.nj, dp.data());
  for (int64_t j = 0; j < nvel; ++j) xout[j] = xin[j] + du[j];
  for (int64_t k = 0; k < L.np; ++k) xout[nvel + k] = xin[nvel + k] + dp[k];
}
// one relaxation sweep of the configured kind ("Relax on u_l and p_l", alg:mg)
void relax(const Ctx& c, const Level& L, const double* xin, const double* b, double* xout) {
  if (c.relax == 1) bs_sweep(c, L, xin, b, xout);
  else if (c.relax == 2) su_sweep(c, L, xin, b, xout);
  else vanka_sweep(L, xin, b, xout);
}

// --------------------------------------------------------------------------
// Interpolation P_{l-1}: coarse -> fine, the finite-element interpolation of the
// nested Q2 / Q1 spaces: row of a fine DOF = coarse basis functions
// evaluated at the fine DOF's coordinates.
// --------------------------------------------------------------------------
void build_prolongation(const Level& C, Level& F) {
  const int64_t fl = F.nlat, cl = C.nlat;
  std::vector<std::vector<std::pair<int32_t, double>>> rows(F.ntot);
  for (int comp = 0; comp < 2; ++comp)
    for (int64_t j = 0; j < fl; ++j)
      for (int64_t i = 0; i < fl; ++i) {
        // fine lattice i sits at i*hf/2 = (i/4)*hc: coarse element floor(i/4)
        int64_t ex = std::min<int64_t>(i / 4, C.N - 1), ey = std::min<int64_t>(j / 4, C.N - 1);
        double t = (i - 4.0 * ex) / 4.0, s = (j - 4.0 * ey) / 4.0;
        auto& row = rows[comp * F.nv + j * fl + i];
        for (int b = 0; b < 3; ++b)
          for (int a = 0; a < 3; ++a) {
            double w = q2(a, t) * q2(b, s);
            if (w != 0.0) row.push_back({(int32_t)(comp * C.nv + (2 * ey + b) * cl + 2 * ex + a), w});
          }
      }
  for (int64_t ky = 0; ky < F.npn; ++ky)
    for (int64_t kx = 0; kx < F.npn; ++kx) {
      int64_t ex = std::min<int64_t>(kx / 2, C.N - 1), ey = std::min<int64_t>(ky / 2, C.N - 1);
      double t = (kx - 2.0 * ex) / 2.0, s = (ky - 2.0 * ey) / 2.0;
      auto& row = rows[2 * F.nv + ky * F.npn + kx];
      for (int d = 0; d < 2; ++d)
        for (int c = 0; c < 2; ++c) {
          double w = q1(c, t) * q1(d, s);
          if (w != 0.0) row.push_back({(int32_t)(2 * C.nv + (ey + d) * C.npn + ex + c), w});
        }
    }
  F.P.nrows = F.ntot;
  F.P.rowptr.assign(F.ntot + 1, 0);
  for (int64_t r = 0; r < F.ntot; ++r) F.P.rowptr[r + 1] = F.P.rowptr[r] + (int64_t)rows[r].size();
  F.P.col.resize(F.P.rowptr[F.ntot]);
  F.P.val.resize(F.P.rowptr[F.ntot]);
  for (int64_t r = 0; r < F.ntot; ++r)
    for (size_t q = 0; q < rows[r].size(); ++q) {
      F.P.col[F.P.rowptr[r] + q] = rows[r][q].first;
      F.P.val[F.P.rowptr[r] + q] = rows[r][q].second;
    }
  // explicit transpose (restriction = P^T)
  Csr& T = F.PT;
  T.nrows = C.ntot;
  T.rowptr.assign(C.ntot + 1, 0);
  for (int64_t q = 0; q < (int64_t)F.P.col.size(); ++q) T.rowptr[F.P.col[q] + 1]++;
  for (int64_t r = 0; r < C.ntot; ++r) T.rowptr[r + 1] += T.rowptr[r];
  T.col.resize(F.P.col.size());
  T.val.resize(F.P.col.size());
  std::vector<int64_t> pos(T.rowptr.begin(), T.rowptr.end() - 1);
  for (int64_t r = 0; r < F.ntot; ++r)
    for (int64_t q = F.P.rowptr[r]; q < F.P.rowptr[r + 1]; ++q) {
      int64_t c = F.P.col[q];
      T.col[pos[c]] = (int32_t)r;
      T.val[pos[c]] = F.P.val[q];
      pos[c]++;
    }
}

// r_c = P^T r_f with coarse Dirichlet rows set to 0 (alg:mg line 4; reading 9)
void restrict_(const Level& C, const Level& F, const double* rf, double* rc) {
#pragma omp parallel for schedule(static)
  for (int64_t r = 0; r < C.ntot; ++r) {
    double s = 0;
    for (int64_t q = F.PT.rowptr[r]; q < F.PT.rowptr[r + 1]; ++q) s += F.PT.val[q] * rf[F.PT.col[q]];
    rc[r] = C.dir[r] ? 0.0 : s;
  }
}
// x_f += P e_c  (alg:mg line 9)
void prolong_add(const Level& F, const double* ec, double* xf) {
#pragma omp parallel for schedule(static)
  for (int64_t r = 0; r < F.ntot; ++r) {
    double s = 0;
    for (int64_t q = F.P.rowptr[r]; q < F.P.rowptr[r + 1]; ++q) s += F.P.val[q] * ec[F.P.col[q]];
    xf[r] += s;
  }
}

// --------------------------------------------------------------------------
// Level-0 solve "A_0^{-1}".  A_0 restricted to the non-Dirichlet
// DOFs is singular with the constant pressure as its null vector (P:66,
// reading 3); we take the minimum-norm solution via the bordered system
//   [[A_II, n],[n^T, 0]] [x; lambda] = [b_I; 0],   n = 1_p / sqrt(m),
// whose x equals pinv(A_II) b_I for any b_I (tests pin this to numpy.pinv).
// --------------------------------------------------------------------------
bool build_coarse(Level& L, std::string& err) {
  L.interior.clear();
  for (int64_t g = 0; g < L.ntot; ++g)
    if (!L.dir[g]) L.interior.push_back(g);
  const int ni = (int)L.interior.size();
  const int n = ni + 1;
  std::vector<int64_t> loc(L.ntot, -1);
  for (int q = 0; q < ni; ++q) loc[L.interior[q]] = q;
  std::vector<double> M((size_t)n * n, 0.0);
  for (int r = 0; r < ni; ++r) {
    int64_t g = L.interior[r];
    for (int64_t q = L.A.rowptr[g]; q < L.A.rowptr[g + 1]; ++q) {
      int64_t c = loc[L.A.col[q]];
      if (c >= 0) M[(size_t)r * n + c] = L.A.val[q];
    }
  }
  const double nv = 1.0 / std::sqrt((double)L.np);
  for (int r = 0; r < ni; ++r)
    if (L.interior[r] >= 2 * L.nv) {
      M[(size_t)r * n + ni] = nv;
      M[(size_t)ni * n + r] = nv;
    }
  if (!lu_factor(M, L.cpiv, n)) { err = "singular coarse matrix"; return false; }
  L.clu = std::move(M);
  L.cn = n;
  return true;
}
void coarse_solve(const Level& L, const double* b, double* x) {
  std::vector<double> rhs(L.cn, 0.0);
  const int ni = L.cn - 1;
  for (int q = 0; q < ni; ++q) rhs[q] = b[L.interior[q]];
  lu_solve(L.clu, L.cpiv, L.cn, rhs.data());
  std::fill(x, x + L.ntot, 0.0);
  for (int q = 0; q < ni; ++q) x[L.interior[q]] = rhs[q];
}

// --------------------------------------------------------------------------
// V-cycle, alg:mg, V(nu1, nu2); x is in/out on level l.
// --------------------------------------------------------------------------
void mg(const Ctx& c, int l, const double* b, double* x) {
  const Level& L = c.lev[l];
  if (l == 0) {  // only reached when the hierarchy has a single level
    if (c.coarse_mode == 0) coarse_solve(L, b, x);
    else {
      std::vector<double> t(L.ntot);
      for (int s = 0; s < 3; ++s) { relax(c, L, x, b, t.data()); std::copy(t.begin(), t.end(), x); }
    }
    return;
  }
  std::vector<double> t(L.ntot), r(L.ntot);
  for (int s = 0; s < c.nu1; ++s) {  // "Relax on u_l and p_l"
    relax(c, L, x, b, t.data());
    std::copy(t.begin(), t.end(), x);
  }
  residual(L, x, b, r.data());  // "Compute residual"
  const Level& C = c.lev[l - 1];
  std::vector<double> rc(C.ntot), ec(C.ntot, 0.0);
  restrict_(C, L, r.data(), rc.data());  // "Restriction"
  if (l == 1) {
    if (c.coarse_mode == 0) coarse_solve(C, rc.data(), ec.data());  // "e_0 = A_0^{-1} r_0"
    else {
      std::vector<double> t0(C.ntot);
      for (int s = 0; s < 3; ++s) { relax(c, C, ec.data(), rc.data(), t0.data()); ec = t0; }
    }
  } else {
    mg(c, l - 1, rc.data(), ec.data());  // "MG(A_{l-1}, 0, 0, r_{u,l-1}, r_{p,l-1}, l-1)"
  }
  prolong_add(L, ec.data(), x);  // "Correction"
  for (int s = 0; s < c.nu2; ++s) {  // "Relax on u_l and p_l"
    relax(c, L, x, b, t.data());
    std::copy(t.begin(), t.end(), x);
  }
}

// --------------------------------------------------------------------------
// Block-triangular preconditioner (alg:bt) for the comparison of
// the upper block-triangular system [[L, B^T],[0, -M]] (d_u, d_p) = r
// with M the Q1 pressure mass matrix (Shat ~ -M), each block inverted
// approximately by multigrid V-cycles with weighted-Jacobi smoothing (P:647-649:
// 3 V(3,3) cycles per block, Jacobi weights 0.6 (pressure) and 1.0 (velocity)).
// Block "part" 0 = the velocity block of the interior system (both components;
// corrections vanish on Dirichlet DOFs), part 1 = M.  Vectors are full-length; the other part is 0.
// --------------------------------------------------------------------------
void assemble_mass(Level& L) {
  const int N = L.N;
  const double h = L.h;
  double Me[4][4] = {{0}};
  for (int qx = 0; qx < 3; ++qx)
    for (int qy = 0; qy < 3; ++qy) {
      const double t = kGP[qx], sy = kGP[qy], w = kGW[qx] * kGW[qy] * h * h;
      double phi[4];
      for (int d = 0; d < 2; ++d)
        for (int c = 0; c < 2; ++c) phi[d * 2 + c] = q1(c, t) * q1(d, sy);
      for (int a = 0; a < 4; ++a)
        for (int b = 0; b < 4; ++b) Me[a][b] += w * phi[a] * phi[b];
    }
  std::vector<std::map<int32_t, double>> rows(L.np);
  for (int ey = 0; ey < N; ++ey)
    for (int ex = 0; ex < N; ++ex) {
      int64_t pi[4];
      for (int d = 0; d < 2; ++d)
        for (int c = 0; c < 2; ++c) pi[d * 2 + c] = (int64_t)(ey + d) * L.npn + ex + c;
      for (int a = 0; a < 4; ++a)
        for (int b = 0; b < 4; ++b) rows[pi[a]][(int32_t)pi[b]] += Me[a][b];
    }
  L.Mp = Csr();
  L.Mp.nrows = L.np;
  L.Mp.rowptr.assign(L.np + 1, 0);
  for (int64_t k = 0; k < L.np; ++k) {
    for (auto& kv : rows[k]) {
      L.Mp.col.push_back(kv.first);
      L.Mp.val.push_back(kv.second);
    }
    L.Mp.rowptr[k + 1] = (int64_t)L.Mp.col.size();
  }
}
// r = b - A_part x on the part's range (velocity: 0 on Dirichlet rows)
void blk_residual(const Level& L, int part, const double* x, const double* b, double* r) {
  const int64_t nvel = 2 * L.nv;
  if (part == 0) {
#pragma omp parallel for schedule(static)
    for (int64_t q = 0; q < nvel; ++q) {
      double s = b[q];
      for (int64_t k = L.A.rowptr[q]; k < L.A.rowptr[q + 1]; ++k)
        if (L.A.col[k] < nvel) s -= L.A.val[k] * x[L.A.col[k]];
      r[q] = L.dir[q] ? 0.0 : s;
    }
  } else {
#pragma omp parallel for schedule(static)
    for (int64_t k = 0; k < L.np; ++k) {
      double s = b[nvel + k];
      for (int64_t q = L.Mp.rowptr[k]; q < L.Mp.rowptr[k + 1]; ++q) s -= L.Mp.val[q] * x[nvel + L.Mp.col[q]];
      r[nvel + k] = s;
    }
  }
}
double blk_diag(const Level& L, int part, int64_t g) {
  const int64_t nvel = 2 * L.nv;
  if (part == 0) {
    for (int64_t k = L.A.rowptr[g]; k < L.A.rowptr[g + 1]; ++k)
      if (L.A.col[k] == g) return L.A.val[k];
    return 1.0;
  }
  for (int64_t q = L.Mp.rowptr[g - nvel]; q < L.Mp.rowptr[g - nvel + 1]; ++q)
    if (L.Mp.col[q] == g - nvel) return L.Mp.val[q];
  return 1.0;
}
// one weighted-Jacobi sweep x <- x + omega D^{-1} (b - A_part x)
void blk_jacobi(const Level& L, int part, double omega, double* x, const double* b) {
  std::vector<double> r(L.ntot, 0.0);
  blk_residual(L, part, x, b, r.data());
  const int64_t lo = part == 0 ? 0 : 2 * L.nv, hi = part == 0 ? 2 * L.nv : L.ntot;
  for (int64_t g = lo; g < hi; ++g) x[g] += omega * r[g] / blk_diag(L, part, g);
}
bool build_block_coarse(Level& L, std::string& err) {
  const int64_t nvel = 2 * L.nv;
  // the interior velocity system: identity rows at Dirichlet DOFs, Dirichlet columns dropped
  L.lu_u.assign((size_t)nvel * nvel, 0.0);
  for (int64_t r = 0; r < nvel; ++r) {
    if (L.dir[r]) {
      L.lu_u[(size_t)r * nvel + r] = 1.0;
      continue;
    }
    for (int64_t k = L.A.rowptr[r]; k < L.A.rowptr[r + 1]; ++k)
      if (L.A.col[k] < nvel && !L.dir[L.A.col[k]]) L.lu_u[(size_t)r * nvel + L.A.col[k]] = L.A.val[k];
  }
  L.lu_m.assign((size_t)L.np * L.np, 0.0);
  for (int64_t r = 0; r < L.np; ++r)
    for (int64_t q = L.Mp.rowptr[r]; q < L.Mp.rowptr[r + 1]; ++q) L.lu_m[(size_t)r * L.np + L.Mp.col[q]] = L.Mp.val[q];
  if (!lu_factor(L.lu_u, L.piv_u, (int)nvel) || !lu_factor(L.lu_m, L.piv_m, (int)L.np)) {
    err = "singular block on level 0";
    return false;
  }
  return true;
}
// scalar V(nu, nu) cycle (alg:mg with a Jacobi smoother) for block `part` on level l
void blk_mg(const Ctx& c, int l, int part, const double* b, double* x) {
  const Level& L = c.lev[l];
  const int64_t nvel = 2 * L.nv;
  const int64_t lo = part == 0 ? 0 : nvel, hi = part == 0 ? nvel : L.ntot;
  if (l == 0) {
    std::vector<double> v(b + lo, b + hi);
    if (part == 0) lu_solve(L.lu_u, L.piv_u, (int)nvel, v.data());
    else lu_solve(L.lu_m, L.piv_m, (int)L.np, v.data());
    std::copy(v.begin(), v.end(), x + lo);
    return;
  }
  const double w = part == 0 ? c.bt_omega_u : c.bt_omega_p;
  for (int s = 0; s < c.bt_nu; ++s) blk_jacobi(L, part, w, x, b);
  std::vector<double> r(L.ntot, 0.0);
  blk_residual(L, part, x, b, r.data());
  const Level& C = c.lev[l - 1];
  std::vector<double> rc(C.ntot), ec(C.ntot, 0.0);
  restrict_(C, L, r.data(), rc.data());
  blk_mg(c, l - 1, part, rc.data(), ec.data());
  prolong_add(L, ec.data(), x);
  for (int s = 0; s < c.bt_nu; ++s) blk_jacobi(L, part, w, x, b);
}
// z = BT(r): alg:bt lines 1-2 (the updates of lines 3-4 are z itself)
void bt_apply(const Ctx& c, const double* r, double* z) {
  const Level& L = c.lev.back();
  const int l = (int)c.lev.size() - 1;
  const int64_t nvel = 2 * L.nv;
  std::vector<double> rhs(L.ntot, 0.0);
  std::fill(z, z + L.ntot, 0.0);
  for (int64_t k = 0; k < L.np; ++k) rhs[nvel + k] = -r[nvel + k];       // M dp = -r_p
  for (int it = 0; it < c.bt_cycles; ++it) blk_mg(c, l, 1, rhs.data(), z);
  std::vector<double> btdp(nvel);
  apply_BT(L, z + nvel, btdp.data());
  for (int64_t j = 0; j < nvel; ++j) rhs[j] = L.dir[j] ? 0.0 : r[j] - btdp[j];  // L du = r_u - B^T dp
  for (int64_t k = 0; k < L.np; ++k) rhs[nvel + k] = 0.0;
  for (int it = 0; it < c.bt_cycles; ++it) blk_mg(c, l, 0, rhs.data(), z);
}
// FGMRES preconditioner z = M r
void precond_apply(const Ctx& c, const double* r, double* z) {
  if (c.precond == 1) bt_apply(c, r, z);
  else {
    std::fill(z, z + c.lev.back().ntot, 0.0);
    mg(c, (int)c.lev.size() - 1, r, z);
  }
}

// deterministic blocked dot product (fixed 4096-element blocks)
double dot(const double* a, const double* b, int64_t n) {
  const int64_t B = 4096;
  int64_t nb = (n + B - 1) / B;
  std::vector<double> part(nb, 0.0);
#pragma omp parallel for schedule(static)
  for (int64_t k = 0; k < nb; ++k) {
    double s = 0;
    for (int64_t q = k * B; q < std::min(n, (k + 1) * B); ++q) s += a[q] * b[q];
    part[k] = s;
  }
  double s = 0;
  for (double v : part) s += v;
  return s;
}

}  // namespace

// =============================================================================
// extern "C" surface used by oracle/__init__.py (ctypes)
// =============================================================================
extern "C" {

void* orc_create(int n_elem, int n_coarse, double nu, double omega, int weighting, int nu1, int nu2,
                 int coarse_mode) {
  if (n_elem < 1 || n_coarse < 1 || n_elem < n_coarse) return nullptr;
  int nl = 1;
  for (int n = n_elem; n > n_coarse; n /= 2) {
    if (n % 2) return nullptr;
    nl++;
  }
  if ((n_elem >> (nl - 1)) != n_coarse) return nullptr;
  Ctx* c = new Ctx;
  c->nu = nu;
  c->omega = omega;
  c->weighting = weighting;
  c->nu1 = nu1;
  c->nu2 = nu2;
  c->coarse_mode = coarse_mode;
  c->lev.resize(nl);
  for (int l = 0; l < nl; ++l) {
    Level& L = c->lev[l];
    L.N = n_coarse << l;
    L.h = 1.0 / L.N;
    L.nlat = 2 * L.N + 1;
    L.nv = L.nlat * L.nlat;
    L.npn = L.N + 1;
    L.np = L.npn * L.npn;
    L.ntot = 2 * L.nv + L.np;
    assemble(L, nu);
    if (!build_patches(L, omega, weighting, c->err)) { delete c; return nullptr; }
    if (l > 0) build_prolongation(c->lev[l - 1], L);
  }
  if (!build_coarse(c->lev[0], c->err)) { delete c; return nullptr; }
  return c;
}
// Select the V-cycle relaxation (0 Vanka, 1 Braess-Sarazin, 2 Schur-Uzawa) and
// its parameters; builds D^{-1} and S on every level.  Returns 0 on success.
int orc_set_relax(void* h, int kind, double t, double omega_r, double omega_j, int nj) {
  Ctx* c = (Ctx*)h;
  if (kind < 0 || kind > 2 || t <= 0 || nj < 0) return 1;
  c->relax = kind;
  c->t = t;
  c->omega_r = omega_r;
  c->omega_j = omega_j;
  c->nj = nj;
  if (kind != 0)
    for (Level& L : c->lev) build_schur(L, t);
  return 0;
}
// one sweep of the configured relaxation on level l
void orc_relax_sweep(void* h, int l, const double* xin, const double* b, double* xout) {
  const Ctx& c = *(Ctx*)h;
  relax(c, c.lev[l], xin, b, xout);
}
// FGMRES preconditioner: 0 monolithic V-cycle, 1 block-triangular (alg:bt)
int orc_set_precond(void* h, int kind, int cycles, int nu, double omega_u, double omega_p) {
  Ctx* c = (Ctx*)h;
  if (kind < 0 || kind > 1 || cycles < 1 || nu < 0) return 1;
  c->precond = kind;
  c->bt_cycles = cycles;
  c->bt_nu = nu;
  c->bt_omega_u = omega_u;
  c->bt_omega_p = omega_p;
  if (kind == 1) {
    for (Level& L : c->lev) assemble_mass(L);
    if (!build_block_coarse(c->lev[0], c->err)) return 2;
  }
  return 0;
}
void orc_precond_apply(void* h, const double* r, double* z) { precond_apply(*(Ctx*)h, r, z); }
int64_t orc_mass_nnz(void* h, int l) { return (int64_t)((Ctx*)h)->lev[l].Mp.col.size(); }
void orc_mass_csr(void* h, int l, int64_t* rowptr, int32_t* col, double* val) {
  const Csr& M = ((Ctx*)h)->lev[l].Mp;
  std::copy(M.rowptr.begin(), M.rowptr.end(), rowptr);
  std::copy(M.col.begin(), M.col.end(), col);
  std::copy(M.val.begin(), M.val.end(), val);
}
int64_t orc_schur_nnz(void* h, int l) { return (int64_t)((Ctx*)h)->lev[l].S.col.size(); }
void orc_schur_csr(void* h, int l, int64_t* rowptr, int32_t* col, double* val) {
  const Csr& S = ((Ctx*)h)->lev[l].S;
  std::copy(S.rowptr.begin(), S.rowptr.end(), rowptr);
  std::copy(S.col.begin(), S.col.end(), col);
  std::copy(S.val.begin(), S.val.end(), val);
}
void orc_destroy(void* h) { delete (Ctx*)h; }
int orc_num_levels(void* h) { return (int)((Ctx*)h)->lev.size(); }
int64_t orc_level_len(void* h, int l) { return ((Ctx*)h)->lev[l].ntot; }
int orc_level_n(void* h, int l) { return ((Ctx*)h)->lev[l].N; }
int orc_num_groups(void* h, int l) { return (int)((Ctx*)h)->lev[l].glu.size(); }
int64_t orc_nnz(void* h, int l) { return (int64_t)((Ctx*)h)->lev[l].A.col.size(); }
int orc_max_threads() {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}

// export the full assembled CSR (before Dirichlet masking)
void orc_csr(void* h, int l, int64_t* rowptr, int32_t* col, double* val) {
  const Csr& A = ((Ctx*)h)->lev[l].A;
  std::memcpy(rowptr, A.rowptr.data(), A.rowptr.size() * sizeof(int64_t));
  std::memcpy(col, A.col.data(), A.col.size() * sizeof(int32_t));
  std::memcpy(val, A.val.data(), A.val.size() * sizeof(double));
}
void orc_dirichlet(void* h, int l, uint8_t* out) {
  const Level& L = ((Ctx*)h)->lev[l];
  std::memcpy(out, L.dir.data(), L.ntot);
}
void orc_weights(void* h, int l, double* out) {
  const Level& L = ((Ctx*)h)->lev[l];
  std::memcpy(out, L.weight.data(), L.ntot * sizeof(double));
}
// patch (kx,ky): n dofs (<=51), global dof list, group id
int orc_patch(void* h, int l, int kx, int ky, int64_t* dofs) {
  const Level& L = ((Ctx*)h)->lev[l];
  int64_t p = (int64_t)ky * (L.N + 1) + kx;
  int64_t s = L.pstart[p], e = L.pstart[p + 1];
  for (int64_t q = s; q < e; ++q) dofs[q - s] = L.pdof[q];
  return (int)(e - s);
}
int orc_patch_group(void* h, int l, int kx, int ky) {
  const Level& L = ((Ctx*)h)->lev[l];
  return L.pgroup[(int64_t)ky * (L.N + 1) + kx];
}
int64_t orc_total_patch_dofs(void* h, int l) { return (int64_t)((Ctx*)h)->lev[l].pdof.size(); }

// problem data on level l (kind: 0 ZERO, 1 MMS_PAPER, 2 MMS_INSPACE, 3 CAVITY)
// b: velocity = (f, psi_i) by quadrature (boundary rows hold the boundary value,
//    they are masked anyway), pressure = 0 (eq:stokesmatrix right side [f; 0]).
// x0: boundary velocity values, zero elsewhere (reading 10).
void orc_problem(void* h, int l, int kind, double* b, double* x0) {
  const Ctx& c = *(Ctx*)h;
  const Level& L = c.lev[l];
  const int N = L.N;
  const double hh = L.h;
  std::fill(b, b + L.ntot, 0.0);
  std::fill(x0, x0 + L.ntot, 0.0);
  for (int ey = 0; ey < N; ++ey)
    for (int ex = 0; ex < N; ++ex)
      for (int qx = 0; qx < 3; ++qx)
        for (int qy = 0; qy < 3; ++qy) {
          double t = kGP[qx], s = kGP[qy], w = kGW[qx] * kGW[qy] * hh * hh;
          double x = (ex + t) * hh, y = (ey + s) * hh, fx, fy;
          forcing(kind, c.nu, x, y, &fx, &fy);
          for (int bb = 0; bb < 3; ++bb)
            for (int a = 0; a < 3; ++a) {
              double psi = q2(a, t) * q2(bb, s);
              int64_t g = (int64_t)(2 * ey + bb) * L.nlat + 2 * ex + a;
              b[g] += w * fx * psi;
              b[L.nv + g] += w * fy * psi;
            }
        }
  for (int64_t j = 0; j < L.nlat; ++j)
    for (int64_t i = 0; i < L.nlat; ++i) {
      int64_t g = j * L.nlat + i;
      if (!L.dir[g]) continue;
      double x = i * hh / 2, y = j * hh / 2, ux, uy;
      if (kind == 3) {  // lid-driven cavity (reading 15): u = (1,0) on the lid, 0 < x < 1
        ux = (j == L.nlat - 1 && i > 0 && i < L.nlat - 1) ? 1.0 : 0.0;
        uy = 0.0;
      } else {
        exact_u(kind, x, y, &ux, &uy);
      }
      x0[g] = ux;
      x0[L.nv + g] = uy;
      b[g] = ux;
      b[L.nv + g] = uy;
    }
}
// exact nodal values of the manufactured solution (for the exactness pins)
void orc_exact(void* h, int l, int kind, double* out) {
  const Level& L = ((Ctx*)h)->lev[l];
  for (int64_t j = 0; j < L.nlat; ++j)
    for (int64_t i = 0; i < L.nlat; ++i) {
      double ux, uy;
      exact_u(kind, i * L.h / 2, j * L.h / 2, &ux, &uy);
      out[j * L.nlat + i] = ux;
      out[L.nv + j * L.nlat + i] = uy;
    }
  for (int64_t ky = 0; ky < L.npn; ++ky)
    for (int64_t kx = 0; kx < L.npn; ++kx) exact_p(kind, kx * L.h, ky * L.h, &out[2 * L.nv + ky * L.npn + kx]);
}

void orc_matvec(void* h, int l, const double* x, double* y) { matvec_masked(((Ctx*)h)->lev[l], x, y); }
void orc_residual(void* h, int l, const double* x, const double* b, double* r) {
  residual(((Ctx*)h)->lev[l], x, b, r);
}
void orc_vanka_sweep(void* h, int l, const double* xin, const double* b, double* xout) {
  vanka_sweep(((Ctx*)h)->lev[l], xin, b, xout);
}
// level l is the FINE level (l >= 1)
void orc_restrict(void* h, int l, const double* rf, double* rc) {
  const Ctx& c = *(Ctx*)h;
  restrict_(c.lev[l - 1], c.lev[l], rf, rc);
}
void orc_prolong_add(void* h, int l, const double* ec, double* xf) { prolong_add(((Ctx*)h)->lev[l], ec, xf); }
void orc_prolongation_csr(void* h, int l, int64_t* rowptr, int32_t* col, double* val) {
  const Csr& P = ((Ctx*)h)->lev[l].P;
  std::memcpy(rowptr, P.rowptr.data(), P.rowptr.size() * sizeof(int64_t));
  std::memcpy(col, P.col.data(), P.col.size() * sizeof(int32_t));
  std::memcpy(val, P.val.data(), P.val.size() * sizeof(double));
}
int64_t orc_prolongation_nnz(void* h, int l) { return (int64_t)((Ctx*)h)->lev[l].P.col.size(); }
void orc_coarse_solve(void* h, const double* b, double* x) { coarse_solve(((Ctx*)h)->lev[0], b, x); }
// one V-cycle on the finest level: x in/out
void orc_vcycle(void* h, const double* b, double* x) {
  const Ctx& c = *(Ctx*)h;
  mg(c, (int)c.lev.size() - 1, b, x);
}

// Right-preconditioned flexible GMRES: Arnoldi with modified
// Gram-Schmidt, Givens rotations, no restart; the preconditioner is one V-cycle
// started from zero.  x is in (x0) / out.  hist[0..its] = |g_{k}|/beta (the
// GMRES residual estimate, = the true relative residual in exact arithmetic).
// returns iterations; *true_rel = ||b - A x|| / ||b - A x0|| recomputed.
// status: 0 converged, 1 not converged, 2 non-finite.
int orc_fgmres(void* h, const double* b, double* x, double rtol, int maxit, double* hist, double* true_rel,
               int* status) {
  const Ctx& c = *(Ctx*)h;
  const Level& L = c.lev.back();
  const int64_t n = L.ntot;
  std::vector<double> r(n);
  residual(L, x, b, r.data());
  double beta = std::sqrt(dot(r.data(), r.data(), n));
  hist[0] = 1.0;
  *status = 0;
  *true_rel = 0.0;
  if (beta == 0.0) return 0;
  std::vector<std::vector<double>> V, Z;
  V.emplace_back(n);
  for (int64_t q = 0; q < n; ++q) V[0][q] = r[q] / beta;
  std::vector<std::vector<double>> H(maxit + 1, std::vector<double>(maxit, 0.0));
  std::vector<double> cs(maxit), sn(maxit), g(maxit + 1, 0.0);
  g[0] = beta;
  int k = 0;
  bool conv = false;
  for (int j = 0; j < maxit; ++j) {
    Z.emplace_back(n, 0.0);
    precond_apply(c, V[j].data(), Z[j].data());              // z_j = M v_j
    std::vector<double> w(n);
    matvec_masked(L, Z[j].data(), w.data());                  // w = A z_j
    for (int i = 0; i <= j; ++i) {                            // modified Gram-Schmidt
      H[i][j] = dot(w.data(), V[i].data(), n);
      for (int64_t q = 0; q < n; ++q) w[q] -= H[i][j] * V[i][q];
    }
    H[j + 1][j] = std::sqrt(dot(w.data(), w.data(), n));
    if (!std::isfinite(H[j + 1][j])) { *status = 2; return j; }
    for (int i = 0; i < j; ++i) {  // previous rotations
      double t = cs[i] * H[i][j] + sn[i] * H[i + 1][j];
      H[i + 1][j] = -sn[i] * H[i][j] + cs[i] * H[i + 1][j];
      H[i][j] = t;
    }
    double a = H[j][j], bb = H[j + 1][j], rr = std::hypot(a, bb);
    cs[j] = a / rr;
    sn[j] = bb / rr;
    H[j][j] = rr;
    H[j + 1][j] = 0.0;
    g[j + 1] = -sn[j] * g[j];
    g[j] = cs[j] * g[j];
    hist[j + 1] = std::fabs(g[j + 1]) / beta;
    k = j + 1;
    double hn = bb;
    if (hist[j + 1] <= rtol || hn == 0.0) { conv = true; break; }
    V.emplace_back(n);
    for (int64_t q = 0; q < n; ++q) V[j + 1][q] = w[q] / hn;
  }
  // y = R^{-1} g ; x = x0 + Z y
  std::vector<double> y(k);
  for (int i = k - 1; i >= 0; --i) {
    double s = g[i];
    for (int m = i + 1; m < k; ++m) s -= H[i][m] * y[m];
    y[i] = s / H[i][i];
  }
  for (int i = 0; i < k; ++i)
    for (int64_t q = 0; q < n; ++q) x[q] += y[i] * Z[i][q];
  residual(L, x, b, r.data());
  *true_rel = std::sqrt(dot(r.data(), r.data(), n)) / beta;
  if (!std::isfinite(*true_rel)) *status = 2;
  else if (!conv) *status = 1;
  return k;
}

}  // extern "C"

// ----------------------------------------------------------------------------
// Sampled evaluation at full size (no global assembly): for a level with N
// elements per side, compute the Vanka-sweep output or the residual at a list of
// DOFs, assembling only the elements around the patches involved.  Same
// quadrature, same sign and BC readings, same dense LU and the same patch / weight
// definitions as the global path (a row of the operator is exact whenever all
// elements adjacent to its DOF are in the box).  x, b are compact full vectors.
// ----------------------------------------------------------------------------
namespace {
struct Box {  // elements [ex0,ex1) x [ey0,ey1) assembled into a dense local matrix
  int N;
  std::vector<int64_t> dofs;            // local -> global
  std::map<int64_t, int> loc;           // global -> local
  std::vector<double> A;                // dense, row-major
  int n() const { return (int)dofs.size(); }
};
void box_assemble(Box& B, int N, double nu, int ex0, int ex1, int ey0, int ey1) {
  const double h = 1.0 / N;
  const int64_t nlat = 2 * (int64_t)N + 1, nv = nlat * nlat, npn = N + 1;
  ex0 = std::max(ex0, 0); ey0 = std::max(ey0, 0); ex1 = std::min(ex1, N); ey1 = std::min(ey1, N);
  B.N = N;
  auto add = [&](int64_t g) {
    if (!B.loc.count(g)) { B.loc[g] = (int)B.dofs.size(); B.dofs.push_back(g); }
  };
  for (int ey = ey0; ey < ey1; ++ey)
    for (int ex = ex0; ex < ex1; ++ex) {
      for (int b = 0; b < 3; ++b)
        for (int a = 0; a < 3; ++a) {
          add((2 * ey + b) * nlat + 2 * ex + a);
          add(nv + (2 * ey + b) * nlat + 2 * ex + a);
        }
      for (int d = 0; d < 2; ++d)
        for (int c = 0; c < 2; ++c) add(2 * nv + (int64_t)(ey + d) * npn + ex + c);
    }
  const int n = B.n();
  B.A.assign((size_t)n * n, 0.0);
  // element matrices exactly as in assemble()
  double Le[9][9] = {{0}}, Bxe[4][9] = {{0}}, Bye[4][9] = {{0}};
  for (int qx = 0; qx < 3; ++qx)
    for (int qy = 0; qy < 3; ++qy) {
      double t = kGP[qx], s = kGP[qy], w = kGW[qx] * kGW[qy] * h * h;
      double dx[9], dy[9];
      for (int b = 0; b < 3; ++b)
        for (int a = 0; a < 3; ++a) {
          dx[b * 3 + a] = dq2(a, t) * q2(b, s) / h;
          dy[b * 3 + a] = q2(a, t) * dq2(b, s) / h;
        }
      for (int m = 0; m < 9; ++m)
        for (int n2 = 0; n2 < 9; ++n2) Le[m][n2] += nu * w * (dx[m] * dx[n2] + dy[m] * dy[n2]);
      for (int d = 0; d < 2; ++d)
        for (int c = 0; c < 2; ++c) {
          double phi = q1(c, t) * q1(d, s);
          for (int m = 0; m < 9; ++m) {
            Bxe[d * 2 + c][m] += -w * phi * dx[m];
            Bye[d * 2 + c][m] += -w * phi * dy[m];
          }
        }
    }
  for (int ey = ey0; ey < ey1; ++ey)
    for (int ex = ex0; ex < ex1; ++ex) {
      int vi[9], pi[4];
      for (int b = 0; b < 3; ++b)
        for (int a = 0; a < 3; ++a) vi[b * 3 + a] = B.loc[(2 * ey + b) * nlat + 2 * ex + a];
      int vj[9];
      for (int b = 0; b < 3; ++b)
        for (int a = 0; a < 3; ++a) vj[b * 3 + a] = B.loc[nv + (2 * ey + b) * nlat + 2 * ex + a];
      for (int d = 0; d < 2; ++d)
        for (int c = 0; c < 2; ++c) pi[d * 2 + c] = B.loc[2 * nv + (int64_t)(ey + d) * npn + ex + c];
      for (int m = 0; m < 9; ++m)
        for (int n2 = 0; n2 < 9; ++n2) {
          B.A[(size_t)vi[m] * n + vi[n2]] += Le[m][n2];
          B.A[(size_t)vj[m] * n + vj[n2]] += Le[m][n2];
        }
      for (int k = 0; k < 4; ++k)
        for (int m = 0; m < 9; ++m) {
          B.A[(size_t)pi[k] * n + vi[m]] += Bxe[k][m];
          B.A[(size_t)pi[k] * n + vj[m]] += Bye[k][m];
          B.A[(size_t)vi[m] * n + pi[k]] += Bxe[k][m];
          B.A[(size_t)vj[m] * n + pi[k]] += Bye[k][m];
        }
    }
}
bool is_dirichlet(int64_t g, int N) {
  const int64_t nlat = 2 * (int64_t)N + 1, nv = nlat * nlat;
  if (g >= 2 * nv) return false;
  const int64_t q = g % nv, i = q % nlat, j = q / nlat;
  return i == 0 || j == 0 || i == nlat - 1 || j == nlat - 1;
}
// the patch DOF list of node (kx,ky) exactly as in build_patches()
std::vector<int64_t> patch_dofs(int N, int kx, int ky) {
  const int64_t nlat = 2 * (int64_t)N + 1, nv = nlat * nlat;
  std::vector<int64_t> d;
  for (int comp = 0; comp < 2; ++comp)
    for (int64_t j = 2 * ky - 2; j <= 2 * ky + 2; ++j)
      for (int64_t i = 2 * kx - 2; i <= 2 * kx + 2; ++i) {
        if (i < 0 || j < 0 || i >= nlat || j >= nlat) continue;
        int64_t g = comp * nv + j * nlat + i;
        if (!is_dirichlet(g, N)) d.push_back(g);
      }
  d.push_back(2 * nv + (int64_t)ky * (N + 1) + kx);
  return d;
}
// patches (kx,ky) whose DOF list contains g
std::vector<std::pair<int, int>> patches_of(int64_t g, int N) {
  const int64_t nlat = 2 * (int64_t)N + 1, nv = nlat * nlat;
  std::vector<std::pair<int, int>> out;
  if (g >= 2 * nv) {
    const int64_t q = g - 2 * nv;
    out.push_back({(int)(q % (N + 1)), (int)(q / (N + 1))});
    return out;
  }
  if (is_dirichlet(g, N)) return out;
  const int64_t q = g % nv, i = q % nlat, j = q / nlat;
  // every node k with |2k - lattice index| <= 2 (candidates j/2-1 .. j/2+1)
  for (int64_t ky = std::max<int64_t>(0, j / 2 - 1); ky <= std::min<int64_t>(N, j / 2 + 1); ++ky)
    if (std::llabs(2 * ky - j) <= 2)
      for (int64_t kx = std::max<int64_t>(0, i / 2 - 1); kx <= std::min<int64_t>(N, i / 2 + 1); ++kx)
        if (std::llabs(2 * kx - i) <= 2) out.push_back({(int)kx, (int)ky});
  return out;
}
// residual of row g from the box (the box must hold all elements adjacent to g)
double box_residual(const Box& B, int64_t g, const double* x, const double* b) {
  if (is_dirichlet(g, B.N)) return 0.0;
  const int n = B.n();
  const int r = B.loc.at(g);
  double s = b[g];
  for (int c = 0; c < n; ++c) s -= B.A[(size_t)r * n + c] * x[B.dofs[c]];
  return s;
}
}  // namespace

extern "C" {
// out[q] = x_out at DOF idx[q] after one Vanka sweep from x (alg:vk)
void orc_sweep_sample(int N, double nu, double omega, int weighting, const double* x, const double* b,
                      const int64_t* idx, int64_t count, double* out) {
#pragma omp parallel for schedule(dynamic, 1)
  for (int64_t q = 0; q < count; ++q) {
    const int64_t g = idx[q];
    double acc = 0.0;
    const auto pats = patches_of(g, N);
    for (auto [kx, ky] : pats) {
      Box B;
      box_assemble(B, N, nu, kx - 2, kx + 2, ky - 2, ky + 2);
      const std::vector<int64_t> d = patch_dofs(N, kx, ky);
      const int m = (int)d.size();
      std::vector<double> Ai((size_t)m * m), rhs(m);
      for (int r2 = 0; r2 < m; ++r2) {
        for (int c = 0; c < m; ++c) Ai[(size_t)r2 * m + c] = B.A[(size_t)B.loc.at(d[r2]) * B.n() + B.loc.at(d[c])];
        rhs[r2] = box_residual(B, d[r2], x, b);
      }
      std::vector<int> piv;
      lu_factor(Ai, piv, m);
      lu_solve(Ai, piv, m, rhs.data());
      for (int r2 = 0; r2 < m; ++r2)
        if (d[r2] == g) acc += rhs[r2];
    }
    // W_i = omega diag(1/mult) (reading 6), mult = number of patches holding g
    double w = pats.empty() ? 0.0 : (weighting == 0 ? omega / (double)pats.size() : omega);
    out[q] = x[g] + w * acc;
  }
}
// out[q] = (b - A x) at DOF idx[q] (0 on Dirichlet rows)
void orc_residual_sample(int N, double nu, const double* x, const double* b, const int64_t* idx, int64_t count,
                         double* out) {
  const int64_t nlat = 2 * (int64_t)N + 1, nv = nlat * nlat;
#pragma omp parallel for schedule(dynamic, 16)
  for (int64_t q = 0; q < count; ++q) {
    const int64_t g = idx[q];
    int i, j;
    if (g >= 2 * nv) { i = 2 * (int)((g - 2 * nv) % (N + 1)); j = 2 * (int)((g - 2 * nv) / (N + 1)); }
    else { i = (int)((g % nv) % nlat); j = (int)((g % nv) / nlat); }
    Box B;
    box_assemble(B, N, nu, i / 2 - 1, i / 2 + 1, j / 2 - 1, j / 2 + 1);
    out[q] = box_residual(B, g, x, b);
  }
}

// Interpolation weights P[f, c] of build_prolongation() evaluated for one
// (fine DOF, coarse DOF) pair on a fine level with Nf elements: the coarse
// basis function of c at the fine DOF's point, 0 if c is not one of
// the 3x3 (Q2) / 2x2 (Q1) basis functions of the coarse element holding f.
double prolongation_weight(int Nf, int64_t f, int64_t c) {
  const int Nc = Nf / 2;
  const int64_t fl = 2 * (int64_t)Nf + 1, fv = fl * fl, cl = 2 * (int64_t)Nc + 1, cv = cl * cl;
  const bool fp = f >= 2 * fv, cp = c >= 2 * cv;
  if (fp != cp) return 0.0;
  if (!fp) {
    if (f / fv != c / cv) return 0.0;  // components
    const int64_t i = (f % fv) % fl, j = (f % fv) / fl, I = (c % cv) % cl, J = (c % cv) / cl;
    const int64_t ex = std::min<int64_t>(i / 4, Nc - 1), ey = std::min<int64_t>(j / 4, Nc - 1);
    const int64_t a = I - 2 * ex, bb = J - 2 * ey;
    if (a < 0 || a > 2 || bb < 0 || bb > 2) return 0.0;
    const double t = (i - 4.0 * ex) / 4.0, sy = (j - 4.0 * ey) / 4.0;
    return q2((int)a, t) * q2((int)bb, sy);
  }
  const int64_t kx = (f - 2 * fv) % (Nf + 1), ky = (f - 2 * fv) / (Nf + 1);
  const int64_t KX = (c - 2 * cv) % (Nc + 1), KY = (c - 2 * cv) / (Nc + 1);
  const int64_t ex = std::min<int64_t>(kx / 2, Nc - 1), ey = std::min<int64_t>(ky / 2, Nc - 1);
  const int64_t cc = KX - ex, d = KY - ey;
  if (cc < 0 || cc > 1 || d < 0 || d > 1) return 0.0;
  return q1((int)cc, (kx - 2.0 * ex) / 2.0) * q1((int)d, (ky - 2.0 * ey) / 2.0);
}

// r_c[idx[q]] = (P^T (b - A x))[idx[q]] on the coarse level (Nf/2 elements) of a
// fine level with Nf elements, Dirichlet coarse rows 0 (alg:mg lines 3-4,
// reading 9): the fine residual at every fine DOF in the coarse basis
// function's support, from locally assembled element boxes, weighted by P.
void orc_restrict_residual_sample(int Nf, double nu, const double* x, const double* b, const int64_t* idx,
                                  int64_t count, double* out) {
  const int Nc = Nf / 2;
  const int64_t fl = 2 * (int64_t)Nf + 1, fv = fl * fl, cl = 2 * (int64_t)Nc + 1, cv = cl * cl;
#pragma omp parallel for schedule(dynamic, 4)
  for (int64_t q = 0; q < count; ++q) {
    const int64_t c = idx[q];
    if (is_dirichlet(c, Nc)) {
      out[q] = 0.0;
      continue;
    }
    std::vector<int64_t> fs;  // fine DOFs in the support, ascending
    if (c < 2 * cv) {
      const int64_t comp = c / cv, I = (c % cv) % cl, J = (c % cv) / cl;
      for (int64_t j = std::max<int64_t>(0, 2 * J - 4); j <= std::min<int64_t>(fl - 1, 2 * J + 4); ++j)
        for (int64_t i = std::max<int64_t>(0, 2 * I - 4); i <= std::min<int64_t>(fl - 1, 2 * I + 4); ++i)
          fs.push_back(comp * fv + j * fl + i);
    } else {
      const int64_t KX = (c - 2 * cv) % (Nc + 1), KY = (c - 2 * cv) / (Nc + 1);
      for (int64_t ky = std::max<int64_t>(0, 2 * KY - 2); ky <= std::min<int64_t>(Nf, 2 * KY + 2); ++ky)
        for (int64_t kx = std::max<int64_t>(0, 2 * KX - 2); kx <= std::min<int64_t>(Nf, 2 * KX + 2); ++kx)
          fs.push_back(2 * fv + ky * (Nf + 1) + kx);
    }
    double sum = 0.0;
    for (int64_t f : fs) {
      const double w = prolongation_weight(Nf, f, c);
      if (w == 0.0) continue;
      int i, j;
      if (f >= 2 * fv) { i = 2 * (int)((f - 2 * fv) % (Nf + 1)); j = 2 * (int)((f - 2 * fv) / (Nf + 1)); }
      else { i = (int)((f % fv) % fl); j = (int)((f % fv) / fl); }
      Box B;
      box_assemble(B, Nf, nu, i / 2 - 1, i / 2 + 1, j / 2 - 1, j / 2 + 1);
      sum += w * box_residual(B, f, x, b);
    }
    out[q] = sum;
  }
}

// out[q] = x_f + (P e_c) at fine DOF idx[q] (alg:mg "Correction"), Nf fine elements
void orc_prolong_sample(int Nf, const double* ec, const double* xf, const int64_t* idx, int64_t count,
                        double* out) {
  const int Nc = Nf / 2;
  const int64_t fl = 2 * (int64_t)Nf + 1, fv = fl * fl, cl = 2 * (int64_t)Nc + 1, cv = cl * cl;
#pragma omp parallel for schedule(static)
  for (int64_t q = 0; q < count; ++q) {
    const int64_t f = idx[q];
    double s = 0.0;
    if (f < 2 * fv) {  // the 3x3 Q2 basis functions of the coarse element holding f (b outer, a inner)
      const int64_t comp = f / fv, i = (f % fv) % fl, j = (f % fv) / fl;
      const int64_t ex = std::min<int64_t>(i / 4, Nc - 1), ey = std::min<int64_t>(j / 4, Nc - 1);
      for (int bb = 0; bb < 3; ++bb)
        for (int a = 0; a < 3; ++a) {
          const int64_t c = comp * cv + (2 * ey + bb) * cl + 2 * ex + a;
          const double w = prolongation_weight(Nf, f, c);
          if (w != 0.0) s += w * ec[c];
        }
    } else {
      const int64_t kx = (f - 2 * fv) % (Nf + 1), ky = (f - 2 * fv) / (Nf + 1);
      const int64_t ex = std::min<int64_t>(kx / 2, Nc - 1), ey = std::min<int64_t>(ky / 2, Nc - 1);
      for (int d = 0; d < 2; ++d)
        for (int cc = 0; cc < 2; ++cc) {
          const int64_t c = 2 * cv + (ey + d) * (Nc + 1) + ex + cc;
          const double w = prolongation_weight(Nf, f, c);
          if (w != 0.0) s += w * ec[c];
        }
    }
    out[q] = xf[f] + s;
  }
}
}  // extern "C"
