// stencil.cuh -- structured-stencil data of the Q2-Q1 Stokes operator for libsvk.
//
// The operator is stored the way P:129-138 ("Structured matrix representation")
// describes: no index arrays, every coefficient is a function of the lattice
// position class.  On a uniform grid it is even simpler than the paper's
// "array of arrays": all rows of one class share one stencil, so the whole
// operator is a few dozen doubles held in __constant__ memory.
//
// 1D element matrices on an element of width h (quadratic nodes 0, h/2, h;
// linear nodes 0, h), exact rationals:
//   h * K_e = (1/3)  [[7,-8,1],[-8,16,-8],[1,-8,7]]     K_e = int psi_a' psi_b'
//   M_e / h = (1/30) [[4,2,-1],[2,16,2],[-1,2,4]]       M_e = int psi_a psi_b
//   C_e / h = (1/6)  [[1,2,0],[0,2,1]]                  C_e = int phi_c psi_a
//   G_e     = (1/6)  [[-5,4,1],[-1,-4,5]]               G_e = int phi_c psi_a'
// and the 2D operator is their tensor product (Q2 = Q2(x) (x) Q2(y)):
//   L   = nu (M (x) K + K (x) M)  per velocity component  (h cancels)
//   B_x = -h C^ (x) G,  B_y = -h G (x) C^   (b(v,q) = -int q div v, reading 1)
// where (x) puts the y factor first (row index j*(2N+1)+i).
#pragma once
#include <cstdint>

namespace svk {

struct StencilConst {
  double Khat[3][3], Mhat[3][3], Chat[2][3], Ge[2][3];  // element matrices (scaled as above)
  // 1D rows of the assembled matrices at NON-Dirichlet lattice points, offsets -2..2:
  // [0] = even lattice index (element node), [1] = odd (element midpoint)
  double KR[2][5], MR[2][5];
  // 1D rows of the pressure-node matrices C^, G over the window [2k-2, 2k+2]:
  // [0] = node k = 0, [1] = interior node, [2] = node k = N
  double CR[3][5], GR[3][5];
  // 1D columns of C^, G at non-Dirichlet lattice points: even i = 2a touches
  // nodes a-1, a, a+1 ([0][0..2]); odd i = 2a+1 touches nodes a, a+1 ([1][0..1])
  double CC[2][3], GC[2][3];
  // the (unscaled) B rows at a pressure node of class (cy, cx) in {0,1,2}^2 over its 5x5
  // window, per component: PB[0] = C^R[cy] (x) GR[cx], PB[1] = GR[cy] (x) C^R[cx]
  // (B_x = -h PB[0], B_y = -h PB[1]); a table indexed by the node class so that the
  // boundary-node branch of the fused kernels holds no loop-invariant registers
  double PB[2][9][25];
};

// pitched vector layout of one level (see include/svk.h)
struct LevelGeom {
  int N;          // elements per side
  int lat;        // 2N+1
  int64_t pu;     // pitch of velocity rows (doubles)
  int64_t pp;     // pitch of pressure rows
  int64_t oux, ouy, op;  // plane offsets
  int64_t len;    // vector length
  double h;       // 1/N
  // row slab owned by this rank (node rows [r0, r1); lattice rows [2 r0, min(2 r1, lat))).
  // Single-GPU / replicated levels own everything: r0 = 0, r1 = N + 1.
  int r0, r1;
};

}  // namespace svk

// one copy for the whole module (single translation unit build)
__constant__ svk::StencilConst c_st;

namespace svk {

// --- general 1D assembled entries (element loops), used only by the setup
// kernels; valid for any pair of lattice / node indices including boundary rows.
__device__ __forceinline__ double k1(int i, int ip, int N) {  // h * K[i][ip]
  double s = 0.0;
  for (int e = max(0, (max(i, ip) - 2 + 1) / 2); e <= min(N - 1, min(i, ip) / 2); ++e) {
    int a = i - 2 * e, b = ip - 2 * e;
    if (a >= 0 && a <= 2 && b >= 0 && b <= 2) s += c_st.Khat[a][b];
  }
  return s;
}
__device__ __forceinline__ double m1(int i, int ip, int N) {  // M[i][ip] / h
  double s = 0.0;
  for (int e = max(0, (max(i, ip) - 2 + 1) / 2); e <= min(N - 1, min(i, ip) / 2); ++e) {
    int a = i - 2 * e, b = ip - 2 * e;
    if (a >= 0 && a <= 2 && b >= 0 && b <= 2) s += c_st.Mhat[a][b];
  }
  return s;
}
__device__ __forceinline__ double c1(int k, int i, int N) {  // C[k][i] / h
  double s = 0.0;
  for (int e = k - 1; e <= k; ++e) {
    if (e < 0 || e >= N) continue;
    int c = k - e, a = i - 2 * e;
    if (a >= 0 && a <= 2) s += c_st.Chat[c][a];
  }
  return s;
}
__device__ __forceinline__ double g1(int k, int i, int N) {  // G[k][i]
  double s = 0.0;
  for (int e = k - 1; e <= k; ++e) {
    if (e < 0 || e >= N) continue;
    int c = k - e, a = i - 2 * e;
    if (a >= 0 && a <= 2) s += c_st.Ge[c][a];
  }
  return s;
}

// DOF descriptor in plane coordinates: kind 0 = u_x, 1 = u_y (i,j lattice), 2 = p (i,j = kx,ky)
struct Dof {
  int kind, i, j;
};

// Entry A[row][col] of the assembled (unmasked) operator, from the 1D tables.
__device__ __forceinline__ double a_entry(Dof r, Dof c, int N, double nu, double h) {
  if (r.kind < 2 && c.kind < 2) {
    if (r.kind != c.kind) return 0.0;  // L is block diagonal over components
    if (abs(r.i - c.i) > 2 || abs(r.j - c.j) > 2) return 0.0;
    return nu * (m1(r.j, c.j, N) * k1(r.i, c.i, N) + k1(r.j, c.j, N) * m1(r.i, c.i, N));
  }
  if (r.kind == 2 && c.kind == 2) return 0.0;
  Dof v = r.kind == 2 ? c : r;  // velocity
  Dof p = r.kind == 2 ? r : c;  // pressure
  if (v.kind == 0) return -h * c1(p.j, v.j, N) * g1(p.i, v.i, N);  // B_x = -h C^ (x) G
  return -h * g1(p.j, v.j, N) * c1(p.i, v.i, N);                   // B_y = -h G (x) C^
}

__host__ __device__ __forceinline__ int pcat(int k, int N) {  // patch category per axis
  return k == 0 ? 0 : k == 1 ? 1 : k == N ? 4 : k == N - 1 ? 3 : 2;
}

}  // namespace svk
