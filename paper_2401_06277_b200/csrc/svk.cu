// svk.cu -- libsvk: C-ABI host side (hierarchy, V-cycle, FGMRES) and the single
// translation unit that includes every kernel.  See include/svk.h for the API
// contract and DESIGN.md for the design.
#include "../../include/svk.h"

#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <map>
#include <mutex>
#include <string>
#include <vector>

#include "stencil.cuh"
#include "kernels_common.cuh"
#include "krylov.cuh"
#include "sweep_fused.cuh"
#include "small_cycle.cuh"
#include "residual_strip.cuh"
#include "relax_bs.cuh"
#include "bt.cuh"
#include "dist.cuh"

using namespace svk;

struct svk_ctx {
  svk_config cfg{};
  int nlev = 0;
  std::vector<LevelGeom> g;
  int* d_Ns = nullptr;
  double* d_inv = nullptr;  // nlev * 25 padded 51x51 group inverses
  double* d_fac = nullptr;  // nlev * FusedFactors (structured factors for the fused sweep)
  std::vector<FusedFactors> h_fac;  // host copy, passed to the fused kernel by value (param space)
  int nsm = 148;
  // level 0 solve
  double* d_cmat = nullptr;
  int* d_cidx = nullptr;
  int cni = 0;
  // per-level workspaces
  std::vector<double*> ws_x, ws_t, ws_r, ws_b;
  double* d_dbuf = nullptr;  // packed patch buffer (unfused sweep), finest-level size
  std::vector<double*> d_inv_simple;  // SIMPLE: per level, every patch's inverse (slot-interleaved)
  double* d_bd = nullptr;    // boundary-patch corrections (fused sweep), finest-level size
  // coarse-level V-cycle in one cluster launch (small_cycle.cuh): levels 1 .. sc_top
  // (N <= SVK_SMALL_N, below the finest level, replicated), sc_cluster CTAs
  int sc_top = 0, sc_cluster = 0;
  double* d_sc = nullptr;  // patch corrections of the largest small level, slot-major
  std::vector<BdTile*> d_sc_tiles;  // per small level: every patch in tiles of one group
  std::vector<int> n_sc_tiles;
  std::vector<BdTile*> d_tiles;  // per level: boundary-patch tiles (k_boundary_patches)
  std::vector<int> ntiles;
  double* d_sw = nullptr;    // extra ping-pong vector for nsweeps > 1, finest-level size
  // Braess-Sarazin / Schur-Uzawa comparators (relax_bs.cuh)
  double* d_schur = nullptr;                 // nlev * kSchurStride class stencils of S
  std::vector<double*> p_rhs, p_dp0, p_dp1;  // per level, pressure-plane sized
  // block-triangular preconditioner (bt.cuh)
  double* d_btb = nullptr;                   // finest-level right-hand side
  double *d_bt_invL = nullptr, *d_bt_invM = nullptr;
  int *d_bt_idxL = nullptr, *d_bt_idxM = nullptr;
  int bt_niL = 0, bt_niM = 0;
  // Krylov
  std::vector<double*> V, Z;
  double* d_w = nullptr;
  double* d_r = nullptr;
  double* d_part = nullptr;
  double* d_coef = nullptr;
  double* h_pin = nullptr;
  double* h_pin_dev = nullptr;  // h_pin is mapped: the device address of the same memory
  int coef_cap = 0;
  double* d_hb = nullptr;  // e2e staging
  double* d_hx = nullptr;
  // svk_solve_host_batch: a second staging pair and two copy streams + events
  double* d_hb2 = nullptr;
  double* d_hx2 = nullptr;
  double* d_cin[2][2] = {{nullptr, nullptr}, {nullptr, nullptr}};  // compact staging: [pair][b, x0]
  double* d_cout[2] = {nullptr, nullptr};                          // compact staging of x
  cudaStream_t s_in = nullptr, s_out = nullptr;
  cudaEvent_t ev_in[2] = {nullptr, nullptr}, ev_solved[2] = {nullptr, nullptr}, ev_out[2] = {nullptr, nullptr};
  cudaEvent_t ev[6]{};
  int64_t launches = 0;
  // sweep profiling (svk_set_profiling / svk_sweep_stats)
  bool prof = false;
  std::vector<cudaEvent_t> prof_ev;  // pool, used in (start, stop) pairs
  size_t prof_used = 0;
  // CUDA graphs of the FGMRES preconditioner (one V-cycle from zero, alg:mg),
  // captured once per (input, output) basis-vector pair and replayed: the ~60
  // kernels of a cycle become one graph launch (programmatic edges kept).
  struct GraphRec {
    const double* in = nullptr;
    double* out = nullptr;
    bool prof = false;
    cudaGraphExec_t exec = nullptr;
    int64_t launches = 0;                                   // kernels in the graph
    std::vector<std::pair<cudaEvent_t, cudaEvent_t>> ev;   // timed finest-level sweeps
  };
  std::vector<std::unique_ptr<GraphRec>> graphs;
  GraphRec* capturing = nullptr;
  std::vector<GraphRec*> prof_pending;  // replayed graphs whose sweep events are not harvested yet
  cudaStream_t cap_stream = nullptr;
  int use_graphs = -1;                  // -1: decide at first use (SVK_GRAPHS=0 disables)
  double prof_acc_ms = 0.0;
  int64_t prof_acc_n = 0;
  // device memory the context holds (cudaMalloc'd bytes + physically mapped
  // bytes of slab-local vectors), svk_device_bytes
  double* d_agg = nullptr;  // agglomeration staging: nranks chunks of the coarse slab pieces
  int64_t agg_cap = 0;
  bool slab_local = true;  // distributed-level workspaces slab-local (SVK_SLAB_LOCAL=0: full size)
  int64_t dev_bytes = 0;
  std::map<const double*, int64_t> plain_bytes;  // cudaMalloc'd vectors -> bytes
  std::map<const double*, SlabMem> slab_mem;     // slab-local vectors (distributed levels)
  // multi-GPU row slabs (dist.cuh): levels la..nlev-1 are distributed
  std::unique_ptr<Transport> tr;
  int la = 1 << 30;
  double t_setup_s = 0.0;  // svk_create wall time (svk_report.t_setup_s)
  cudaEvent_t sweep_ev0 = nullptr;  // start event of the next timed sweep (op_sweep -> op_sweep_impl)
  unsigned sweep_ev0_flags = 0;
  bool poison = false;  // SVK_POISON_HALO=1: NaN-fill rows beyond the halo after each exchange (tests)
  std::string err;
};

namespace {

constexpr int kDotBlocks = 148 * 4;
constexpr double kReorthKappa = 10.0;  // ADAPTIVE orthogonalisation: re-orthogonalise if |w'| < |w| / kappa

std::mutex g_tab_mu;
bool g_tab_done[64] = {false};

int64_t round_up(int64_t a, int64_t m) { return (a + m - 1) / m * m; }

// first distributed level: the coarsest level l >= 1 with at least agglom_rows
// node rows per rank; Ns.size() if none
int first_dist_level(const std::vector<int>& Ns, int nranks, int agglom_rows) {
  for (int l = 1; l < (int)Ns.size(); ++l)
    if ((int64_t)Ns[l] >= (int64_t)agglom_rows * nranks) return l;
  return (int)Ns.size();
}

LevelGeom make_geom(int N) {
  LevelGeom g{};
  g.N = N;
  g.lat = 2 * N + 1;
  g.pu = round_up(g.lat, 8);
  g.pp = round_up(N + 1, 8);
  const int64_t plane = round_up((int64_t)g.lat * g.pu, 32);
  g.oux = 0;
  g.ouy = plane;
  g.op = 2 * plane;
  g.len = g.op + round_up((int64_t)(N + 1) * g.pp, 32);
  g.h = 1.0 / N;
  g.r0 = 0;
  g.r1 = N + 1;
  return g;
}

// Stencil tables from the exact 1D element matrices (stencil.cuh header).
// 1D global matrices are assembled on a small grid and their generic rows and
// columns read off; uniformity of every non-Dirichlet row/column is asserted.
bool build_tables(StencilConst& t, std::string& err) {
  const double K[3][3] = {{7, -8, 1}, {-8, 16, -8}, {1, -8, 7}};
  const double M[3][3] = {{4, 2, -1}, {2, 16, 2}, {-1, 2, 4}};
  const double Cm[2][3] = {{1, 2, 0}, {0, 2, 1}};
  const double G[2][3] = {{-5, 4, 1}, {-1, -4, 5}};
  std::memset(&t, 0, sizeof(t));
  for (int a = 0; a < 3; ++a)
    for (int b = 0; b < 3; ++b) {
      t.Khat[a][b] = K[a][b] / 3.0;
      t.Mhat[a][b] = M[a][b] / 30.0;
    }
  for (int c = 0; c < 2; ++c)
    for (int a = 0; a < 3; ++a) {
      t.Chat[c][a] = Cm[c][a] / 6.0;
      t.Ge[c][a] = G[c][a] / 6.0;
    }
  const int N = 8, lat = 2 * N + 1;
  std::vector<double> k1(lat * lat, 0), m1(lat * lat, 0), c1((N + 1) * lat, 0), g1((N + 1) * lat, 0);
  for (int e = 0; e < N; ++e)
    for (int a = 0; a < 3; ++a) {
      for (int b = 0; b < 3; ++b) {
        k1[(2 * e + a) * lat + 2 * e + b] += t.Khat[a][b];
        m1[(2 * e + a) * lat + 2 * e + b] += t.Mhat[a][b];
      }
      for (int c = 0; c < 2; ++c) {
        c1[(e + c) * lat + 2 * e + a] += t.Chat[c][a];
        g1[(e + c) * lat + 2 * e + a] += t.Ge[c][a];
      }
    }
  auto at = [&](const std::vector<double>& v, int r, int c, int ncol) {
    return (c < 0 || c >= ncol) ? 0.0 : v[r * ncol + c];
  };
  for (int i = 1; i < lat - 1; ++i) {
    const int par = i & 1;
    for (int o = -2; o <= 2; ++o) {
      const double kv = at(k1, i, i + o, lat), mv = at(m1, i, i + o, lat);
      if (i == 4 || i == 5) {
        t.KR[par][o + 2] = kv;
        t.MR[par][o + 2] = mv;
      } else if (kv != t.KR[par][o + 2] && i > 5) {
        err = "stencil rows not uniform";
        return false;
      }
    }
  }
  for (int k = 0; k <= N; ++k) {
    const int cls = k == 0 ? 0 : (k == N ? 2 : 1);
    for (int o = 0; o < 5; ++o) {
      t.CR[cls][o] = at(c1, k, 2 * k - 2 + o, lat);
      t.GR[cls][o] = at(g1, k, 2 * k - 2 + o, lat);
    }
  }
  for (int cy = 0; cy < 3; ++cy)
    for (int cx = 0; cx < 3; ++cx)
      for (int r = 0; r < 5; ++r)
        for (int o = 0; o < 5; ++o) {
          t.PB[0][cy * 3 + cx][r * 5 + o] = t.CR[cy][r] * t.GR[cx][o];
          t.PB[1][cy * 3 + cx][r * 5 + o] = t.GR[cy][r] * t.CR[cx][o];
        }
  // columns at non-Dirichlet lattice points (checked uniform)
  for (int i = 1; i < lat - 1; ++i) {
    const int par = i & 1;
    const int k0 = par ? (i - 1) / 2 : i / 2 - 1, nk = par ? 2 : 3;
    for (int q = 0; q < nk; ++q) {
      const double cv = c1[(k0 + q) * lat + i], gv = g1[(k0 + q) * lat + i];
      if (i <= 2) {
        t.CC[par][q] = cv;
        t.GC[par][q] = gv;
      } else if (cv != t.CC[par][q] || gv != t.GC[par][q]) {
        err = "stencil columns not uniform";
        return false;
      }
    }
  }
  // the fused sweep visits only the structurally non-zero taps; check them here
  const bool zeros_ok = t.KR[1][0] == 0 && t.KR[1][4] == 0 && t.MR[1][0] == 0 && t.MR[1][4] == 0 &&
                        t.CC[0][0] == 0 && t.CC[0][2] == 0 && t.GC[0][1] == 0 && t.CR[1][0] == 0 &&
                        t.CR[1][4] == 0 && t.GR[1][2] == 0;
  if (!zeros_ok) {
    err = "unexpected stencil sparsity";
    return false;
  }
  return true;
}

#define CK(call)                                                             \
  do {                                                                       \
    cudaError_t e_ = (call);                                                 \
    if (e_ != cudaSuccess) {                                                 \
      ctx->err = std::string(#call) + ": " + cudaGetErrorString(e_);        \
      return SVK_ERR_CUDA;                                                   \
    }                                                                        \
  } while (0)
#define CKL()                                                                \
  do {                                                                       \
    ctx->launches++;                                                         \
    cudaError_t e_ = cudaGetLastError();                                     \
    if (e_ != cudaSuccess) {                                                 \
      ctx->err = std::string("kernel launch: ") + cudaGetErrorString(e_);   \
      return SVK_ERR_CUDA;                                                   \
    }                                                                        \
  } while (0)
#define TRY(expr)                 \
  do {                            \
    int s_ = (expr);              \
    if (s_ < 0) return s_;        \
  } while (0)

dim3 plane_grid(const LevelGeom& g) {
  return dim3((unsigned)((g.pu + 31) / 32), (unsigned)((g.lat + 7) / 8), 3);
}
const dim3 kPlaneBlock(32, 8, 1);

int valid_level(svk_ctx* ctx, int level) {
  if (!ctx) return SVK_ERR_INVALID;
  if (level < 0 || level >= ctx->nlev) {
    ctx->err = "level out of range";
    return SVK_ERR_INVALID;
  }
  return SVK_OK;
}
int valid_ptr(svk_ctx* ctx, const void* p, const char* what) {
  if (!p || ((uintptr_t)p & 15u)) {
    ctx->err = std::string(what) + ": NULL or not 16-byte aligned";
    return SVK_ERR_INVALID;
  }
  return SVK_OK;
}

int alloc_vec(svk_ctx* ctx, double** p, int64_t n) {
  const int64_t bytes = n * (int64_t)sizeof(double);
  if (ctx->cfg.alloc_fn) {
    // caller's allocator (svk_config.alloc_fn): the block may have been in use on
    // any stream until now, so order the zero-fill after all of the device's work
    CK(cudaDeviceSynchronize());
    *p = (double*)ctx->cfg.alloc_fn(bytes, ctx->cfg.device, ctx->cfg.alloc_user);
    if (!*p || ((uintptr_t)*p & 255u)) {
      if (*p) ctx->cfg.free_fn(*p, bytes, ctx->cfg.device, ctx->cfg.alloc_user);
      *p = nullptr;
      ctx->err = "svk_config.alloc_fn returned NULL or a block not aligned to 256 bytes";
      return SVK_ERR_CUDA;
    }
  } else {
    CK(cudaMalloc(p, bytes));
  }
  CK(cudaMemset(*p, 0, bytes));
  ctx->dev_bytes += n * (int64_t)sizeof(double);
  ctx->plain_bytes[*p] = n * (int64_t)sizeof(double);
  return SVK_OK;
}
// release a vector from alloc_vec / alloc_level_vec
void free_vec(svk_ctx* ctx, double* p) {
  if (!p) return;
  auto it = ctx->slab_mem.find(p);
  if (it != ctx->slab_mem.end()) {
    ctx->dev_bytes -= it->second.mapped;
    slab_free(it->second);
    ctx->slab_mem.erase(it);
    return;
  }
  auto jt = ctx->plain_bytes.find(p);
  if (jt != ctx->plain_bytes.end()) {
    const int64_t bytes = jt->second;
    ctx->dev_bytes -= bytes;
    ctx->plain_bytes.erase(jt);
    if (ctx->cfg.free_fn) {
      ctx->cfg.free_fn(p, bytes, ctx->cfg.device, ctx->cfg.alloc_user);
      return;
    }
  }
  cudaFree(p);
}

// ------------------------------------------------------------------ level ops
// r = b - A x (b != NULL) or r = A x (b == NULL), streaming strip kernel
int op_residual(svk_ctx* ctx, int l, const double* x, const double* b, double* r, cudaStream_t s) {
  if (launch_residual_strip(ctx->g[l], nullptr, ctx->h_fac[l], x, b, r, ctx->nsm, s) != 0) {
    ctx->err = "residual: " + tma_error();
    return SVK_ERR_CUDA;
  }
  CKL();
  return SVK_OK;
}
// r_c = P^T (b - A x) on level l-1 in one pass (alg:mg lines 3-4)
// (coarse rows computed: the halves of this rank's fine slab, so that on the
// agglomeration level every coarse row is produced by exactly one rank)
int op_residual_restrict(svk_ctx* ctx, int l, const double* x, const double* b, double* rc, cudaStream_t s) {
  const LevelGeom& gf = ctx->g[l];
  LevelGeom gc = ctx->g[l - 1];
  gc.r0 = gf.r0 / 2;
  gc.r1 = gf.r1 == gf.N + 1 ? gc.N + 1 : gf.r1 / 2;
  if (launch_residual_strip(gf, &gc, ctx->h_fac[l], x, b, rc, ctx->nsm, s) != 0) {
    ctx->err = "residual+restrict: " + tma_error();
    return SVK_ERR_CUDA;
  }
  CKL();
  return SVK_OK;
}

// ------------------------------------------------------------ multi-GPU plumbing
constexpr int kHalo = 4;  // node rows of halo per side (2 kHalo lattice rows)

bool dist_level(const svk_ctx* ctx, int l) { return ctx->tr && l >= ctx->la; }

Block plane_rows(double* v, int64_t off, int64_t pitch, int a, int b) {
  return Block{v + off + (int64_t)a * pitch, (int64_t)std::max(0, b - a) * pitch};
}

// Rows of each plane a rank's kernels may touch on a distributed level: its
// slab plus the halo (kHalo node rows) and a margin of 2 node rows; lattice rows
// [ua, ub) of the velocity planes, node rows [pa, pb) of the pressure plane.
struct SlabRows {
  int ua, ub, pa, pb;
};
SlabRows slab_rows_touched(const LevelGeom& g) {
  const int m = kHalo + 2;
  return SlabRows{std::max(0, 2 * (g.r0 - m)), std::min(g.lat, 2 * (g.r1 + m)), std::max(0, g.r0 - m),
                  std::min(g.N + 1, g.r1 + m)};
}
// Slab-local vector of a distributed level: the full pitched
// layout is reserved as virtual address space, but device memory is mapped only
// for the rows the rank touches, so every kernel keeps global row indexing while
// a rank holds ~1/P of the vector (plus halos).  Replicated levels: alloc_vec.
int alloc_level_vec(svk_ctx* ctx, int l, double** p) {
  const LevelGeom& g = ctx->g[l];
  if (!dist_level(ctx, l) || !ctx->slab_local) return alloc_vec(ctx, p, g.len);
  const SlabRows R = slab_rows_touched(g);
  const int64_t b8 = (int64_t)sizeof(double);
  std::vector<std::pair<int64_t, int64_t>> ranges = {
      {(g.oux + (int64_t)R.ua * g.pu) * b8, (g.oux + (int64_t)R.ub * g.pu) * b8},
      {(g.ouy + (int64_t)R.ua * g.pu) * b8, (g.ouy + (int64_t)R.ub * g.pu) * b8},
      {(g.op + (int64_t)R.pa * g.pp) * b8, (g.op + (int64_t)R.pb * g.pp) * b8}};
  SlabMem m;
  std::string err;
  if (slab_alloc(ctx->cfg.device, g.len * b8, ranges, &m, err) != 0) {
    ctx->err = "slab-local vector: " + err;
    return SVK_ERR_ALLOC;
  }
  *p = reinterpret_cast<double*>(m.base);
  if (const char* e = std::getenv("SVK_DEBUG_SLAB"); e && e[0] == '1') {
    std::string rs;
    for (const auto& r : m.maps) rs += " [" + std::to_string(r.first) + "," + std::to_string(r.first + r.second) + ")";
    std::fprintf(stderr, "[slab-alloc] rank %d level N=%d rows %d..%d base %p reserved %zu maps%s\n", ctx->cfg.rank,
                 g.N, g.r0, g.r1, (void*)m.base, m.reserved, rs.c_str());
  }
  for (const auto& r : m.maps) CK(cudaMemset(reinterpret_cast<char*>(m.base) + r.first, 0, r.second));
  ctx->dev_bytes += m.mapped;
  ctx->slab_mem[*p] = m;
  return SVK_OK;
}
// the byte ranges of v that hold device memory (the whole vector unless slab-local)
std::vector<std::pair<int64_t, int64_t>> vec_ranges(const svk_ctx* ctx, const double* v, int64_t len) {
  auto it = ctx->slab_mem.find(v);
  if (it == ctx->slab_mem.end()) return {{0, len * (int64_t)sizeof(double)}};
  return it->second.maps;
}
// x = 0 / y = x over the memory both vectors hold on level l
int op_zero_level(svk_ctx* ctx, int l, double* x, cudaStream_t s) {
  for (const auto& r : vec_ranges(ctx, x, ctx->g[l].len))
    CK(cudaMemsetAsync(reinterpret_cast<char*>(x) + r.first, 0, r.second, s));
  return SVK_OK;
}
int op_copy_level(svk_ctx* ctx, int l, double* y, const double* x, cudaStream_t s) {
  const bool sy = ctx->slab_mem.count(y), sx = ctx->slab_mem.count(x);
  const auto ranges = vec_ranges(ctx, sy ? y : x, ctx->g[l].len);  // slab maps of one level are identical
  for (const auto& r : (sy || sx) ? ranges : vec_ranges(ctx, y, ctx->g[l].len))
    CK(cudaMemcpyAsync(reinterpret_cast<char*>(y) + r.first, reinterpret_cast<const char*>(x) + r.first, r.second,
                       cudaMemcpyDeviceToDevice, s));
  return SVK_OK;
}

// refresh the halo rows of v on level l from the neighbouring ranks
int op_halo(svk_ctx* ctx, int l, double* v, cudaStream_t s) {
  if (!dist_level(ctx, l)) return SVK_OK;
  const LevelGeom& g = ctx->g[l];
  const int rank = ctx->cfg.rank, P = ctx->cfg.nranks, lat = g.lat, np = g.N + 1;
  const int lo = g.r0, hi = g.r1, H = kHalo;
  std::vector<Block> ls, lr, hs, hr;
  auto add = [&](std::vector<Block>& dst, int ua, int ub, int pa, int pb) {
    dst.push_back(plane_rows(v, g.oux, g.pu, ua, ub));
    dst.push_back(plane_rows(v, g.ouy, g.pu, ua, ub));
    dst.push_back(plane_rows(v, g.op, g.pp, pa, pb));
  };
  if (rank > 0) {
    add(ls, 2 * lo, std::min(2 * lo + 2 * H, lat), lo, std::min(lo + H, np));
    add(lr, 2 * lo - 2 * H, 2 * lo, lo - H, lo);
  }
  if (rank < P - 1) {
    add(hs, 2 * hi - 2 * H, 2 * hi, hi - H, hi);
    add(hr, 2 * hi, std::min(2 * hi + 2 * H, lat), hi, std::min(hi + H, np));
  }
  if (ctx->tr->exchange(ls, lr, hs, hr, s, ctx->err) != 0) return SVK_ERR_NCCL;
  ctx->launches++;
  if (ctx->poison) {  // rows no kernel may read: NaN (0xFF bytes); a slab-local vector
                      // holds no memory beyond its margin rows, so only those are poisoned
    const int ua = std::max(0, 2 * lo - 2 * H), ub = std::min(lat, 2 * hi + 2 * H);
    const int pa = std::max(0, lo - H), pb = std::min(np, hi + H);
    const bool slab = ctx->slab_mem.count(v) != 0;
    const SlabRows T = slab ? slab_rows_touched(g) : SlabRows{0, lat, 0, np};
    for (int64_t off : {g.oux, g.ouy}) {
      CK(cudaMemsetAsync(v + off + (int64_t)T.ua * g.pu, 0xFF, (size_t)std::max(0, ua - T.ua) * g.pu * sizeof(double), s));
      CK(cudaMemsetAsync(v + off + (int64_t)ub * g.pu, 0xFF, (size_t)std::max(0, T.ub - ub) * g.pu * sizeof(double), s));
    }
    CK(cudaMemsetAsync(v + g.op + (int64_t)T.pa * g.pp, 0xFF, (size_t)std::max(0, pa - T.pa) * g.pp * sizeof(double), s));
    CK(cudaMemsetAsync(v + g.op + (int64_t)pb * g.pp, 0xFF, (size_t)std::max(0, T.pb - pb) * g.pp * sizeof(double), s));
  }
  return SVK_OK;
}

int op_allreduce(svk_ctx* ctx, double* buf, int64_t count, cudaStream_t s) {
  if (!ctx->tr) return SVK_OK;
  if (ctx->tr->allreduce_sum(buf, count, s, ctx->err) != 0) return SVK_ERR_NCCL;
  ctx->launches++;
  return SVK_OK;
}

// zero every entry of v outside this rank's owned rows on level l (and the plane tails)
int op_zero_unowned(svk_ctx* ctx, int l, double* v, cudaStream_t s) {
  const LevelGeom& g = ctx->g[l];
  const int a = 2 * g.r0, b = std::min(2 * g.r1, g.lat);
  const int64_t ends[3] = {g.ouy, g.op, g.len};
  const int64_t offs[3] = {g.oux, g.ouy, g.op};
  for (int k = 0; k < 3; ++k) {
    const int64_t pitch = k < 2 ? g.pu : g.pp;
    const int ra = k < 2 ? a : g.r0, rb = k < 2 ? b : g.r1;
    CK(cudaMemsetAsync(v + offs[k], 0, (size_t)ra * pitch * sizeof(double), s));
    const int64_t e = offs[k] + (int64_t)rb * pitch;
    CK(cudaMemsetAsync(v + e, 0, (size_t)(ends[k] - e) * sizeof(double), s));
  }
  return SVK_OK;
}

// owned index segments of a level-l vector, in double2 units
Seg3 owned_segments(const svk_ctx* ctx, int l) {
  const LevelGeom& g = ctx->g[l];
  Seg3 S{};
  if (!dist_level(ctx, l)) {
    const int64_t n2 = g.len / 2;
    S.cum2[1] = S.cum2[2] = S.cum2[3] = n2;
    return S;
  }
  const int a = 2 * g.r0, b = std::min(2 * g.r1, g.lat);
  const int64_t nu2 = (int64_t)(b - a) * g.pu / 2, np2 = (int64_t)(g.r1 - g.r0) * g.pp / 2;
  S.off2[0] = (g.oux + (int64_t)a * g.pu) / 2;
  S.off2[1] = (g.ouy + (int64_t)a * g.pu) / 2;
  S.off2[2] = (g.op + (int64_t)g.r0 * g.pp) / 2;
  S.cum2[1] = nu2;
  S.cum2[2] = 2 * nu2;
  S.cum2[3] = 2 * nu2 + np2;
  return S;
}

int op_sweep_impl(svk_ctx* ctx, int l, const double* xin, const double* b, double* xout, bool x_zero,
                  cudaStream_t s);
int op_sweep(svk_ctx* ctx, int l, const double* xin, const double* b, double* xout, bool x_zero, cudaStream_t s) {
  // only full sweeps (non-zero x_in) are timed, so the roofline's per-unit counts apply
  const bool timed = ctx->prof && l == ctx->nlev - 1 && !x_zero;
  if (timed && ctx->capturing) {  // events owned by the graph being captured
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    ctx->capturing->ev.emplace_back(e0, e1);
    // cudaEventRecordExternal: real event-record nodes in the captured graph
    // (a plain record during capture only expresses a dependency)
    ctx->sweep_ev0 = e0;
    ctx->sweep_ev0_flags = cudaEventRecordExternal;
    TRY(op_sweep_impl(ctx, l, xin, b, xout, x_zero, s));
    CK(cudaEventRecordWithFlags(e1, s, cudaEventRecordExternal));
    return SVK_OK;
  }
  if (timed) {
    while (ctx->prof_ev.size() < ctx->prof_used + 2) {
      cudaEvent_t e;
      CK(cudaEventCreate(&e));
      ctx->prof_ev.push_back(e);
    }
    ctx->sweep_ev0 = ctx->prof_ev[ctx->prof_used];
    ctx->sweep_ev0_flags = cudaEventRecordDefault;
  }
  TRY(op_sweep_impl(ctx, l, xin, b, xout, x_zero, s));
  if (timed) {
    CK(cudaEventRecord(ctx->prof_ev[ctx->prof_used + 1], s));
    ctx->prof_used += 2;
  }
  return SVK_OK;
}
// SVK_DEBUG_SLAB=1: report slab-local inputs whose mapped rows do not cover the
// rows a sweep reads (2(r0-1)-6 .. 2 r1 + 6 lattice rows)
void debug_slab_rows(const svk_ctx* ctx, int l, const double* v, const char* what) {
  static const bool on = [] { const char* e = std::getenv("SVK_DEBUG_SLAB"); return e && e[0] == '1'; }();
  if (!on || !v) return;
  auto it = ctx->slab_mem.find(v);
  const LevelGeom& g = ctx->g[l];
  if (it == ctx->slab_mem.end()) {
    std::fprintf(stderr, "[slab] rank %d level N=%d %s %p: plain (full)\n", ctx->cfg.rank, g.N, what, (const void*)v);
    return;
  }
  std::fprintf(stderr, "[slab] rank %d level N=%d rows %d..%d %s %p: slab\n", ctx->cfg.rank, g.N, g.r0, g.r1, what,
               (const void*)v);
  const int lo = std::max(0, 2 * (g.r0 - 1) - 6), hi = std::min(g.lat - 1, 2 * g.r1 + 6);
  for (int64_t off : {g.oux, g.ouy}) {
    const int64_t a = (off + (int64_t)lo * g.pu) * 8, b = (off + (int64_t)(hi + 1) * g.pu) * 8;
    bool ok = false;
    for (const auto& r : it->second.maps) ok = ok || (r.first <= a && b <= r.first + r.second);
    if (!ok)
      std::fprintf(stderr, "[slab] rank %d level N=%d rows %d..%d (r0 %d r1 %d) %s %p: NOT MAPPED\n", ctx->cfg.rank,
                   g.N, lo, hi, g.r0, g.r1, what, (const void*)v);
  }
}
int op_sweep_impl(svk_ctx* ctx, int l, const double* xin, const double* b, double* xout, bool x_zero,
                  cudaStream_t s) {
  debug_slab_rows(ctx, l, b, "sweep b");
  if (!x_zero) debug_slab_rows(ctx, l, xin, "sweep x");
  const LevelGeom& g = ctx->g[l];
  const int scalar_w = ctx->cfg.weighting == SVK_WEIGHT_SCALAR;
  // timed sweep (op_sweep): the start event brackets the sweep kernel alone --
  // recorded after the boundary-patch kernel in the fused path
  const cudaEvent_t ev0 = ctx->sweep_ev0;
  ctx->sweep_ev0 = nullptr;
  if (ev0 && ctx->cfg.sweep_impl != SVK_SWEEP_FUSED) CK(cudaEventRecordWithFlags(ev0, s, ctx->sweep_ev0_flags));
  if (ctx->cfg.sweep_impl == SVK_SWEEP_FUSED) {
    const int lst = launch_fused_sweep(g, ctx->cfg.nu, ctx->cfg.omega_v, scalar_w, ctx->h_fac[l],
                                       ctx->d_inv + (size_t)l * 25 * kGroupStride, ctx->d_tiles[l], ctx->ntiles[l],
                                       ctx->d_bd, x_zero ? nullptr : xin, b, xout, ctx->nsm, s, ev0,
                                       ctx->sweep_ev0_flags);
    if (lst != 0) {
      ctx->err = lst == -3 ? std::string("sweep: profiling event record failed") : "sweep: " + tma_error();
      return SVK_ERR_CUDA;
    }
    CKL();
    ctx->launches++;  // two kernels: boundary patches + fused sweep
    return SVK_OK;
  }
  // unfused: residual, packed patch solves, gather update
  double* r = ctx->ws_r[l];
  if (x_zero) {  // "initial approximation ... a zero vector": make the input really zero
    CK(cudaMemsetAsync(const_cast<double*>(xin), 0, g.len * sizeof(double), s));
  }
  TRY(op_residual(ctx, l, xin, b, r, s));
  const int64_t np = (int64_t)(g.N + 1) * (g.N + 1);
  if (ctx->cfg.sweep_impl == SVK_SWEEP_SIMPLE)
    k_patch_solve_simple<<<(unsigned)((np + 127) / 128), 128, 0, s>>>(g, r, ctx->d_inv_simple[l], ctx->d_dbuf);
  else
    k_patch_solve_unfused<<<(unsigned)((np + 127) / 128), 128, 0, s>>>(g, r, ctx->d_inv + (size_t)l * 25 * kGroupStride,
                                                                       ctx->d_dbuf);
  CKL();
  k_vanka_update<<<plane_grid(g), kPlaneBlock, 0, s>>>(g, ctx->cfg.omega_v, scalar_w, xin, ctx->d_dbuf, xout);
  CKL();
  return SVK_OK;
}

// alg:bs / alg:uz sweep (relax_bs.cuh) on level l
int op_bs(svk_ctx* ctx, int l, const double* xin, const double* b, double* xout, bool x_zero, cudaStream_t s) {
  const LevelGeom& g = ctx->g[l];
  const svk_config& c = ctx->cfg;
  if (x_zero) CK(cudaMemsetAsync(const_cast<double*>(xin), 0, g.len * sizeof(double), s));
  double* r = ctx->ws_r[l];
  TRY(op_residual(ctx, l, xin, b, r, s));
  BsArgs a{};
  a.g = g;
  a.inv_t = 1.0 / c.relax_t;
  a.su = c.relax == SVK_RELAX_SCHUR_UZAWA;
  a.omega_r = a.su ? 1.0 : c.relax_omega;
  const FusedFactors& F = ctx->h_fac[l];
  for (int py = 0; py < 2; ++py)
    for (int px = 0; px < 2; ++px) a.dinv[py][px] = 1.0 / F.L2D[py][px][2][2];
  const dim3 pb(32, 4), pg((unsigned)((g.pp + 31) / 32), (unsigned)((g.N + 1 + 3) / 4));
  k_bs_rhs<<<pg, pb, 0, s>>>(a, r, ctx->p_rhs[l]);
  CKL();
  const double* st = ctx->d_schur + (size_t)l * kSchurStride;
  double* dp = ctx->p_dp0[l];
  if (c.jacobi_sweeps == 0) CK(cudaMemsetAsync(dp, 0, (size_t)(g.N + 1) * g.pp * sizeof(double), s));
  for (int k = 0; k < c.jacobi_sweeps; ++k) {
    double* out = (k & 1) ? ctx->p_dp0[l] : ctx->p_dp1[l];
    k_schur_jacobi<<<pg, pb, 0, s>>>(g, st, c.jacobi_omega, ctx->p_rhs[l], k == 0 ? nullptr : dp, out);
    CKL();
    dp = out;
  }
  {
    const dim3 blk(32, 8), grd((unsigned)((std::max<int64_t>(g.pu, g.pp) / 2 + 32) / 32), (unsigned)((g.lat + 7) / 8), 3);
    k_bs_update2<<<grd, blk, 0, s>>>(a, xin, r, dp, xout);
  }
  CKL();
  ctx->launches += 3 + c.jacobi_sweeps;
  return SVK_OK;
}
// "Relax on u_l and p_l" (alg:mg) with the configured relaxation
int op_relax(svk_ctx* ctx, int l, const double* xin, const double* b, double* xout, bool x_zero, cudaStream_t s) {
  if (ctx->cfg.relax == SVK_RELAX_VANKA) return op_sweep(ctx, l, xin, b, xout, x_zero, s);
  return op_bs(ctx, l, xin, b, xout, x_zero, s);
}

// ---- block-triangular preconditioner (alg:bt) -------------------------------
// plane range of a part: 0 = velocity planes [oux, op), 1 = pressure plane [op, len)
void bt_range(const LevelGeom& g, int part, int64_t* off, int64_t* cnt) {
  *off = part ? g.op : g.oux;
  *cnt = part ? g.len - g.op : g.op - g.oux;
}
// scalar V(nu, nu) cycle with weighted Jacobi for block `part` on level l; x in/out
int op_blk_mg(svk_ctx* ctx, int l, int part, const double* b, double* x, cudaStream_t s) {
  const LevelGeom& g = ctx->g[l];
  const svk_config& c = ctx->cfg;
  int64_t off, cnt;
  bt_range(g, part, &off, &cnt);
  if (l == 0) {
    CK(cudaMemsetAsync(x + off, 0, cnt * sizeof(double), s));
    if (part == 0) k_coarse_apply<<<(ctx->bt_niL + 3) / 4, 128, 0, s>>>(ctx->d_bt_invL, ctx->bt_niL, ctx->d_bt_idxL, b, x);
    else k_coarse_apply<<<(ctx->bt_niM + 3) / 4, 128, 0, s>>>(ctx->d_bt_invM, ctx->bt_niM, ctx->d_bt_idxM, b, x);
    CKL();
    ++ctx->launches;
    return SVK_OK;
  }
  BtArgs a{};
  a.g = g;
  a.nu = c.nu;
  a.part = part;
  a.omega = part ? c.bt_omega_p : c.bt_omega_u;
  const FusedFactors& F = ctx->h_fac[l];
  for (int py = 0; py < 2; ++py)
    for (int px = 0; px < 2; ++px) a.dinv[py][px] = 1.0 / F.L2D[py][px][2][2];
  dim3 grid = plane_grid(g);
  grid.z = part ? 1 : 2;
  if (part) grid = dim3((unsigned)((g.pp + 31) / 32), (unsigned)((g.N + 1 + 7) / 8), 1);
  L2DTab tab;
  std::memcpy(&tab, F.L2D, sizeof(tab));
  const dim3 vblk(32, 8), vgrid((unsigned)((g.pu / 2 + 31) / 32), (unsigned)((g.lat + 7) / 8), 2);
  auto smooth = [&]() -> int {
    const double* src = x;
    double* dst = ctx->ws_t[l];
    for (int k = 0; k < c.bt_nu; ++k) {
      if (part == 0) k_bt_smooth_vel<1><<<vgrid, vblk, 0, s>>>(a, tab, src, b, dst);
      else k_bt_smooth<1><<<grid, kPlaneBlock, 0, s>>>(a, src, b, dst);
      CKL();
      ++ctx->launches;
      double* nsrc = dst;
      dst = const_cast<double*>(src);
      src = nsrc;
    }
    if (src != x) CK(cudaMemcpyAsync(x + off, src + off, cnt * sizeof(double), cudaMemcpyDeviceToDevice, s));
    return SVK_OK;
  };
  TRY(smooth());
  if (part == 0) k_bt_smooth_vel<0><<<vgrid, vblk, 0, s>>>(a, tab, x, b, ctx->ws_r[l]);
  else k_bt_smooth<0><<<grid, kPlaneBlock, 0, s>>>(a, x, b, ctx->ws_r[l]);
  CKL();
  const LevelGeom& gc = ctx->g[l - 1];
  dim3 cg = plane_grid(gc);
  cg.z = part ? 1 : 2;
  k_restrict<<<cg, kPlaneBlock, 0, s>>>(g, gc, ctx->ws_r[l], ctx->ws_b[l - 1], part ? 2 : 0);
  CKL();
  int64_t coff, ccnt;
  bt_range(gc, part, &coff, &ccnt);
  CK(cudaMemsetAsync(ctx->ws_x[l - 1] + coff, 0, ccnt * sizeof(double), s));
  TRY(op_blk_mg(ctx, l - 1, part, ctx->ws_b[l - 1], ctx->ws_x[l - 1], s));
  {  // velocity blocks (z = 0, 1) for part 0, pressure blocks (z = 2) for part 1
    const dim3 blk(32, 4), grd((unsigned)((gc.N + 1 + 31) / 32), (unsigned)((gc.N + 1 + 3) / 4), part ? 3 : 2);
    k_prolong<<<grd, blk, 0, s>>>(g, gc, ctx->ws_x[l - 1], x, 0, part ? 0 : gc.N, 0, part ? gc.N + 1 : 0);
  }
  CKL();
  ctx->launches += 3;
  TRY(smooth());
  return SVK_OK;
}
// z = BT(r) on the finest level (alg:bt lines 1-2)
int op_bt(svk_ctx* ctx, const double* r, double* z, cudaStream_t s) {
  const int L = ctx->nlev - 1;
  const LevelGeom& g = ctx->g[L];
  k_bt_rhs<0><<<plane_grid(g), kPlaneBlock, 0, s>>>(g, r, nullptr, ctx->d_btb);  // (0, 0, -r_p)
  CKL();
  CK(cudaMemsetAsync(z, 0, g.len * sizeof(double), s));
  for (int k = 0; k < ctx->cfg.bt_cycles; ++k) TRY(op_blk_mg(ctx, L, 1, ctx->d_btb, z, s));  // M dp = -r_p
  k_bt_rhs<1><<<plane_grid(g), kPlaneBlock, 0, s>>>(g, r, z, ctx->d_btb);  // (r_u - B^T dp, 0)
  CKL();
  for (int k = 0; k < ctx->cfg.bt_cycles; ++k) TRY(op_blk_mg(ctx, L, 0, ctx->d_btb, z, s));  // L du = ...
  ctx->launches += 2;
  return SVK_OK;
}

int op_restrict(svk_ctx* ctx, int l, const double* rf, double* rc, cudaStream_t s) {
  k_restrict<<<plane_grid(ctx->g[l - 1]), kPlaneBlock, 0, s>>>(ctx->g[l], ctx->g[l - 1], rf, rc, 0);
  CKL();
  return SVK_OK;
}
int op_prolong_add(svk_ctx* ctx, int l, const double* ec, double* xf, cudaStream_t s) {
  const LevelGeom &gf = ctx->g[l], &gc = ctx->g[l - 1];
  // velocity: coarse element rows covering the owned fine lattice rows [max(2 r0, 1), min(2 r1, lat - 1));
  // pressure: coarse node rows covering the owned fine node rows; one launch for both
  const int jlo = std::max(2 * gf.r0, 1), jhi = std::min(2 * gf.r1, gf.lat - 1);
  const int ey0 = jlo / 4, ney = jhi > jlo ? (jhi - 1) / 4 - ey0 + 1 : 0;
  const int ay0 = gf.r0 / 2, nay = (gf.r1 - 1) / 2 - ay0 + 1;
  const dim3 blk(32, 4), grd((unsigned)((gc.N + 1 + 31) / 32), (unsigned)((std::max(ney, nay) + 3) / 4), 3);
  launch_pdl(k_prolong, grd, blk, 0, s, gf, gc, ec, xf, ey0, ney, ay0, nay);
  CKL();
  return SVK_OK;
}
int op_coarse(svk_ctx* ctx, const double* b, double* x, cudaStream_t s) {
  const LevelGeom& g = ctx->g[0];
  if (ctx->cfg.coarse == SVK_COARSE_SWEEPS3) {
    // three relaxation sweeps from zero, ping-pong x <-> ws_t[0]
    TRY(op_relax(ctx, 0, x, b, ctx->ws_t[0], true, s));
    TRY(op_relax(ctx, 0, ctx->ws_t[0], b, x, false, s));
    TRY(op_relax(ctx, 0, x, b, ctx->ws_t[0], false, s));
    CK(cudaMemcpyAsync(x, ctx->ws_t[0], g.len * sizeof(double), cudaMemcpyDeviceToDevice, s));
    return SVK_OK;
  }
  CK(cudaMemsetAsync(x, 0, g.len * sizeof(double), s));
  launch_pdl(k_coarse_apply, dim3((ctx->cni + 3) / 4), dim3(128), 0, s, (const double*)ctx->d_cmat, ctx->cni,
             (const int*)ctx->d_cidx, b, x);
  CKL();
  return SVK_OK;
}

// Agglomeration: level l is the coarsest distributed level and
// level l-1 is replicated.  Each rank has restricted its slab's coarse rows into
// rc (the halves of its fine slab, op_residual_restrict); the three plane pieces
// are packed into one fixed-size chunk, all-gathered (each rank receives the
// other ranks' rows once: (P-1)/P of the coarse vector, half the bytes of an
// all-reduce of zero-padded copies) and unpacked into every rank's full rc.
int op_agglomerate(svk_ctx* ctx, int l, double* rc, cudaStream_t s) {
  const LevelGeom& gf = ctx->g[l];
  const LevelGeom& gc = ctx->g[l - 1];
  const int P = ctx->cfg.nranks;
  const int Nla = ctx->g[ctx->la].N;
  // coarse node rows of rank r: the halves of its fine slab (as op_residual_restrict)
  std::vector<int> c0(P), c1(P);
  int64_t K = 0;
  for (int r = 0; r < P; ++r) {
    int f0, f1;
    slab_rows(gf.N, Nla, P, r, &f0, &f1);
    c0[r] = f0 / 2;
    c1[r] = f1 == gf.N + 1 ? gc.N + 1 : f1 / 2;
    const int64_t u = (int64_t)(std::min(2 * c1[r], gc.lat) - std::min(2 * c0[r], gc.lat)) * gc.pu;
    K = std::max<int64_t>(K, 2 * u + (int64_t)(c1[r] - c0[r]) * gc.pp);
  }
  if (ctx->agg_cap < (int64_t)P * K) {
    if (ctx->d_agg) cudaFree(ctx->d_agg);
    ctx->d_agg = nullptr;
    CK(cudaMalloc(&ctx->d_agg, (size_t)P * K * sizeof(double)));
    ctx->agg_cap = (int64_t)P * K;
  }
  auto pieces = [&](int r, double* v, std::vector<Block>& out) {
    const int ua = std::min(2 * c0[r], gc.lat), ub = std::min(2 * c1[r], gc.lat);
    out = {plane_rows(v, gc.oux, gc.pu, ua, ub), plane_rows(v, gc.ouy, gc.pu, ua, ub),
           plane_rows(v, gc.op, gc.pp, c0[r], c1[r])};
  };
  const int me = ctx->cfg.rank;
  std::vector<Block> bl;
  pieces(me, rc, bl);
  double* mine = ctx->d_agg + (int64_t)me * K;
  int64_t o = 0;
  for (const Block& b : bl) {
    if (b.count) CK(cudaMemcpyAsync(mine + o, b.ptr, b.count * sizeof(double), cudaMemcpyDeviceToDevice, s));
    o += b.count;
  }
  if (ctx->tr->allgather(mine, ctx->d_agg, K, s, ctx->err) != 0) return SVK_ERR_NCCL;
  ctx->launches++;
  for (int r = 0; r < P; ++r) {
    if (r == me) continue;
    pieces(r, rc, bl);
    const double* src = ctx->d_agg + (int64_t)r * K;
    int64_t q = 0;
    for (const Block& b : bl) {
      if (b.count) CK(cudaMemcpyAsync(b.ptr, src + q, b.count * sizeof(double), cudaMemcpyDeviceToDevice, s));
      q += b.count;
    }
  }
  return SVK_OK;
}

// alg:mg on level l; x in/out; x_zero: x is known to be 0 on entry
// Distributed levels (row slabs): every operation computes the owned rows; the
// halos of b (on entry), of x after every relaxation and after the correction,
// are refreshed by op_halo, so the returned x has valid halos.  On the
// agglomeration level the restricted residual is assembled on every rank by an
// all-reduce of the disjoint, zero-padded slab pieces; the coarser levels then
// run redundantly (replicated) on every rank.
// compact [u_x lat^2, u_y lat^2, p (N+1)^2] <-> pitched finest-level layout, on the device
// (svk_solve_host_batch: the host copies stay 1D and contiguous)
template <bool TO_PITCHED>
__global__ void k_repitch(LevelGeom g, const double* __restrict__ src, double* __restrict__ dst) {
  const int64_t nv = (int64_t)g.lat * g.lat, np = (int64_t)(g.N + 1) * (g.N + 1);
  for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < 2 * nv + np; q += (int64_t)gridDim.x * blockDim.x) {
    int64_t o;
    if (q < 2 * nv) {
      const int64_t qq = q < nv ? q : q - nv;
      o = (q < nv ? g.oux : g.ouy) + (qq / g.lat) * g.pu + qq % g.lat;
    } else {
      const int64_t qq = q - 2 * nv;
      o = g.op + (qq / (g.N + 1)) * g.pp + qq % (g.N + 1);
    }
    if (TO_PITCHED) dst[o] = src[q];
    else dst[q] = src[o];
  }
}

// Which coarse levels run in the one-launch V-cycle, and on how many CTAs.
// SVK_SMALL_N (default 16, measured best: 4096^2 V-cycle 5378 -> 5341 us, 1024^2
// 859 -> 813 us; at 32 / 64 the grid-stride phases of the larger levels cost
// more than the launches they replace): largest N; 0 disables.  Only the fused Vanka
// relaxation, only replicated levels below the finest.  Cluster: 16 CTAs
// (non-portable size) when the device can co-schedule it, else 8.
int setup_small_cycle(svk_ctx* ctx) {
  ctx->sc_top = 0;
  const char* e = std::getenv("SVK_SMALL_N");
  const int lc = e ? std::atoi(e) : 16;
  const svk_config& c = ctx->cfg;
  if (lc <= 0 || c.relax != SVK_RELAX_VANKA || c.sweep_impl != SVK_SWEEP_FUSED) return SVK_OK;
  int top = 0;
  for (int l = 1; l < ctx->nlev - 1 && l < kScMaxLevels; ++l)
    if (ctx->g[l].N <= lc && !dist_level(ctx, l)) top = l;
  if (top < 1) return SVK_OK;
  CK(cudaFuncSetAttribute(k_small_cycle, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  const char* ce = std::getenv("SVK_SMALL_CLUSTER");  // taken as given (no occupancy check): a test hook
  int cl = ce ? std::atoi(ce) : 16;
  for (; cl >= 1 && !ce; cl /= 2) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)cl);
    cfg.blockDim = dim3(kScThreads);
      cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = (unsigned)cl;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    int n = 0;
    if (cudaOccupancyMaxActiveClusters(&n, k_small_cycle, &cfg) == cudaSuccess && n >= 1) break;
    cudaGetLastError();
  }
  if (cl < 1) return SVK_OK;
  const int64_t np = (int64_t)(ctx->g[top].N + 1) * (ctx->g[top].N + 1);
  TRY(alloc_vec(ctx, &ctx->d_sc, (int64_t)kSlots * np));
  for (int l = 0; l <= top; ++l) {  // boundary tiles + the generic patches in row segments of <= kBdTile
    const int N = ctx->g[l].N;
    std::vector<BdTile> t = make_bd_tiles(N);
    for (int ky = 2; ky <= N - 2; ++ky)
      for (int kx = 2; kx <= N - 2; kx += kBdTile)
        t.push_back(BdTile{kx, ky, 1, 0, std::min(kBdTile, N - 1 - kx), 2 * 5 + 2});
    BdTile* d = nullptr;
    CK(cudaMalloc(&d, t.size() * sizeof(BdTile)));
    CK(cudaMemcpy(d, t.data(), t.size() * sizeof(BdTile), cudaMemcpyHostToDevice));
    ctx->d_sc_tiles.push_back(d);
    ctx->n_sc_tiles.push_back((int)t.size());
  }
  ctx->sc_cluster = cl;
  ctx->sc_top = top;
  if (const char* d = std::getenv("SVK_DEBUG_SMALL"); d && d[0] == '1')
    std::fprintf(stderr, "[small-cycle] levels 1..%d (N <= %d), cluster of %d CTAs\n", top, ctx->g[top].N, cl);
  return SVK_OK;
}

int op_mg(svk_ctx* ctx, int l, const double* b, double* x, bool x_zero, cudaStream_t s);
// MG(l) from x = 0 on the levels l .. 0 (alg:mg) as ONE cluster launch
// (small_cycle.cuh): same steps and operators as the per-kernel recursion below.
int op_small_cycle(svk_ctx* ctx, int l, const double* b, double* x, cudaStream_t s) {
  ScArgs a{};
  a.top = l;
  for (int k = 0; k <= l; ++k) {
    ScLevel& L = a.lv[k];
    L.g = ctx->g[k];
    L.dinv = ctx->d_inv + (size_t)k * 25 * kGroupStride;
    L.tiles = ctx->d_sc_tiles[k];
    L.ntiles = ctx->n_sc_tiles[k];
    L.b = k == l ? const_cast<double*>(b) : ctx->ws_b[k];
    L.x = k == l ? x : ctx->ws_x[k];
    L.r = ctx->ws_r[k];
  }
  const svk_config& c = ctx->cfg;
  a.nu = c.nu;
  a.omega = c.omega_v;
  a.scalar_w = c.weighting == SVK_WEIGHT_SCALAR;
  a.nu_pre = c.nu_pre;
  a.nu_post = c.nu_post;
  a.sweeps3 = c.coarse == SVK_COARSE_SWEEPS3;
  a.cmat = ctx->d_cmat;
  a.cidx = ctx->d_cidx;
  a.cni = ctx->cni;
  a.d = ctx->d_sc;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)ctx->sc_cluster);
  cfg.blockDim = dim3(kScThreads);
  cfg.stream = s;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = (unsigned)ctx->sc_cluster;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl_enabled() ? 2 : 1;
  const char* dbg = std::getenv("SVK_DEBUG_SMALL");
  static unsigned long long* stamps = nullptr;  // development aid only (run with SVK_GRAPHS=0)
  if (dbg && dbg[0] == '2') {
    if (!stamps) CK(cudaMallocManaged(&stamps, 4096 * sizeof(unsigned long long)));
    a.stamps = stamps;
  }
  if (const cudaError_t le = cudaLaunchKernelEx(&cfg, k_small_cycle, a); le != cudaSuccess) {
    // a cluster the device cannot place right now (e.g. a partitioned GPU): outside a
    // stream capture, fall back to the per-kernel recursion for good
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    cudaStreamIsCapturing(s, &cs);
    if (cs != cudaStreamCaptureStatusNone) {
      ctx->err = std::string("coarse cycle launch: ") + cudaGetErrorString(le);
      return SVK_ERR_CUDA;
    }
    cudaGetLastError();
    ctx->sc_top = 0;
    return op_mg(ctx, l, b, x, true, s);
  }
  if (a.stamps) {
    CK(cudaStreamSynchronize(s));
    std::string o = "[small-cycle us]";
    for (int k = 1; k < 4096 && stamps[k] > stamps[k - 1] && stamps[k] - stamps[0] < 100000000ull; ++k)
      o += " " + std::to_string((stamps[k] - stamps[k - 1]) / 100 / 10.0);
    std::fprintf(stderr, "%s\n", o.c_str());
    std::memset(stamps, 0, 4096 * sizeof(unsigned long long));
  }
  ctx->launches++;
  return SVK_OK;
}

int op_mg(svk_ctx* ctx, int l, const double* b, double* x, bool x_zero, cudaStream_t s) {
  const LevelGeom& g = ctx->g[l];
  if (l == 0) return op_coarse(ctx, b, x, s);
  if (x_zero && l <= ctx->sc_top) return op_small_cycle(ctx, l, b, x, s);  // levels l .. 0 in one launch
  const bool D = dist_level(ctx, l);
  if (D) {
    TRY(op_halo(ctx, l, const_cast<double*>(b), s));
    if (!x_zero) TRY(op_halo(ctx, l, x, s));
  }
  double* cur = x;
  double* oth = ctx->ws_t[l];
  for (int k = 0; k < ctx->cfg.nu_pre; ++k) {  // "Relax on u_l and p_l"
    TRY(op_relax(ctx, l, cur, b, oth, x_zero && k == 0, s));
    std::swap(cur, oth);
    if (D) TRY(op_halo(ctx, l, cur, s));
  }
  if (ctx->cfg.nu_pre == 0 && x_zero) TRY(op_zero_level(ctx, l, cur, s));
  const bool agglomerate = D && !dist_level(ctx, l - 1);
  TRY(op_residual_restrict(ctx, l, cur, b, ctx->ws_b[l - 1], s));  // "Compute residual" + "Restriction"
  if (agglomerate) TRY(op_agglomerate(ctx, l, ctx->ws_b[l - 1], s));
  TRY(op_mg(ctx, l - 1, ctx->ws_b[l - 1], ctx->ws_x[l - 1], true, s));  // A_0^{-1} or MG(l-1)
  TRY(op_prolong_add(ctx, l, ctx->ws_x[l - 1], cur, s));       // "Correction"
  if (D) TRY(op_halo(ctx, l, cur, s));
  for (int k = 0; k < ctx->cfg.nu_post; ++k) {                 // "Relax on u_l and p_l"
    TRY(op_relax(ctx, l, cur, b, oth, false, s));
    std::swap(cur, oth);
    if (D) TRY(op_halo(ctx, l, cur, s));
  }
  if (cur != x) TRY(op_copy_level(ctx, l, x, cur, s));
  return SVK_OK;
}

// Validation mode (see k_validate_batch): max relative deviation on level l of
// (a) every patch's own inverse from its group's stored inverse, (b) the generic
// reflection-basis factors from the generic group's inverse.
int op_validate(svk_ctx* ctx, int l, double* max_dev, int64_t* n_patch) {
  const LevelGeom& g = ctx->g[l];
  const int64_t np = (int64_t)(g.N + 1) * (g.N + 1);
  std::vector<double> ginv((size_t)25 * kGroupStride), scale(25, 0.0);
  const double* dg = ctx->d_inv + (size_t)l * 25 * kGroupStride;
  CK(cudaMemcpy(ginv.data(), dg, ginv.size() * sizeof(double), cudaMemcpyDeviceToHost));
  for (int k = 0; k < 25; ++k)
    for (int q = 0; q < kGroupStride; ++q) scale[k] = std::max(scale[k], std::fabs(ginv[(size_t)k * kGroupStride + q]));
  const int64_t nb = std::min<int64_t>(np, 8192);
  double *d_batch = nullptr, *d_scale = nullptr, *d_dev = nullptr;
  int* d_st = nullptr;
  auto cleanup = [&]() {
    cudaFree(d_batch);
    cudaFree(d_scale);
    cudaFree(d_dev);
    cudaFree(d_st);
  };
  if (cudaMalloc(&d_batch, (size_t)nb * kGroupStride * sizeof(double)) != cudaSuccess ||
      cudaMalloc(&d_scale, 25 * sizeof(double)) != cudaSuccess || cudaMalloc(&d_dev, 2 * sizeof(double)) != cudaSuccess ||
      cudaMalloc(&d_st, sizeof(int)) != cudaSuccess) {
    cudaGetLastError();
    cleanup();
    ctx->err = "validation: workspace allocation failed";
    return SVK_ERR_ALLOC;
  }
  cudaMemcpy(d_scale, scale.data(), 25 * sizeof(double), cudaMemcpyHostToDevice);
  cudaMemset(d_dev, 0, 2 * sizeof(double));
  cudaMemset(d_st, 0, sizeof(int));
  for (int64_t p0 = 0; p0 < np; p0 += nb) {
    const int64_t n = std::min(nb, np - p0);
    k_patch_setup_simple<<<(unsigned)n, 128>>>(g, ctx->cfg.nu, p0, d_batch, d_st, nb, p0);
    k_validate_batch<<<(unsigned)std::min<int64_t>((n * kGroupStride + 255) / 256, 4096), 256>>>(
        g, p0, nb, d_batch, dg, d_scale, d_dev);
  }
  k_validate_factors<<<1, 64>>>(ctx->h_fac[l], dg + (size_t)12 * kGroupStride, scale[12], d_dev + 1);
  double dev[2] = {0, 0};
  int st = 0;
  const cudaError_t e1 = cudaMemcpy(dev, d_dev, 2 * sizeof(double), cudaMemcpyDeviceToHost);
  const cudaError_t e2 = cudaMemcpy(&st, d_st, sizeof(int), cudaMemcpyDeviceToHost);
  cleanup();
  if (e1 != cudaSuccess || e2 != cudaSuccess) {
    ctx->err = std::string("validation: ") + cudaGetErrorString(e1 != cudaSuccess ? e1 : e2);
    return SVK_ERR_CUDA;
  }
  if (st) {
    ctx->err = "validation: singular patch matrix";
    return SVK_ERR_SINGULAR;
  }
  *max_dev = std::max(dev[0], g.N >= 4 ? dev[1] : 0.0);
  *n_patch = np;
  return SVK_OK;
}
constexpr double kValidateTol = 1e-12;

// Sweep times of replayed graphs (their events are re-recorded at every replay,
// so each replay is harvested after the stream synchronisation that follows it).
int harvest_graph_prof(svk_ctx* ctx) {
  for (auto* gr : ctx->prof_pending)
    for (auto& pr : gr->ev) {
      float ms = 0.f;
      CK(cudaEventElapsedTime(&ms, pr.first, pr.second));
      ctx->prof_acc_ms += ms;
      ctx->prof_acc_n++;
    }
  ctx->prof_pending.clear();
  return SVK_OK;
}

// z = M v (one V-cycle from zero on the finest level) for FGMRES: replayed from a
// CUDA graph captured on the library's own stream at the first use of the pair
// (v, z); not with the emulated transport (it synchronises host
// threads inside a cycle, which a graph cannot hold).  Falls back to direct
// launches if capture is unavailable.  Multi-GPU (NCCL): the cycle's halo
// exchanges and the agglomeration all-gather are captured with it.
int op_precond_mg(svk_ctx* ctx, const double* v, double* z, cudaStream_t s) {
  const int L = ctx->nlev - 1;
  if (ctx->use_graphs < 0) {
    const char* e = std::getenv("SVK_GRAPHS");
    ctx->use_graphs = (e && e[0] == '0') ? 0 : 1;
  }
  if (!ctx->use_graphs || (ctx->tr && !ctx->tr->capturable())) return op_mg(ctx, L, v, z, true, s);
  svk_ctx::GraphRec* gr = nullptr;
  for (auto& g : ctx->graphs)
    if (g->in == v && g->out == z && g->prof == ctx->prof) gr = g.get();
  if (!gr) {
    if (!ctx->cap_stream) CK(cudaStreamCreateWithFlags(&ctx->cap_stream, cudaStreamNonBlocking));
    auto rec = std::make_unique<svk_ctx::GraphRec>();
    rec->in = v;
    rec->out = z;
    rec->prof = ctx->prof;
    const int64_t l0 = ctx->launches;
    ctx->capturing = rec.get();
    CK(cudaStreamBeginCapture(ctx->cap_stream, cudaStreamCaptureModeRelaxed));
    const int st = op_mg(ctx, L, v, z, true, ctx->cap_stream);
    cudaGraph_t graph = nullptr;
    const cudaError_t ce = cudaStreamEndCapture(ctx->cap_stream, &graph);
    ctx->capturing = nullptr;
    rec->launches = ctx->launches - l0;
    ctx->launches = l0;
    cudaError_t ie = cudaErrorUnknown;
    if (st == SVK_OK && ce == cudaSuccess && graph) ie = cudaGraphInstantiate(&rec->exec, graph, 0);
    if (graph) cudaGraphDestroy(graph);
    if (ie != cudaSuccess) {  // no graph: direct launches from now on
      cudaGetLastError();
      for (auto& pr : rec->ev) {
        cudaEventDestroy(pr.first);
        cudaEventDestroy(pr.second);
      }
      ctx->use_graphs = 0;
      return op_mg(ctx, L, v, z, true, s);
    }
    gr = rec.get();
    ctx->graphs.push_back(std::move(rec));
  }
  CK(cudaGraphLaunch(gr->exec, s));
  ctx->launches += gr->launches;
  if (gr->prof && !gr->ev.empty()) ctx->prof_pending.push_back(gr);
  return SVK_OK;
}

int ensure_coef(svk_ctx* ctx, int need) {
  if (need <= ctx->coef_cap) return SVK_OK;
  int cap = std::max(need, 2 * ctx->coef_cap);
  if (ctx->d_coef) cudaFree(ctx->d_coef);
  if (ctx->h_pin) cudaFreeHost(ctx->h_pin);
  CK(cudaMalloc(&ctx->d_coef, cap * sizeof(double)));
  CK(cudaMemset(ctx->d_coef, 0, cap * sizeof(double)));  // read back in whole blocks: keep it defined
  CK(cudaHostAlloc(&ctx->h_pin, cap * sizeof(double), cudaHostAllocMapped));
  CK(cudaHostGetDevicePointer(&ctx->h_pin_dev, ctx->h_pin, 0));
  std::memset(ctx->h_pin, 0, cap * sizeof(double));
  ctx->coef_cap = cap;
  return SVK_OK;
}
// Krylov coefficients back to the host: a one-CTA kernel stores them straight into the
// mapped pinned buffer (posted PCIe writes) instead of a cudaMemcpyAsync D2H, which a
// copy engine would queue behind any large device-to-host transfer in flight (the
// pipelined svk_solve_host_batch copies solution k-1 out while solving problem k: a
// per-iteration D2H readback then waits for it, +10% solve time).
__global__ void k_to_mapped(const double* __restrict__ src, double* __restrict__ dst, int n) {
  for (int i = threadIdx.x; i < n; i += blockDim.x) dst[i] = src[i];
}
int readback(svk_ctx* ctx, const double* src, int n, cudaStream_t s) {
  k_to_mapped<<<1, 128, 0, s>>>(src, ctx->h_pin_dev, n);
  CKL();
  ctx->launches++;
  CK(cudaStreamSynchronize(s));
  return SVK_OK;
}
// ---------------------------------------------------------------------------
// Gram-Schmidt passes; basis pointers are passed by value (kernel-parameter space).
// out[0..m) = V_i . w (deterministic), written to d_coef + off.
VecList veclist(const double* const* v, int m) {
  VecList L{};
  for (int i = 0; i < m && i < kCgsMax; ++i) L.p[i] = v[i];
  return L;
}
// Distributed: the dots run over the owned segments S and are all-reduced.
int cgs_dots(svk_ctx* ctx, const double* const* dV, int m, const double* w, const Seg3& S, int off, cudaStream_t s) {
  constexpr int kDot = 16;
  for (int c0 = 0; c0 < m; c0 += kDot) {
    const int mm = std::min(kDot, m - c0);
    if (mm <= 4) launch_pdl(k_cgs_dots<4>, dim3(kDotBlocks), dim3(kRedThreads), 0, s, veclist(dV + c0, mm), mm, w, S, ctx->d_part);
    else if (mm <= 8) launch_pdl(k_cgs_dots<8>, dim3(kDotBlocks), dim3(kRedThreads), 0, s, veclist(dV + c0, mm), mm, w, S, ctx->d_part);
    else launch_pdl(k_cgs_dots<16>, dim3(kDotBlocks), dim3(kRedThreads), 0, s, veclist(dV + c0, mm), mm, w, S, ctx->d_part);
    CKL();
    launch_pdl(k_reduce_partials, dim3(mm), dim3(kRedThreads), 0, s, (const double*)ctx->d_part, kDotBlocks, ctx->d_coef + off + c0, 0);
    CKL();
  }
  if (ctx->tr) TRY(op_allreduce(ctx, ctx->d_coef + off, m, s));
  return SVK_OK;
}
// w_out = w - sum_i c_i V_i (c at d_coef + coff); squared norm of w_out -> d_coef + noff (if noff >= 0)
int cgs_update(svk_ctx* ctx, const double* const* dV, int m, int coff, const double* w, double* wout, int64_t n,
               const Seg3& S, int noff, cudaStream_t s) {
  const double* src = w;
  if (m == 0 && w != wout) CK(cudaMemcpyAsync(wout, w, n * sizeof(double), cudaMemcpyDeviceToDevice, s));
  for (int c0 = 0; c0 < m; c0 += kCgsMax) {
    const int mm = std::min(kCgsMax, m - c0);
    launch_pdl(k_cgs_update, dim3(kDotBlocks), dim3(kRedThreads), 0, s, veclist(dV + c0, mm), mm,
               (const double*)(ctx->d_coef + coff + c0), src, wout, S, ctx->d_part);
    CKL();
    src = wout;
  }
  if (noff >= 0) {
    launch_pdl(k_reduce_partials, dim3(1), dim3(kRedThreads), 0, s, (const double*)ctx->d_part, kDotBlocks, ctx->d_coef + noff, 0);
    CKL();
    if (ctx->tr) TRY(op_allreduce(ctx, ctx->d_coef + noff, 1, s));
  }
  return SVK_OK;
}
// |v| on the host (owned segments, all-reduced)
int host_norm(svk_ctx* ctx, const double* v, const Seg3& S, double* out, cudaStream_t s) {
  TRY(cgs_dots(ctx, &v, 1, v, S, 0, s));
  TRY(readback(ctx, ctx->d_coef, 1, s));
  *out = std::sqrt(std::max(ctx->h_pin[0], 0.0));
  return SVK_OK;
}

// Right-preconditioned flexible GMRES with an un-normalised
// Arnoldi basis: V~_j = n_j v_j and Z~_j = M V~_j = n_j z_j are stored without
// scaling (the V-cycle from zero is linear), so no vector pass is spent on
// normalisation; the scales n_j live on the host and enter the Hessenberg:
//   w~ = A Z~_j = n_j A z_j;  CGS2: w~'' = w~ - sum_i C_i V~_i  (C = c1 + c2,
//   c_k,i = (V~_i . w) / n_i^2);  h_ij = C_i n_i / n_j;  h_j+1,j = |w~''| / n_j;
//   V~_j+1 = w~'', n_j+1 = |w~''|;  x = x0 + sum_i (y_i / n_i) Z~_i.
int fgmres_impl(svk_ctx* ctx, const double* b, double* x, double rtol, int maxit, double* hist, svk_report* rep,
                cudaStream_t s) {
  auto t0 = std::chrono::steady_clock::now();
  const int L = ctx->nlev - 1;
  const LevelGeom& g = ctx->g[L];
  const int64_t n = g.len;
  const Seg3 S = owned_segments(ctx, L);
  svk_report R{};
  double tv = 0, to = 0;
  // coefficient area: [c1 (maxit+1) | c2 (maxit+1) | raw (maxit+1) | nrm | n^-2 (maxit+1)]
  const int o1 = 0, o2 = maxit + 1, oraw = 2 * (maxit + 1), onrm = 3 * (maxit + 1), oinv = 3 * (maxit + 1) + 1;
  TRY(ensure_coef(ctx, 4 * (maxit + 1) + 8));
  if (!ctx->d_w) TRY(alloc_level_vec(ctx, L, &ctx->d_w));
  if (!ctx->d_r) TRY(alloc_level_vec(ctx, L, &ctx->d_r));
  auto ensure_vec = [&](std::vector<double*>& pool, int k) -> int {
    while ((int)pool.size() <= k) {
      double* p;
      TRY(alloc_level_vec(ctx, L, &p));
      pool.push_back(p);
    }
    return SVK_OK;
  };
  TRY(ensure_vec(ctx->V, 0));
  // V~_0 = r0 = b - A x0, n_0 = |r0|
  TRY(op_halo(ctx, L, x, s));
  TRY(op_residual(ctx, L, x, b, ctx->V[0], s));
  TRY(cgs_dots(ctx, (const double* const*)ctx->V.data(), 1, ctx->V[0], S, onrm, s));
  TRY(readback(ctx, ctx->d_coef + onrm, 1, s));
  const double beta = std::sqrt(std::max(ctx->h_pin[0], 0.0));
  if (hist) hist[0] = 1.0;
  if (!std::isfinite(beta)) {
    ctx->err = "non-finite initial residual";
    return SVK_ERR_NONFINITE;
  }
  int status = SVK_OK, k = 0, n_reorth = 0;
  // low-memory mode: one z buffer (only with the fixed-linear MG preconditioner)
  const bool store_z = ctx->cfg.krylov_store_z != 0 || ctx->cfg.precond == SVK_PRECOND_BLOCK_TRIANGULAR;
  std::vector<const double*> dlist;
  bool conv = beta == 0.0;
  std::vector<double> H((size_t)(maxit + 1) * maxit, 0.0), cs(maxit), sn(maxit), gv(maxit + 1, 0.0), nv(maxit + 2);
  std::vector<double> inv_nsq(maxit + 1);
  auto Hij = [&](int i, int j) -> double& { return H[(size_t)i * maxit + j]; };
  if (!conv) {
    gv[0] = beta;
    nv[0] = beta;
    inv_nsq[0] = 1.0 / (beta * beta);
    for (int j = 0; j < maxit; ++j) {
      const int m = j + 1;
      TRY(ensure_vec(ctx->Z, store_z ? j : 0));
      TRY(ensure_vec(ctx->V, j + 1));
      double* const zj = ctx->Z[store_z ? j : 0];
      // basis pointers and scales for this iteration (small H2D copies, stream ordered)
      std::memcpy(ctx->h_pin, inv_nsq.data(), m * sizeof(double));
      CK(cudaMemcpyAsync(ctx->d_coef + oinv, ctx->h_pin, m * sizeof(double), cudaMemcpyHostToDevice, s));
      const double* const* hV = (const double* const*)ctx->V.data();
      // z~_j = M V~_j : one V-cycle from zero
      CK(cudaEventRecord(ctx->ev[0], s));
      if (ctx->cfg.precond == SVK_PRECOND_BLOCK_TRIANGULAR) TRY(op_bt(ctx, ctx->V[j], zj, s));
      else TRY(op_precond_mg(ctx, ctx->V[j], zj, s));
      CK(cudaEventRecord(ctx->ev[1], s));
      // w~ = A z~_j ; classical Gram-Schmidt pass against V~_0..V~_j (its dot
      // pass also yields |w~|^2) ; V~_j+1 = w~' with |w~'|
      TRY(op_residual(ctx, L, zj, nullptr, ctx->d_w, s));
      dlist.assign(hV, hV + m);
      dlist.push_back(ctx->d_w);
      TRY(cgs_dots(ctx, dlist.data(), m + 1, ctx->d_w, S, oraw, s));
      launch_pdl(k_scale_coef, dim3((m + 63) / 64), dim3(64), 0, s, (const double*)(ctx->d_coef + oraw), (const double*)(ctx->d_coef + oinv), ctx->d_coef + o1, m);
      CKL();
      TRY(cgs_update(ctx, hV, m, o1, ctx->d_w, ctx->V[j + 1], n, S, onrm, s));
      CK(cudaEventRecord(ctx->ev[2], s));
      TRY(readback(ctx, ctx->d_coef, (onrm + 1), s));
      TRY(harvest_graph_prof(ctx));
      if (ctx->tr && ctx->tr->async_error(ctx->err) != 0) return SVK_ERR_NCCL;  // polled once per iteration
      float a01 = 0, a12 = 0;
      cudaEventElapsedTime(&a01, ctx->ev[0], ctx->ev[1]);
      cudaEventElapsedTime(&a12, ctx->ev[1], ctx->ev[2]);
      tv += a01 * 1e-3;
      to += a12 * 1e-3;
      // second pass: always (CGS2) or when the first pass cancelled more than kappa (DGKS-type test)
      const double wn2 = ctx->h_pin[oraw + m], wp2 = ctx->h_pin[onrm];
      if (ctx->cfg.orth == SVK_ORTH_CGS2 || !(wp2 * kReorthKappa * kReorthKappa >= wn2)) {
        CK(cudaEventRecord(ctx->ev[3], s));
        TRY(cgs_dots(ctx, hV, m, ctx->V[j + 1], S, oraw, s));
        launch_pdl(k_scale_coef, dim3((m + 63) / 64), dim3(64), 0, s, (const double*)(ctx->d_coef + oraw), (const double*)(ctx->d_coef + oinv), ctx->d_coef + o2, m);
        CKL();
        TRY(cgs_update(ctx, hV, m, o2, ctx->V[j + 1], ctx->V[j + 1], n, S, onrm, s));
        CK(cudaEventRecord(ctx->ev[4], s));
        TRY(readback(ctx, ctx->d_coef, (onrm + 1), s));
        float a34 = 0;
        cudaEventElapsedTime(&a34, ctx->ev[3], ctx->ev[4]);
        to += a34 * 1e-3;
        ++n_reorth;
      } else {
        for (int i = 0; i < m; ++i) ctx->h_pin[o2 + i] = 0.0;
      }
      for (int i = 0; i <= j; ++i) Hij(i, j) = (ctx->h_pin[o1 + i] + ctx->h_pin[o2 + i]) * nv[i] / nv[j];
      const double nn = std::sqrt(std::max(ctx->h_pin[onrm], 0.0));
      const double hn = nn / nv[j];
      if (!std::isfinite(hn)) {
        status = SVK_ERR_NONFINITE;
        ctx->err = "non-finite Arnoldi vector";
        k = j;
        break;
      }
      nv[j + 1] = nn;
      if (j + 1 <= maxit) inv_nsq[j + 1] = nn > 0 ? 1.0 / (nn * nn) : 0.0;
      Hij(j + 1, j) = hn;
      for (int i = 0; i < j; ++i) {
        const double t = cs[i] * Hij(i, j) + sn[i] * Hij(i + 1, j);
        Hij(i + 1, j) = -sn[i] * Hij(i, j) + cs[i] * Hij(i + 1, j);
        Hij(i, j) = t;
      }
      const double a = Hij(j, j), bb = Hij(j + 1, j), rr = std::hypot(a, bb);
      cs[j] = a / rr;
      sn[j] = bb / rr;
      Hij(j, j) = rr;
      Hij(j + 1, j) = 0.0;
      gv[j + 1] = -sn[j] * gv[j];
      gv[j] = cs[j] * gv[j];
      const double est = std::fabs(gv[j + 1]) / beta;
      if (hist) hist[j + 1] = est;
      k = j + 1;
      if (est <= rtol || hn == 0.0) {
        conv = true;
        break;
      }
    }
    if (k > 0) {  // x += sum_i (y_i / n_i) Z~_i  (as w_out = w - sum c_i V_i with c_i = -y_i / n_i)
      std::vector<double> y(k);
      for (int i = k - 1; i >= 0; --i) {
        double t = gv[i];
        for (int mm = i + 1; mm < k; ++mm) t -= Hij(i, mm) * y[mm];
        y[i] = t / Hij(i, i);
      }
      for (int i = 0; i < k; ++i) ctx->h_pin[i] = -y[i] / nv[i];
      CK(cudaMemcpyAsync(ctx->d_coef + o1, ctx->h_pin, k * sizeof(double), cudaMemcpyHostToDevice, s));
      if (store_z) {
        for (int c0 = 0; c0 < k; c0 += kCgsMax) {
          const int mm = std::min(kCgsMax, k - c0);
          k_cgs_update<<<kDotBlocks, kRedThreads, 0, s>>>(veclist((const double* const*)ctx->Z.data() + c0, mm), mm,
                                                           ctx->d_coef + o1 + c0, x, x, S, ctx->d_part);
          CKL();
        }
      } else {  // x += M (sum_i (y_i / n_i) V~_i): u in d_w (w_out = 0 - sum c_i V~_i), then one V-cycle
        TRY(op_zero_level(ctx, L, ctx->d_w, s));
        for (int c0 = 0; c0 < k; c0 += kCgsMax) {
          const int mm = std::min(kCgsMax, k - c0);
          k_cgs_update<<<kDotBlocks, kRedThreads, 0, s>>>(veclist((const double* const*)ctx->V.data() + c0, mm), mm,
                                                           ctx->d_coef + o1 + c0, ctx->d_w, ctx->d_w, S, ctx->d_part);
          CKL();
        }
        TRY(op_halo(ctx, L, ctx->d_w, s));
        TRY(op_precond_mg(ctx, ctx->d_w, ctx->Z[0], s));
        ctx->h_pin[0] = -1.0;
        CK(cudaMemcpyAsync(ctx->d_coef + o1, ctx->h_pin, sizeof(double), cudaMemcpyHostToDevice, s));
        const double* zl[1] = {ctx->Z[0]};
        k_cgs_update<<<kDotBlocks, kRedThreads, 0, s>>>(veclist(zl, 1), 1, ctx->d_coef + o1, x, x, S, ctx->d_part);
        CKL();
      }
    }
  }
  double rn = 0.0;
  if (beta > 0) {
    TRY(op_halo(ctx, L, x, s));
    TRY(op_residual(ctx, L, x, b, ctx->d_r, s));
    TRY(host_norm(ctx, ctx->d_r, S, &rn, s));
  }
  R.iterations = k;
  R.n_reorth = n_reorth;
  R.converged = conv ? 1 : 0;
  R.rel_residual = beta > 0 ? rn / beta : 0.0;
  R.t_vcycle_s = tv;
  R.t_orth_s = to;
  R.t_total_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  R.t_setup_s = ctx->t_setup_s;
  if (status == SVK_OK && !conv) status = SVK_NOT_CONVERGED;
  if (status == SVK_OK && !std::isfinite(R.rel_residual)) status = SVK_ERR_NONFINITE;
  R.status = status;
  if (rep) *rep = R;
  return status;
}

int free_ctx(svk_ctx* ctx) {
  auto F = [ctx](void* p) {  // alloc_vec blocks go back to their allocator
    if (!p) return;
    if (ctx->plain_bytes.count((const double*)p))
      free_vec(ctx, (double*)p);
    else
      cudaFree(p);
  };
  F(ctx->d_Ns);
  F(ctx->d_inv);
  F(ctx->d_fac);
  F(ctx->d_cmat);
  F(ctx->d_cidx);
  for (auto* v : {&ctx->ws_x, &ctx->ws_t, &ctx->ws_r, &ctx->ws_b})
    for (double* p : *v) free_vec(ctx, p);
  F(ctx->d_dbuf);
  for (double* p : ctx->d_inv_simple) F(p);
  F(ctx->d_bd);
  F(ctx->d_sc);
  for (BdTile* p : ctx->d_sc_tiles) F(p);
  for (BdTile* p : ctx->d_tiles) F(p);
  free_vec(ctx, ctx->d_sw);
  F(ctx->d_schur);
  F(ctx->d_btb);
  F(ctx->d_bt_invL);
  F(ctx->d_bt_invM);
  F(ctx->d_bt_idxL);
  F(ctx->d_bt_idxM);
  for (auto* v : {&ctx->p_rhs, &ctx->p_dp0, &ctx->p_dp1})
    for (double* p : *v) F(p);
  for (double* p : ctx->V) free_vec(ctx, p);
  for (double* p : ctx->Z) free_vec(ctx, p);
  F(ctx->d_agg);
  free_vec(ctx, ctx->d_w);
  free_vec(ctx, ctx->d_r);
  F(ctx->d_part);
  F(ctx->d_coef);
  F(ctx->d_hb);
  F(ctx->d_hx);
  F(ctx->d_hb2);
  F(ctx->d_hx2);
  for (int q = 0; q < 2; ++q) {
    F(ctx->d_cin[q][0]);
    F(ctx->d_cin[q][1]);
    F(ctx->d_cout[q]);
  }
  for (cudaEvent_t* e : {ctx->ev_in, ctx->ev_solved, ctx->ev_out})
    for (int k = 0; k < 2; ++k)
      if (e[k]) cudaEventDestroy(e[k]);
  if (ctx->s_in) cudaStreamDestroy(ctx->s_in);
  if (ctx->s_out) cudaStreamDestroy(ctx->s_out);
  if (ctx->h_pin) cudaFreeHost(ctx->h_pin);
  for (auto e : ctx->prof_ev) cudaEventDestroy(e);
  for (auto& gr : ctx->graphs) {
    if (gr->exec) cudaGraphExecDestroy(gr->exec);
    for (auto& pr : gr->ev) {
      cudaEventDestroy(pr.first);
      cudaEventDestroy(pr.second);
    }
  }
  if (ctx->cap_stream) cudaStreamDestroy(ctx->cap_stream);
  for (auto& e : ctx->ev)
    if (e) cudaEventDestroy(e);
  delete ctx;
  return SVK_OK;
}

int create_impl(svk_ctx* ctx) {
  const svk_config& c = ctx->cfg;
  CK(cudaSetDevice(c.device));
  {
    std::lock_guard<std::mutex> lk(g_tab_mu);
    if (c.device < 0 || c.device >= 64) {
      ctx->err = "device ordinal out of range";
      return SVK_ERR_INVALID;
    }
    if (!g_tab_done[c.device]) {
      StencilConst t;
      if (!build_tables(t, ctx->err)) return SVK_ERR_INVALID;
      CK(cudaMemcpyToSymbol(c_st, &t, sizeof(t)));
      g_tab_done[c.device] = true;
    }
  }
  // hierarchy N0, 2 N0, ..., N (level 0 coarsest)
  std::vector<int> Ns;
  for (int N = c.n_coarse; N <= c.n_elem; N *= 2) Ns.push_back(N);
  ctx->nlev = (int)Ns.size();
  for (int N : Ns) ctx->g.push_back(make_geom(N));
  // row slabs (dist.cuh).  Without a distributed level every rank runs the whole
  // problem redundantly and no transport is created.
  if (c.nranks > 1) {
    ctx->la = first_dist_level(Ns, c.nranks, c.agglom_rows);
    if (ctx->la < ctx->nlev) {
      for (int l = ctx->la; l < ctx->nlev; ++l)
        slab_rows(Ns[l], Ns[ctx->la], c.nranks, c.rank, &ctx->g[l].r0, &ctx->g[l].r1);
      if (c.transport == SVK_TRANSPORT_NCCL) {
        auto* t = new NcclTransport(c.rank, c.nranks);
        ctx->tr.reset(t);
        if (t->init(c.nccl_id, ctx->err) != 0) return SVK_ERR_NCCL;
      } else {
        ctx->tr.reset(new EmulTransport(c.rank, c.nranks, c.emul_group));
      }
    }
    const char* pz = std::getenv("SVK_POISON_HALO");
    ctx->poison = pz && pz[0] == '1';
    const char* sl = std::getenv("SVK_SLAB_LOCAL");
    ctx->slab_local = !(sl && sl[0] == '0');
  }
  CK(cudaMalloc(&ctx->d_Ns, Ns.size() * sizeof(int)));
  CK(cudaMemcpy(ctx->d_Ns, Ns.data(), Ns.size() * sizeof(int), cudaMemcpyHostToDevice));
  for (int k = 0; k < 6; ++k) CK(cudaEventCreate(&ctx->ev[k]));
  // patch setup: 25 groups x levels, one CTA each
  int* d_status;
  CK(cudaMalloc(&d_status, sizeof(int)));
  CK(cudaMemset(d_status, 0, sizeof(int)));
  CK(cudaMalloc(&ctx->d_inv, (size_t)ctx->nlev * 25 * kGroupStride * sizeof(double)));
  k_patch_setup<<<dim3(25, ctx->nlev), 256>>>(ctx->d_Ns, c.nu, ctx->d_inv, d_status);
  CKL();
  CK(cudaMalloc(&ctx->d_fac, (size_t)ctx->nlev * kFacStride * sizeof(double)));
  TRY(launch_factor_setup(ctx->d_Ns, ctx->nlev, c.nu, ctx->d_inv, ctx->d_fac, d_status));
  CKL();
  if (const char* cg = std::getenv("SVK_TEST_CORRUPT_GROUP")) {  // test aid: "level,group,slot"
    int cl = -1, cgp = -1, cq = -1;
    if (std::sscanf(cg, "%d,%d,%d", &cl, &cgp, &cq) == 3 && cl >= 0 && cl < ctx->nlev && cgp >= 0 && cgp < 25 &&
        cq >= 0 && cq < kGroupStride) {
      double* e = ctx->d_inv + ((size_t)cl * 25 + cgp) * kGroupStride + cq;
      double v;
      CK(cudaMemcpy(&v, e, sizeof(double), cudaMemcpyDeviceToHost));
      v += 1e-8 * (1.0 + std::fabs(v));  // far above the 1e-12 validation tolerance
      CK(cudaMemcpy(e, &v, sizeof(double), cudaMemcpyHostToDevice));
    }
  }
  // level-0 bordered pseudo-inverse
  const LevelGeom& g0 = ctx->g[0];
  std::vector<int> idx;
  for (int comp = 0; comp < 2; ++comp)
    for (int j = 1; j < g0.lat - 1; ++j)
      for (int i = 1; i < g0.lat - 1; ++i) idx.push_back((int)((comp ? g0.ouy : g0.oux) + (int64_t)j * g0.pu + i));
  for (int ky = 0; ky <= g0.N; ++ky)
    for (int kx = 0; kx <= g0.N; ++kx) idx.push_back((int)p_at(g0, kx, ky));
  ctx->cni = (int)idx.size();
  const int nb = ctx->cni + 1;
  CK(cudaMalloc(&ctx->d_cidx, idx.size() * sizeof(int)));
  CK(cudaMemcpy(ctx->d_cidx, idx.data(), idx.size() * sizeof(int), cudaMemcpyHostToDevice));
  CK(cudaMalloc(&ctx->d_cmat, (size_t)nb * nb * sizeof(double)));
  k_coarse_build<<<nb, 128>>>(g0, c.nu, ctx->d_cidx, ctx->cni, ctx->d_cmat);
  CKL();
  int* d_perm;
  double* d_colk;
  CK(cudaMalloc(&d_perm, nb * sizeof(int)));
  CK(cudaMalloc(&d_colk, nb * sizeof(double)));
  k_coarse_invert<<<1, 256>>>(ctx->d_cmat, nb, d_perm, d_colk, d_status);
  CKL();
  int hs = 0;
  CK(cudaMemcpy(&hs, d_status, sizeof(int), cudaMemcpyDeviceToHost));
  ctx->h_fac.resize(ctx->nlev);
  CK(cudaMemcpy(ctx->h_fac.data(), ctx->d_fac, (size_t)ctx->nlev * sizeof(FusedFactors), cudaMemcpyDeviceToHost));
  CK(cudaDeviceGetAttribute(&ctx->nsm, cudaDevAttrMultiProcessorCount, c.device));
  cudaFree(d_perm);
  cudaFree(d_colk);
  cudaFree(d_status);
  if (hs) {
    ctx->err = "singular patch or coarse matrix";
    return SVK_ERR_SINGULAR;
  }
  // workspaces
  ctx->ws_x.assign(ctx->nlev, nullptr);
  ctx->ws_t.assign(ctx->nlev, nullptr);
  ctx->ws_r.assign(ctx->nlev, nullptr);
  ctx->ws_b.assign(ctx->nlev, nullptr);
  for (int l = 0; l < ctx->nlev; ++l) {
    if (l < ctx->nlev - 1) {
      TRY(alloc_level_vec(ctx, l, &ctx->ws_x[l]));
      TRY(alloc_level_vec(ctx, l, &ctx->ws_b[l]));
    }
    TRY(alloc_level_vec(ctx, l, &ctx->ws_t[l]));
    TRY(alloc_level_vec(ctx, l, &ctx->ws_r[l]));
  }
  TRY(alloc_vec(ctx, &ctx->d_bd, (int64_t)kSlots * bd_count(ctx->g.back().N)));
  for (int l = 0; l < ctx->nlev; ++l) {
    const std::vector<BdTile> t = make_bd_tiles(ctx->g[l].N);
    BdTile* d = nullptr;
    CK(cudaMalloc(&d, t.size() * sizeof(BdTile)));
    ctx->d_tiles.push_back(d);
    ctx->ntiles.push_back((int)t.size());
    CK(cudaMemcpy(d, t.data(), t.size() * sizeof(BdTile), cudaMemcpyHostToDevice));
  }
  TRY(setup_small_cycle(ctx));
  if (c.sweep_impl == SVK_SWEEP_SIMPLE) {  // simple Vanka: build and store every patch's inverse
    int* d_st;
    CK(cudaMalloc(&d_st, sizeof(int)));
    CK(cudaMemset(d_st, 0, sizeof(int)));
    for (int l = 0; l < ctx->nlev; ++l) {
      const int64_t np = (int64_t)(ctx->g[l].N + 1) * (ctx->g[l].N + 1);
      double* p = nullptr;
      if (cudaMalloc(&p, (size_t)np * kGroupStride * sizeof(double)) != cudaSuccess) {
        cudaGetLastError();
        cudaFree(d_st);
        ctx->err = "simple Vanka: per-patch inverses do not fit in device memory";
        return SVK_ERR_CUDA;
      }
      ctx->d_inv_simple.push_back(p);
      for (int64_t p0 = 0; p0 < np; p0 += (1 << 30))
        k_patch_setup_simple<<<(unsigned)std::min<int64_t>(np - p0, 1 << 30), 128>>>(ctx->g[l], c.nu, p0, p, d_st,
                                                                                      np, 0);
      CKL();
    }
    int hst = 0;
    CK(cudaMemcpy(&hst, d_st, sizeof(int), cudaMemcpyDeviceToHost));
    cudaFree(d_st);
    if (hst) {
      ctx->err = "simple Vanka: singular patch matrix";
      return SVK_ERR_SINGULAR;
    }
  }
  if (c.sweep_impl == SVK_SWEEP_UNFUSED || c.sweep_impl == SVK_SWEEP_SIMPLE) {
    const LevelGeom& gf = ctx->g.back();
    TRY(alloc_vec(ctx, &ctx->d_dbuf, (int64_t)kSlots * (gf.N + 1) * (gf.N + 1)));
  }
  CK(cudaMalloc(&ctx->d_part, (size_t)(kCgsMax + 1) * kDotBlocks * sizeof(double)));
  if (c.precond == SVK_PRECOND_BLOCK_TRIANGULAR) {  // level-0 block inverses + finest rhs buffer
    StencilConst t;
    if (!build_tables(t, ctx->err)) return SVK_ERR_INVALID;
    std::vector<double> iL, iM;
    std::vector<int> xL, xM;
    if (!build_bt_coarse(t, ctx->g[0], c.nu, iL, xL, iM, xM)) {
      ctx->err = "block-triangular: singular level-0 block";
      return SVK_ERR_SINGULAR;
    }
    ctx->bt_niL = (int)xL.size();
    ctx->bt_niM = (int)xM.size();
    CK(cudaMalloc(&ctx->d_bt_invL, iL.size() * sizeof(double)));
    CK(cudaMalloc(&ctx->d_bt_invM, iM.size() * sizeof(double)));
    CK(cudaMalloc(&ctx->d_bt_idxL, xL.size() * sizeof(int)));
    CK(cudaMalloc(&ctx->d_bt_idxM, xM.size() * sizeof(int)));
    CK(cudaMemcpy(ctx->d_bt_invL, iL.data(), iL.size() * sizeof(double), cudaMemcpyHostToDevice));
    CK(cudaMemcpy(ctx->d_bt_invM, iM.data(), iM.size() * sizeof(double), cudaMemcpyHostToDevice));
    CK(cudaMemcpy(ctx->d_bt_idxL, xL.data(), xL.size() * sizeof(int), cudaMemcpyHostToDevice));
    CK(cudaMemcpy(ctx->d_bt_idxM, xM.data(), xM.size() * sizeof(int), cudaMemcpyHostToDevice));
    TRY(alloc_vec(ctx, &ctx->d_btb, ctx->g.back().len));
  }
  if (c.relax != SVK_RELAX_VANKA) {  // comparator workspaces: S stencils + pressure-plane buffers
    StencilConst t;
    if (!build_tables(t, ctx->err)) return SVK_ERR_INVALID;
    std::vector<double> h((size_t)ctx->nlev * kSchurStride);
    for (int l = 0; l < ctx->nlev; ++l) build_schur_stencils(t, ctx->g[l].N, c.nu, c.relax_t, &h[(size_t)l * kSchurStride]);
    CK(cudaMalloc(&ctx->d_schur, h.size() * sizeof(double)));
    CK(cudaMemcpy(ctx->d_schur, h.data(), h.size() * sizeof(double), cudaMemcpyHostToDevice));
    for (int l = 0; l < ctx->nlev; ++l) {
      const int64_t np = (int64_t)(ctx->g[l].N + 1) * ctx->g[l].pp;
      for (auto* v : {&ctx->p_rhs, &ctx->p_dp0, &ctx->p_dp1}) {
        double* p;
        TRY(alloc_vec(ctx, &p, np));
        v->push_back(p);
      }
    }
  }
  if (c.validate) {  // validation mode: every patch of every level against its group
    for (int l = 0; l < ctx->nlev; ++l) {
      double dev = 0.0;
      int64_t n = 0;
      TRY(op_validate(ctx, l, &dev, &n));
      if (!(dev <= kValidateTol)) {
        char buf[160];
        std::snprintf(buf, sizeof buf, "validation: patch inverses deviate from their group by %.3e on level %d", dev, l);
        ctx->err = buf;
        return SVK_ERR_VALIDATION;
      }
    }
  }
  CK(cudaDeviceSynchronize());
  return SVK_OK;
}

}  // namespace

// =============================================================================
// C ABI
// =============================================================================
// Every entry point that takes a context runs on the context's device (the
// caller's current device is restored on return) and maps C++ exceptions to
// status codes, so none crosses the extern "C" boundary.
template <class F>
int guarded(svk_ctx* ctx, F&& f) {
  if (!ctx) return SVK_ERR_INVALID;
  int prev = -1;
  if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
  if (prev != ctx->cfg.device && cudaSetDevice(ctx->cfg.device) != cudaSuccess) {
    ctx->err = "cudaSetDevice failed";
    return SVK_ERR_CUDA;
  }
  int st;
  try {
    st = f();
  } catch (const std::bad_alloc&) {
    ctx->err = "host allocation failed";
    st = SVK_ERR_ALLOC;
  } catch (const std::exception& e) {
    ctx->err = std::string("exception: ") + e.what();
    st = SVK_ERR_INVALID;
  } catch (...) {
    ctx->err = "unknown exception";
    st = SVK_ERR_INVALID;
  }
  if (prev >= 0 && prev != ctx->cfg.device) cudaSetDevice(prev);
  return st;
}

extern "C" {

int svk_config_default(svk_config* cfg, int32_t n_elem) {
  if (!cfg) return SVK_ERR_INVALID;
  std::memset(cfg, 0, sizeof(*cfg));
  cfg->n_elem = n_elem;
  cfg->n_coarse = 4;
  cfg->nu = 1.0;
  cfg->omega_v = 0.8;
  cfg->weighting = SVK_WEIGHT_MULT;
  cfg->nu_pre = 1;
  cfg->nu_post = 1;
  cfg->coarse = SVK_COARSE_EXACT;
  cfg->sweep_impl = SVK_SWEEP_FUSED;
  cfg->device = 0;
  cfg->rank = 0;
  cfg->nranks = 1;
  cfg->transport = SVK_TRANSPORT_NONE;
  cfg->agglom_rows = 64;
  cfg->orth = SVK_ORTH_ADAPTIVE;
  cfg->relax = SVK_RELAX_VANKA;
  cfg->relax_t = 1.0;
  cfg->relax_omega = 1.0;
  cfg->jacobi_omega = 0.8;
  cfg->jacobi_sweeps = 3;
  cfg->precond = SVK_PRECOND_MG;
  cfg->bt_cycles = 3;
  cfg->bt_nu = 3;
  cfg->bt_omega_u = 1.0;
  cfg->bt_omega_p = 0.6;
  cfg->krylov_store_z = 1;
  return SVK_OK;
}

int svk_create(const svk_config* cfg, svk_ctx** out) {
  if (!out) return SVK_ERR_INVALID;
  *out = nullptr;
  if (!cfg) return SVK_ERR_INVALID;
  if (cfg->n_coarse < 4 || cfg->n_elem < cfg->n_coarse || cfg->nu <= 0 || cfg->nu_pre < 0 || cfg->nu_post < 0 ||
      cfg->n_elem > (1 << 15))
    return SVK_ERR_INVALID;
  int n = cfg->n_elem;
  while (n > cfg->n_coarse) {
    if (n % 2) return SVK_ERR_INVALID;
    n /= 2;
  }
  if (n != cfg->n_coarse) return SVK_ERR_INVALID;
  if (cfg->nranks < 1 || cfg->rank < 0 || cfg->rank >= cfg->nranks) return SVK_ERR_INVALID;
  if (cfg->orth != SVK_ORTH_ADAPTIVE && cfg->orth != SVK_ORTH_CGS2) return SVK_ERR_INVALID;
  if (cfg->relax < SVK_RELAX_VANKA || cfg->relax > SVK_RELAX_SCHUR_UZAWA) return SVK_ERR_INVALID;
  if (cfg->sweep_impl < SVK_SWEEP_FUSED || cfg->sweep_impl > SVK_SWEEP_SIMPLE) return SVK_ERR_INVALID;
  if (cfg->precond < SVK_PRECOND_MG || cfg->precond > SVK_PRECOND_BLOCK_TRIANGULAR) return SVK_ERR_INVALID;
  if (cfg->precond == SVK_PRECOND_BLOCK_TRIANGULAR && (cfg->nranks > 1 || cfg->bt_cycles < 1 || cfg->bt_nu < 0))
    return SVK_ERR_INVALID;  // single-GPU comparator
  if (cfg->relax != SVK_RELAX_VANKA && (cfg->nranks > 1 || !(cfg->relax_t > 0) || cfg->jacobi_sweeps < 0))
    return SVK_ERR_INVALID;  // the comparators are single-GPU
  if (cfg->nranks > 1 && (cfg->agglom_rows < kHalo || cfg->sweep_impl != SVK_SWEEP_FUSED ||
                          (cfg->transport != SVK_TRANSPORT_NCCL && cfg->transport != SVK_TRANSPORT_EMULATED)))
    return SVK_ERR_INVALID;
  if ((cfg->alloc_fn == nullptr) != (cfg->free_fn == nullptr)) return SVK_ERR_INVALID;
  const auto t0 = std::chrono::steady_clock::now();
  svk_ctx* ctx = new svk_ctx;
  ctx->cfg = *cfg;
  int st = guarded(ctx, [&]() -> int { return create_impl(ctx); });
  ctx->t_setup_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  if (st != SVK_OK) {
    std::fprintf(stderr, "svk_create: %s\n", ctx->err.c_str());
    free_ctx(ctx);
    return st;
  }
  *out = ctx;
  return SVK_OK;
}

int svk_destroy(svk_ctx* ctx) {
  if (!ctx) return SVK_ERR_INVALID;
  int prev = -1;
  if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
  const int dev = ctx->cfg.device;
  cudaSetDevice(dev);
  cudaDeviceSynchronize();
  const int st = free_ctx(ctx);
  if (prev >= 0 && prev != dev) cudaSetDevice(prev);
  return st;
}

int svk_num_levels(const svk_ctx* ctx, int32_t* levels) {
  if (!ctx || !levels) return SVK_ERR_INVALID;
  *levels = ctx->nlev;
  return SVK_OK;
}

int svk_level_info(const svk_ctx* ctx, int32_t level, svk_level* out) {
  if (!ctx || !out || level < 0 || level >= ctx->nlev) return SVK_ERR_INVALID;
  const LevelGeom& g = ctx->g[level];
  out->N = g.N;
  out->lat = g.lat;
  out->vec_len = g.len;
  out->off_ux = g.oux;
  out->off_uy = g.ouy;
  out->off_p = g.op;
  out->pitch_u = g.pu;
  out->pitch_p = g.pp;
  out->n_dof = 2 * (int64_t)g.lat * g.lat + (int64_t)(g.N + 1) * (g.N + 1);
  out->n_patch = (int64_t)(g.N + 1) * (g.N + 1);
  out->row0 = g.r0;
  out->row1 = g.r1;
  out->distributed = dist_level(ctx, level) ? 1 : 0;
  out->halo_rows = out->distributed ? kHalo : 0;
  return SVK_OK;
}

int svk_set_problem(svk_ctx* ctx, int32_t level, int32_t kind, double* b, double* x0, void* stream) {
  return guarded(ctx, [&]() -> int {
    TRY(valid_level(ctx, level));
    if (kind < 0 || kind > 3) return SVK_ERR_INVALID;
    if (b) TRY(valid_ptr(ctx, b, "b"));
    if (x0) TRY(valid_ptr(ctx, x0, "x0"));
    const LevelGeom& g = ctx->g[level];
    cudaStream_t s = (cudaStream_t)stream;
    if (b) CK(cudaMemsetAsync(b, 0, g.len * sizeof(double), s));
    if (x0) CK(cudaMemsetAsync(x0, 0, g.len * sizeof(double), s));
    k_set_problem<<<plane_grid(g), kPlaneBlock, 0, s>>>(g, kind, ctx->cfg.nu, b, x0);
    CKL();
    return SVK_OK;
  });
}

int svk_residual(svk_ctx* ctx, int32_t level, const double* x, const double* b, double* r, void* stream) {
  return guarded(ctx, [&]() -> int {
    TRY(valid_level(ctx, level));
    TRY(valid_ptr(ctx, x, "x"));
    TRY(valid_ptr(ctx, b, "b"));
    TRY(valid_ptr(ctx, r, "r"));
    TRY(op_halo(ctx, level, const_cast<double*>(x), (cudaStream_t)stream));
    return op_residual(ctx, level, x, b, r, (cudaStream_t)stream);
  });
}

int svk_matvec(svk_ctx* ctx, int32_t level, const double* x, double* y, void* stream) {
  return guarded(ctx, [&]() -> int {
    TRY(valid_level(ctx, level));
    TRY(valid_ptr(ctx, x, "x"));
    TRY(valid_ptr(ctx, y, "y"));
    TRY(op_halo(ctx, level, const_cast<double*>(x), (cudaStream_t)stream));
    return op_residual(ctx, level, x, nullptr, y, (cudaStream_t)stream);
  });
}

int svk_vanka_sweep(svk_ctx* ctx, int32_t level, const double* x_in, const double* b, double* x_out, int32_t nsweeps,
                    void* stream) {
  return guarded(ctx, [&]() -> int {
    TRY(valid_level(ctx, level));
    TRY(valid_ptr(ctx, x_in, "x_in"));
    TRY(valid_ptr(ctx, b, "b"));
    TRY(valid_ptr(ctx, x_out, "x_out"));
    if (nsweeps < 1 || x_in == x_out || b == x_out) {
      ctx->err = "nsweeps < 1 or aliasing x_out";
      return SVK_ERR_INVALID;
    }
    cudaStream_t s = (cudaStream_t)stream;
    const LevelGeom& g = ctx->g[level];
    if (ctx->cfg.sweep_impl != SVK_SWEEP_FUSED && !ctx->d_dbuf) return SVK_ERR_INVALID;
    TRY(op_halo(ctx, level, const_cast<double*>(b), s));
    TRY(op_halo(ctx, level, const_cast<double*>(x_in), s));
    if (nsweeps == 1) return op_sweep(ctx, level, x_in, b, x_out, false, s);
    if (!ctx->d_sw) TRY(alloc_level_vec(ctx, ctx->nlev - 1, &ctx->d_sw));
    // ping-pong so that the last sweep lands in x_out
    double* bufs[2] = {x_out, ctx->d_sw};
    int dst = (nsweeps % 2 == 1) ? 0 : 1;
    const double* cur = x_in;
    for (int k = 0; k < nsweeps; ++k) {
      if (k > 0) TRY(op_halo(ctx, level, const_cast<double*>(cur), s));
      TRY(op_sweep(ctx, level, cur, b, bufs[dst], false, s));
      cur = bufs[dst];
      dst ^= 1;
    }
    (void)g;
    return SVK_OK;
  });
}

int svk_relax_sweep(svk_ctx* ctx, int32_t level, const double* x_in, const double* b, double* x_out, void* stream) {
  return guarded(ctx, [&]() -> int {
    TRY(valid_level(ctx, level));
    TRY(valid_ptr(ctx, x_in, "x_in"));
    TRY(valid_ptr(ctx, b, "b"));
    TRY(valid_ptr(ctx, x_out, "x_out"));
    if (x_in == x_out || b == x_out) {
      ctx->err = "x_out aliases x_in or b";
      return SVK_ERR_INVALID;
    }
    if (ctx->cfg.relax == SVK_RELAX_VANKA) return svk_vanka_sweep(ctx, level, x_in, b, x_out, 1, stream);
    return op_bs(ctx, level, x_in, b, x_out, false, (cudaStream_t)stream);
  });
}

int svk_precond_apply(svk_ctx* ctx, const double* b, double* z, void* stream) {
  return guarded(ctx, [&]() -> int {
    if (!ctx) return SVK_ERR_INVALID;
    TRY(valid_ptr(ctx, b, "b"));
    TRY(valid_ptr(ctx, z, "z"));
    if (b == z) {
      ctx->err = "z aliases b";
      return SVK_ERR_INVALID;
    }
    cudaStream_t s = (cudaStream_t)stream;
    const int L = ctx->nlev - 1;
    if (ctx->cfg.precond == SVK_PRECOND_BLOCK_TRIANGULAR) return op_bt(ctx, b, z, s);
    TRY(op_halo(ctx, L, const_cast<double*>(b), s));
    return op_mg(ctx, L, b, z, true, s);
  });
}

int svk_restrict(svk_ctx* ctx, int32_t level, const double* r_fine, double* r_coarse, void* stream) {
  return guarded(ctx, [&]() -> int {
    TRY(valid_level(ctx, level));
    if (level < 1) return SVK_ERR_INVALID;
    TRY(valid_ptr(ctx, r_fine, "r_fine"));
    TRY(valid_ptr(ctx, r_coarse, "r_coarse"));
    return op_restrict(ctx, level, r_fine, r_coarse, (cudaStream_t)stream);
  });
}

int svk_residual_restrict(svk_ctx* ctx, int32_t level, const double* x, const double* b, double* r_coarse,
                          void* stream) {
  return guarded(ctx, [&]() -> int {
    TRY(valid_level(ctx, level));
    if (level < 1) return SVK_ERR_INVALID;
    TRY(valid_ptr(ctx, x, "x"));
    TRY(valid_ptr(ctx, b, "b"));
    TRY(valid_ptr(ctx, r_coarse, "r_coarse"));
    if (r_coarse == x || r_coarse == b) {
      ctx->err = "r_coarse aliases an input";
      return SVK_ERR_INVALID;
    }
    cudaStream_t s = (cudaStream_t)stream;
    TRY(op_halo(ctx, level, const_cast<double*>(x), s));
    TRY(op_halo(ctx, level, const_cast<double*>(b), s));
    TRY(op_residual_restrict(ctx, level, x, b, r_coarse, s));
    if (dist_level(ctx, level) && !dist_level(ctx, level - 1)) TRY(op_agglomerate(ctx, level, r_coarse, s));
    return SVK_OK;
  });
}

int svk_prolong_add(svk_ctx* ctx, int32_t level, const double* e_coarse, double* x_fine, void* stream) {
  return guarded(ctx, [&]() -> int {
    TRY(valid_level(ctx, level));
    if (level < 1) return SVK_ERR_INVALID;
    TRY(valid_ptr(ctx, e_coarse, "e_coarse"));
    TRY(valid_ptr(ctx, x_fine, "x_fine"));
    return op_prolong_add(ctx, level, e_coarse, x_fine, (cudaStream_t)stream);
  });
}

int svk_coarse_solve(svk_ctx* ctx, const double* b, double* x, void* stream) {
  return guarded(ctx, [&]() -> int {
    if (!ctx) return SVK_ERR_INVALID;
    TRY(valid_ptr(ctx, b, "b"));
    TRY(valid_ptr(ctx, x, "x"));
    return op_coarse(ctx, b, x, (cudaStream_t)stream);
  });
}

int svk_vcycle(svk_ctx* ctx, const double* b, double* x, void* stream) {
  return guarded(ctx, [&]() -> int {
    if (!ctx) return SVK_ERR_INVALID;
    TRY(valid_ptr(ctx, b, "b"));
    TRY(valid_ptr(ctx, x, "x"));
    if (b == x) return SVK_ERR_INVALID;
    return op_mg(ctx, ctx->nlev - 1, b, x, false, (cudaStream_t)stream);
  });
}

int svk_fgmres(svk_ctx* ctx, const double* b, double* x, double rtol, int32_t maxit, double* hist, svk_report* rep,
               void* stream) {
  return guarded(ctx, [&]() -> int {
    if (!ctx) return SVK_ERR_INVALID;
    TRY(valid_ptr(ctx, b, "b"));
    TRY(valid_ptr(ctx, x, "x"));
    if (maxit < 1 || !(rtol >= 0) || b == x) return SVK_ERR_INVALID;
    return fgmres_impl(ctx, b, x, rtol, maxit, hist, rep, (cudaStream_t)stream);
  });
}

int svk_solve_host(svk_ctx* ctx, const double* b_host, const double* x0_host, double* x_host, double rtol,
                   int32_t maxit, svk_report* rep, void* stream) {
  return guarded(ctx, [&]() -> int {
    if (!b_host || !x0_host || !x_host) return SVK_ERR_INVALID;
    if (maxit < 1 || !(rtol >= 0)) {
      ctx->err = "maxit < 1 or rtol not >= 0";
      return SVK_ERR_INVALID;
    }
    if (x_host == b_host || x_host == x0_host) {
      ctx->err = "x_host aliases an input";
      return SVK_ERR_INVALID;
    }
    cudaStream_t s = (cudaStream_t)stream;
    const LevelGeom& g = ctx->g.back();
    if (!ctx->d_hb) TRY(alloc_vec(ctx, &ctx->d_hb, g.len));
    if (!ctx->d_hx) TRY(alloc_vec(ctx, &ctx->d_hx, g.len));
    const int64_t nv = (int64_t)g.lat * g.lat;
    const size_t wu = g.lat * sizeof(double), wp = (g.N + 1) * sizeof(double);
    for (int which = 0; which < 2; ++which) {
      const double* src = which ? x0_host : b_host;
      double* dst = which ? ctx->d_hx : ctx->d_hb;
      CK(cudaMemcpy2DAsync(dst + g.oux, g.pu * sizeof(double), src, wu, wu, g.lat, cudaMemcpyHostToDevice, s));
      CK(cudaMemcpy2DAsync(dst + g.ouy, g.pu * sizeof(double), src + nv, wu, wu, g.lat, cudaMemcpyHostToDevice, s));
      CK(cudaMemcpy2DAsync(dst + g.op, g.pp * sizeof(double), src + 2 * nv, wp, wp, g.N + 1, cudaMemcpyHostToDevice, s));
    }
    int st = fgmres_impl(ctx, ctx->d_hb, ctx->d_hx, rtol, maxit, nullptr, rep, s);
    if (st < 0) return st;
    if (ctx->tr) {  // assemble the full solution on every rank
      TRY(op_zero_unowned(ctx, ctx->nlev - 1, ctx->d_hx, s));
      TRY(op_allreduce(ctx, ctx->d_hx, g.len, s));
    }
    CK(cudaMemcpy2DAsync(x_host, wu, ctx->d_hx + g.oux, g.pu * sizeof(double), wu, g.lat, cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpy2DAsync(x_host + nv, wu, ctx->d_hx + g.ouy, g.pu * sizeof(double), wu, g.lat, cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpy2DAsync(x_host + 2 * nv, wp, ctx->d_hx + g.op, g.pp * sizeof(double), wp, g.N + 1,
                         cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    return st;
  });
}

int svk_solve_host_batch(svk_ctx* ctx, int32_t count, const double* const* b_host, const double* const* x0_host,
                         double* const* x_host, double rtol, int32_t maxit, svk_report* reps, void* stream) {
  return guarded(ctx, [&]() -> int {
    if (count < 1 || !b_host || !x0_host || !x_host) return SVK_ERR_INVALID;
    if (maxit < 1 || !(rtol >= 0)) {
      ctx->err = "maxit < 1 or rtol not >= 0";
      return SVK_ERR_INVALID;
    }
    for (int k = 0; k < count; ++k) {
      if (!b_host[k] || !x0_host[k] || !x_host[k]) return SVK_ERR_INVALID;
      if (x_host[k] == b_host[k] || x_host[k] == x0_host[k]) {
        ctx->err = "x_host aliases an input";
        return SVK_ERR_INVALID;
      }
    }
    cudaStream_t s = (cudaStream_t)stream;
    const LevelGeom& g = ctx->g.back();
    if (!ctx->d_hb) TRY(alloc_vec(ctx, &ctx->d_hb, g.len));
    if (!ctx->d_hx) TRY(alloc_vec(ctx, &ctx->d_hx, g.len));
    if (!ctx->d_hb2) TRY(alloc_vec(ctx, &ctx->d_hb2, g.len));
    if (!ctx->d_hx2) TRY(alloc_vec(ctx, &ctx->d_hx2, g.len));
    const int64_t nc = 2 * (int64_t)g.lat * g.lat + (int64_t)(g.N + 1) * (g.N + 1);  // compact length
    for (int q = 0; q < 2; ++q) {
      if (!ctx->d_cin[q][0]) TRY(alloc_vec(ctx, &ctx->d_cin[q][0], nc));
      if (!ctx->d_cin[q][1]) TRY(alloc_vec(ctx, &ctx->d_cin[q][1], nc));
      if (!ctx->d_cout[q]) TRY(alloc_vec(ctx, &ctx->d_cout[q], nc));
    }
    const size_t cbytes = (size_t)nc * sizeof(double);
    const dim3 rgrid((unsigned)std::min<int64_t>((nc + 255) / 256, 8 * ctx->nsm)), rblk(256);
    if (!ctx->s_in) {
      CK(cudaStreamCreateWithFlags(&ctx->s_in, cudaStreamNonBlocking));
      CK(cudaStreamCreateWithFlags(&ctx->s_out, cudaStreamNonBlocking));
      for (cudaEvent_t* e : {ctx->ev_in, ctx->ev_solved, ctx->ev_out})
        for (int k = 0; k < 2; ++k) CK(cudaEventCreateWithFlags(&e[k], cudaEventDisableTiming));
    }
    double* hb[2] = {ctx->d_hb, ctx->d_hb2};
    double* hx[2] = {ctx->d_hx, ctx->d_hx2};
    // the copy streams start after everything already queued on `stream`
    CK(cudaEventRecord(ctx->ev_solved[1], s));
    CK(cudaStreamWaitEvent(ctx->s_in, ctx->ev_solved[1], 0));
    CK(cudaStreamWaitEvent(ctx->s_out, ctx->ev_solved[1], 0));
    auto stage_in = [&](int k) -> int {  // problem k into staging pair k % 2 (after its previous D2H)
      const int q = k & 1;
      if (k >= 2) CK(cudaStreamWaitEvent(ctx->s_in, ctx->ev_solved[q], 0));  // staging pair q is free again
      CK(cudaMemcpyAsync(ctx->d_cin[q][0], b_host[k], cbytes, cudaMemcpyHostToDevice, ctx->s_in));
      CK(cudaMemcpyAsync(ctx->d_cin[q][1], x0_host[k], cbytes, cudaMemcpyHostToDevice, ctx->s_in));
      CK(cudaEventRecord(ctx->ev_in[q], ctx->s_in));
      return SVK_OK;
    };
    TRY(stage_in(0));
    int worst = SVK_OK;
    for (int k = 0; k < count; ++k) {
      const int q = k & 1;
      if (k + 1 < count) TRY(stage_in(k + 1));  // overlaps the solve of problem k
      CK(cudaStreamWaitEvent(s, ctx->ev_in[q], 0));
      k_repitch<true><<<rgrid, rblk, 0, s>>>(g, ctx->d_cin[q][0], hb[q]);
      k_repitch<true><<<rgrid, rblk, 0, s>>>(g, ctx->d_cin[q][1], hx[q]);
      CKL();
      const int st = fgmres_impl(ctx, hb[q], hx[q], rtol, maxit, nullptr, reps ? &reps[k] : nullptr, s);
      if (st < 0) {
        cudaStreamSynchronize(ctx->s_in);
        cudaStreamSynchronize(ctx->s_out);
        return st;
      }
      if (st > worst) worst = st;
      if (ctx->tr) {  // assemble the full solution on every rank
        TRY(op_zero_unowned(ctx, ctx->nlev - 1, hx[q], s));
        TRY(op_allreduce(ctx, hx[q], g.len, s));
      }
      if (k >= 2) CK(cudaStreamWaitEvent(s, ctx->ev_out[q], 0));  // D2H of problem k-2 has left d_cout[q]
      k_repitch<false><<<rgrid, rblk, 0, s>>>(g, hx[q], ctx->d_cout[q]);
      CKL();
      ctx->launches += 3;
      CK(cudaEventRecord(ctx->ev_solved[q], s));
      CK(cudaStreamWaitEvent(ctx->s_out, ctx->ev_solved[q], 0));
      CK(cudaMemcpyAsync(x_host[k], ctx->d_cout[q], cbytes, cudaMemcpyDeviceToHost, ctx->s_out));  // overlaps solve k+1
      CK(cudaEventRecord(ctx->ev_out[q], ctx->s_out));
    }
    CK(cudaStreamSynchronize(ctx->s_out));
    CK(cudaStreamSynchronize(ctx->s_in));
    return worst;
  });
}

int svk_patch_inverse(svk_ctx* ctx, int32_t level, int32_t cat_x, int32_t cat_y, double* out, int32_t* n) {
  return guarded(ctx, [&]() -> int {
    TRY(valid_level(ctx, level));
    if (cat_x < 0 || cat_x > 4 || cat_y < 0 || cat_y > 4 || !out || !n) return SVK_ERR_INVALID;
    const LevelGeom& g = ctx->g[level];
    std::vector<double> pad(kGroupStride);
    CK(cudaMemcpy(pad.data(), ctx->d_inv + ((size_t)level * 25 + cat_y * 5 + cat_x) * kGroupStride,
                  kGroupStride * sizeof(double), cudaMemcpyDeviceToHost));
    const int kx = cat_rep(cat_x, g.N), ky = cat_rep(cat_y, g.N);
    std::vector<int> slots;
    for (int comp = 0; comp < 2; ++comp)
      for (int oy = 0; oy < 5; ++oy)
        for (int ox = 0; ox < 5; ++ox) {
          const int i = 2 * kx - 2 + ox, j = 2 * ky - 2 + oy;
          if (i < 1 || j < 1 || i > g.lat - 2 || j > g.lat - 2) continue;
          slots.push_back(comp * 25 + oy * 5 + ox);
        }
    slots.push_back(50);
    const int m = (int)slots.size();
    for (int r = 0; r < m; ++r)
      for (int c = 0; c < m; ++c) out[r * m + c] = pad[slots[r] * kSlots + slots[c]];
    *n = m;
    return SVK_OK;
  });
}

int svk_validate_patches(svk_ctx* ctx, int32_t level, double* max_rel_dev, int64_t* n_patches) {
  return guarded(ctx, [&]() -> int {
    TRY(valid_level(ctx, level));
    double dev = 0.0;
    int64_t n = 0;
    TRY(op_validate(ctx, level, &dev, &n));
    if (max_rel_dev) *max_rel_dev = dev;
    if (n_patches) *n_patches = n;
    if (!(dev <= kValidateTol)) {
      char buf[160];
      std::snprintf(buf, sizeof buf, "validation: patch inverses deviate from their group by %.3e (> %.0e) on level %d",
                    dev, kValidateTol, level);
      ctx->err = buf;
      return SVK_ERR_VALIDATION;
    }
    return SVK_OK;
  });
}

int svk_device_bytes(const svk_ctx* ctx, int64_t* bytes) {
  if (!ctx || !bytes) return SVK_ERR_INVALID;
  *bytes = ctx->dev_bytes;
  return SVK_OK;
}

int64_t svk_launch_count(const svk_ctx* ctx) { return ctx ? ctx->launches : -1; }

int svk_set_profiling(svk_ctx* ctx, int32_t enable) {
  if (!ctx) return SVK_ERR_INVALID;
  ctx->prof = enable != 0;
  return SVK_OK;
}

int svk_sweep_stats(svk_ctx* ctx, int64_t* count, double* total_ms) {
  return guarded(ctx, [&]() -> int {
    if (!ctx || !count || !total_ms) return SVK_ERR_INVALID;
    CK(cudaDeviceSynchronize());
    double t = 0.0;
    for (size_t k = 0; k + 1 < ctx->prof_used; k += 2) {
      float ms = 0.f;
      CK(cudaEventElapsedTime(&ms, ctx->prof_ev[k], ctx->prof_ev[k + 1]));
      t += ms;
    }
    TRY(harvest_graph_prof(ctx));
    *count = (int64_t)(ctx->prof_used / 2) + ctx->prof_acc_n;
    *total_ms = t + ctx->prof_acc_ms;
    ctx->prof_used = 0;
    ctx->prof_acc_n = 0;
    ctx->prof_acc_ms = 0.0;
    return SVK_OK;
  });
}

int svk_partition(int32_t n_elem, int32_t n_coarse, int32_t nranks, int32_t rank, int32_t agglom_rows, int32_t N,
                  int32_t* r0, int32_t* r1, int32_t* distributed) {
  if (!r0 || !r1 || !distributed || n_coarse < 4 || n_elem < n_coarse || nranks < 1 || rank < 0 || rank >= nranks ||
      agglom_rows < kHalo)
    return SVK_ERR_INVALID;
  std::vector<int> Ns;
  for (int64_t m = n_coarse; m <= n_elem; m *= 2) Ns.push_back((int)m);
  if (Ns.back() != n_elem) return SVK_ERR_INVALID;
  int l = -1;
  for (int k = 0; k < (int)Ns.size(); ++k)
    if (Ns[k] == N) l = k;
  if (l < 0) return SVK_ERR_INVALID;
  const int la = nranks > 1 ? first_dist_level(Ns, nranks, agglom_rows) : (int)Ns.size();
  if (l >= la) {
    slab_rows(N, Ns[la], nranks, rank, r0, r1);
    *distributed = 1;
  } else {
    *r0 = 0;
    *r1 = N + 1;
    *distributed = 0;
  }
  return SVK_OK;
}

int svk_nccl_unique_id(uint8_t* out) {
  if (!out) return SVK_ERR_INVALID;
  NcclApi& a = nccl_api();
  if (!a.ok()) return SVK_ERR_NCCL;
  NcclId id;
  if (a.GetUniqueId(&id) != 0) return SVK_ERR_NCCL;
  std::memcpy(out, id.internal, 128);
  return SVK_OK;
}

int svk_allgather(svk_ctx* ctx, double* v, void* stream) {
  return guarded(ctx, [&]() -> int {
    if (!ctx) return SVK_ERR_INVALID;
    TRY(valid_ptr(ctx, v, "v"));
    if (!ctx->tr) return SVK_OK;
    cudaStream_t s = (cudaStream_t)stream;
    TRY(op_zero_unowned(ctx, ctx->nlev - 1, v, s));
    return op_allreduce(ctx, v, ctx->g.back().len, s);
  });
}

const char* svk_status_string(int status) {
  switch (status) {
    case SVK_OK: return "ok";
    case SVK_NOT_CONVERGED: return "not converged";
    case SVK_ERR_INVALID: return "invalid argument";
    case SVK_ERR_CUDA: return "CUDA error";
    case SVK_ERR_NCCL: return "NCCL error";
    case SVK_ERR_SINGULAR: return "singular factorisation";
    case SVK_ERR_NONFINITE: return "non-finite value";
    case SVK_ERR_ALLOC: return "allocation failed";
    case SVK_ERR_VALIDATION: return "patch validation failed";
    default: return "unknown status";
  }
}

const char* svk_last_error(const svk_ctx* ctx) { return ctx ? ctx->err.c_str() : "null context"; }

}  // extern "C"
