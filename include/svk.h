/*
 * svk.h -- C ABI of libsvk: B200-native (sm_100a, fp64) additive-Vanka
 * monolithic multigrid for Q2-Q1 Taylor-Hood Stokes, after Spies, Olson,
 * MacLachlan, "Exploiting mesh structure to improve multigrid performance for
 * saddle point problems" (arXiv 2401.06277).
 *
 * Citations: P:n = line n of the paper's text, with its label.
 *
 * Problem: -nu Lap u + grad p = f, div u = 0 on [0,1]^2, Q2-Q1
 * Taylor-Hood on a uniform N x N grid, A = [[L, B^T],[B, 0]]
 * (eq:stokesmatrix), velocity Dirichlet on every edge.  The library solves the
 * interior system: Dirichlet entries of a vector hold boundary data and are
 * never changed by a correction; every residual is 0 on Dirichlet rows.
 *
 * ---------------------------------------------------------------------------
 * VECTORS.  Every vector argument is a caller-owned DEVICE buffer of double
 * (16-byte aligned -- the kernels use 16-byte vector and TMA accesses, and a
 * less aligned pointer is rejected with SVK_ERR_INVALID; 256-byte aligned
 * recommended) holding one level's vector
 * in the PITCHED layout reported by svk_level_info():
 *   u_x plane at off_ux: (2N+1) rows (y) of pitch_u doubles, column i = x index
 *   u_y plane at off_uy: same shape
 *   p   plane at off_p : (N+1) rows of pitch_p doubles
 * Lattice point (i,j), 0<=i,j<=2N, is at (i h/2, j h/2), h = 1/N; pressure
 * node (kx,ky) at (kx h, ky h).  Padding columns (i > 2N, kx > N) and the gaps
 * between planes must be 0 on input; the library keeps them 0 in outputs.
 * Length vec_len doubles.  Levels: 0 = coarsest (N0), L-1 = finest (P:146,
 * alg:mg "level 0 is the coarsest grid").
 *
 * OWNERSHIP.  The library never frees or retains caller pointers beyond the
 * stream-ordered completion of the call.  It owns its workspaces (patch
 * inverses, per-level temporaries, Krylov basis), allocated with cudaMalloc
 * on cfg.device in svk_create / on first use, and freed in svk_destroy.
 *
 * STREAMS.  `stream` is a cudaStream_t (NULL = legacy default stream).  Every
 * call is asynchronous on `stream` except svk_create, svk_destroy,
 * svk_fgmres / svk_solve_host (synchronise once per Krylov iteration for the
 * Givens update and return on completion) and the introspection calls.
 *
 * ERRORS.  int status: SVK_OK = 0; negative = error (message via
 * svk_last_error); SVK_NOT_CONVERGED = 1 is non-fatal (the report is filled).
 * SVK_ERR_INVALID: bad level / size / NULL or misaligned pointer;
 * SVK_ERR_CUDA: a CUDA runtime error (the context may be unusable afterwards);
 * SVK_ERR_SINGULAR: a patch or coarse factorisation met a zero pivot;
 * SVK_ERR_NONFINITE: FGMRES met NaN/Inf;
 * SVK_ERR_VALIDATION: validation mode found a patch that differs from its group.
 *
 * THREADING.  One context per device; calls on one context must not overlap
 * (scratch is per context).  Different contexts are independent: every call
 * taking a context runs on cfg.device (the caller's current device is
 * restored on return), and C++ exceptions never cross this boundary (they map
 * to SVK_ERR_ALLOC / SVK_ERR_INVALID with a message).
 *
 * MULTI-GPU (nranks > 1).  Every rank creates one context with the same
 * configuration except `rank`.  The finest levels are split into row slabs;
 * every call then computes only the rank's owned rows, and the library refreshes
 * halo rows (4 node rows per side) of its input vectors itself, so rows outside
 * a rank's slab are library-managed scratch.  svk_fgmres / svk_vcycle /
 * svk_vanka_sweep / svk_residual / svk_matvec must be called by all ranks
 * together (they communicate).  svk_allgather assembles a full vector.
 * svk_restrict / svk_prolong_add do not exchange halos: on a distributed level
 * they compute the rank's owned rows from the rows it already holds, so the
 * caller must pass inputs whose halo rows are current (as svk_vcycle does).
 *
 * ENVIRONMENT (tuning and test aids; read once per process unless noted):
 *   SVK_PDL=0          launch kernels without programmatic dependent launch;
 *   SVK_CHUNK_ROWS=n   node rows per CTA the strip kernels' wave sizing aims at
 *                      (default 64);
 *   SVK_POISON_HALO=1  NaN-fill rows beyond the halo after each exchange (tests);
 *   SVK_SMALL_N=n      levels with N <= n below the finest run as one cluster launch
 *                      (default 16; 0: every level as separate kernels) -- read at
 *                      svk_create (results agree to rounding: same operators);
 *   SVK_SMALL_CLUSTER=c  CTAs of that cluster (default 16, halved until the device
 *                      can co-schedule it; an explicit c is used as given, and a
 *                      launch the device rejects falls back to separate kernels);
 *   SVK_GRAPHS=0       replay no CUDA graphs (direct launches) inside svk_fgmres.
 * Compile time: -DSVK_STRIP_THREADS=64|128 (threads per strip CTA, default 64).
 */
#ifndef SVK_H_
#define SVK_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SVK_VERSION 1

enum svk_status {
  SVK_OK = 0,
  SVK_NOT_CONVERGED = 1,
  SVK_ERR_INVALID = -1,
  SVK_ERR_CUDA = -2,
  SVK_ERR_NCCL = -3,
  SVK_ERR_SINGULAR = -4,
  SVK_ERR_NONFINITE = -5,
  SVK_ERR_ALLOC = -6,
  SVK_ERR_VALIDATION = -7
};

/* W_i of alg:vk ("the matrix with the weights"; unstated in the paper):
 * MULT: omega_v / (number of patches holding the DOF) -- default (reading 6);
 * SCALAR: omega_v * I. */
enum svk_weighting { SVK_WEIGHT_MULT = 0, SVK_WEIGHT_SCALAR = 1 };

/* level-0 solve ("an exact solve ... or three sweeps of the relaxation"):
 * EXACT = minimum-norm solve (pressure mean 0; reading 3), SWEEPS3. */
enum svk_coarse { SVK_COARSE_EXACT = 0, SVK_COARSE_SWEEPS3 = 1 };

/* problem kinds for svk_set_problem:
 * ZERO: b = 0, x0 = 0;
 * MMS_PAPER: the paper's manufactured solution, f = -nu Lap u + grad p;
 * MMS_INSPACE: u = (2x^2y, -2xy^2), p = xy - 1/4 (lies in the Q2-Q1 space);
 * CAVITY: f = 0, u = (1,0) on lattice points of the lid y=1 with 0<x<1
 *         (not in the paper; reading 15). */
enum svk_problem { SVK_PROBLEM_ZERO = 0, SVK_PROBLEM_MMS_PAPER = 1, SVK_PROBLEM_MMS_INSPACE = 2, SVK_PROBLEM_CAVITY = 3 };

/* sweep kernel selection (all compute alg:vk exactly; they differ in data flow):
 * FUSED  (default) -- residual + patch solve + owner-computes gather in one kernel;
 * UNFUSED -- residual, per-patch solve into a packed buffer, gather update
 *            (the paper's form/apply/update kernel split), kept as a
 *            cross-check of the fused kernel. */
enum svk_sweep_impl { SVK_SWEEP_FUSED = 0, SVK_SWEEP_UNFUSED = 1, SVK_SWEEP_SIMPLE = 2 };
/* SIMPLE -- the paper's "simple Vanka" baseline: every patch's
 *           inverse is built and stored at svk_create (51 x 51 doubles per patch
 *           and level, about 28 KB per fine-grid node over the hierarchy: N <= 2048
 *           on one B200; larger N returns SVK_ERR_CUDA from svk_create), applied by
 *           the unfused kernel split.  Comparator only; same arithmetic as alg:vk. */

typedef struct svk_config {
  int32_t n_elem;     /* N, elements per side of the finest grid; N = n_coarse * 2^k */
  int32_t n_coarse;   /* N0 >= 4 (all 25 patch categories exist; reading 4); default 4 */
  double nu;          /* viscosity; default 1 */
  double omega_v;     /* Vanka damping (reading 6); default 0.8 */
  int32_t weighting;  /* enum svk_weighting; default MULT */
  int32_t nu_pre;     /* pre-smoothing sweeps (V(1,1)); default 1 */
  int32_t nu_post;    /* post-smoothing sweeps; default 1 */
  int32_t coarse;     /* enum svk_coarse; default EXACT */
  int32_t sweep_impl; /* enum svk_sweep_impl; default FUSED */
  int32_t device;     /* CUDA device ordinal; default 0 */
  /* multi-GPU row slabs (the paper is single-GPU): */
  int32_t rank;        /* this process's rank; default 0 */
  int32_t nranks;      /* number of ranks; default 1 (no communication) */
  int32_t transport;   /* enum svk_transport; default NONE */
  int32_t agglom_rows; /* levels with fewer than agglom_rows node rows per rank are
                          replicated on every rank (coarse agglomeration); default 64, >= 4 */
  int32_t emul_group;  /* EMULATED transport: id of the in-process group to join */
  int32_t orth;        /* enum svk_orth: FGMRES Gram-Schmidt; default ADAPTIVE */
  int32_t relax;         /* enum svk_relax: relaxation inside the V-cycle; default VANKA */
  int32_t jacobi_sweeps; /* BS / SU: weighted-Jacobi sweeps on S; default 3 */
  uint8_t nccl_id[128]; /* NCCL transport: ncclUniqueId from svk_nccl_unique_id() on rank 0,
                           broadcast to every rank by the caller */
  double relax_t;        /* BS / SU: t in tD ~ L; default 1 */
  double relax_omega;    /* BS: omega_BS of alg:bs line 3-4 (unused by SU); default 1 */
  double jacobi_omega;   /* BS / SU: weight of the Jacobi iteration on S; default 0.8
                            (SU: 0.4, "optimal Jacobi weight") */
  int32_t precond;       /* enum svk_precond: FGMRES preconditioner; default MG */
  int32_t bt_cycles;     /* BLOCK_TRIANGULAR: V-cycles per block; default 3 */
  int32_t bt_nu;         /* BLOCK_TRIANGULAR: Jacobi sweeps before / after; default 3 (V(3,3)) */
  int32_t validate;      /* validation mode ("only 25 different patch matrices"):
                            svk_create rebuilds every patch of every level on its own and
                            checks it against its group (svk_validate_patches); default 0 */
  double bt_omega_u;     /* BLOCK_TRIANGULAR: Jacobi weight on L; default 1.0 */
  double bt_omega_p;     /* BLOCK_TRIANGULAR: Jacobi weight on M; default 0.6 */
  int32_t krylov_store_z; /* 1 (default): FGMRES keeps Z_j = M V_j;
                             0: low-memory mode for the MG preconditioner, whose V-cycle
                             from zero is a FIXED linear operator M -- only V_j is kept,
                             each z_j lives in one buffer until A z_j is formed, and the
                             update is x = x0 + M (sum_j y_j V_j) with one extra V-cycle:
                             the same iterates as FGMRES up to rounding (right-
                             preconditioned GMRES), half the Krylov memory (8192^2 fits
                             one B200).  Not with BLOCK_TRIANGULAR (kept as FGMRES). */
  int32_t reserved0;
  /* Optional device allocator for the context's vector-sized workspaces (level
   * work vectors, the Krylov basis, boundary-patch staging, host-solve staging),
   * e.g. to route them through a framework's caching allocator (the Python
   * binding's Solver(allocator="torch") passes torch.cuda.caching_allocator_*).
   * Both or neither must be set (else svk_create returns SVK_ERR_INVALID).
   * alloc_fn(bytes, device, user) returns device memory on cfg.device aligned to
   * 256 bytes, or NULL (the calling entry point then returns SVK_ERR_CUDA); the
   * library zero-fills it after a device synchronisation, so the memory may have
   * been in use on any stream before.  free_fn(ptr, bytes, device, user) is called
   * once per block, from svk_destroy after a device synchronisation (no kernel of
   * the context uses the block any more).  Calls happen inside svk_create and, for
   * lazily sized workspaces, inside the first svk_fgmres / svk_solve_host /
   * svk_vcycle of a size -- from the thread making that call.  Small tables
   * (patch factors, coefficients, the coarse LU) and the slab-local vectors of
   * distributed levels (mapped with the CUDA VMM API) always use the driver.
   * NULL (default): cudaMalloc / cudaFree. */
  void* (*alloc_fn)(int64_t bytes, int32_t device, void* user);
  void (*free_fn)(void* ptr, int64_t bytes, int32_t device, void* user);
  void* alloc_user;
} svk_config;

/* FGMRES preconditioner:
 * MG               -- one monolithic V(nu_pre, nu_post) cycle with svk_config.relax (alg:mg);
 * BLOCK_TRIANGULAR -- alg:bt: [[L, B^T],[0, -M]] (du, dp) = r with M the Q1
 *                     pressure mass matrix; M dp = -r_p, then L du = r_u - B^T dp, each by
 *                     bt_cycles V(bt_nu, bt_nu) multigrid cycles with weighted Jacobi.
 *                     Single-GPU comparator. */
enum svk_precond { SVK_PRECOND_MG = 0, SVK_PRECOND_BLOCK_TRIANGULAR = 1 };

/* Relaxation of the V-cycle (alg:mg "Relax on u_l and p_l"):
 * VANKA           -- additive Vanka (alg:vk), the hot path;
 * BRAESS_SARAZIN  -- inexact Braess-Sarazin (alg:bs): S dp ~= r_p - (1/t) B D^-1 r_u
 *                    by jacobi_sweeps weighted-Jacobi sweeps on S = -(1/t) B D^-1 B^T,
 *                    du = (1/t) D^-1 (r_u - B^T dp), x += relax_omega (du, dp);
 * SCHUR_UZAWA     -- Schur-Uzawa (alg:uz): du = (1/t) D^-1 r_u,
 *                    S dp ~= r_p - B du (eq:uzblock; reading 19), x += (du, dp).
 * D = diag(L) on non-Dirichlet velocity DOFs.  The comparators are single-GPU
 * (nranks == 1) and exist as the paper's same-run baselines. */
enum svk_relax { SVK_RELAX_VANKA = 0, SVK_RELAX_BRAESS_SARAZIN = 1, SVK_RELAX_SCHUR_UZAWA = 2 };

/* transports for nranks > 1:
 * NCCL     -- one process per GPU; halos by ncclSend/ncclRecv with the two slab
 *             neighbours, dot products by ncclAllReduce (libnccl.so.2 is loaded
 *             with dlopen on first use);
 * EMULATED -- nranks logical ranks inside ONE process on one device, one host
 *             thread per rank (test mode; same partition, halos and reductions). */
enum svk_transport { SVK_TRANSPORT_NONE = 0, SVK_TRANSPORT_NCCL = 1, SVK_TRANSPORT_EMULATED = 2 };

/* Arnoldi orthogonalisation of svk_fgmres (the paper does not fix it):
 * CGS2     -- classical Gram-Schmidt, always two passes ("twice is enough");
 * ADAPTIVE -- one classical pass; a second pass only when the pass cancelled
 *             more than a factor kappa = 10 of the vector's norm
 *             (||w'|| < ||w|| / kappa, a DGKS-type test; reading 18). */
enum svk_orth { SVK_ORTH_ADAPTIVE = 0, SVK_ORTH_CGS2 = 1 };

typedef struct svk_level {
  int32_t N;          /* elements per side on this level */
  int32_t lat;        /* 2N+1 velocity lattice points per side */
  int64_t vec_len;    /* doubles per vector */
  int64_t off_ux, off_uy, off_p;  /* plane offsets (doubles) */
  int64_t pitch_u, pitch_p;       /* row pitches (doubles), multiples of 8 */
  int64_t n_dof;      /* 2(2N+1)^2 + (N+1)^2 (Dirichlet DOFs included) */
  int64_t n_patch;    /* (N+1)^2 Vanka patches, one per pressure node */
  int32_t row0, row1; /* owned node rows [row0, row1) of this rank (lattice rows
                         [2 row0, min(2 row1, lat))); 0, N+1 on a single rank */
  int32_t distributed; /* 1 if this level is split into row slabs */
  int32_t halo_rows;   /* node rows of halo refreshed per side (0 if not distributed) */
} svk_level;

typedef struct svk_report {
  int32_t iterations;      /* FGMRES iterations (= preconditioner applications) */
  int32_t converged;       /* 1 if estimate <= rtol */
  int32_t status;          /* same as the return value */
  int32_t n_reorth;        /* iterations that needed a second Gram-Schmidt pass */
  double rel_residual;     /* true ||b - A x|| / ||b - A x0||, recomputed at exit */
  double t_total_s;        /* wall time of the call (host clock) */
  double t_vcycle_s;       /* device time in V-cycles (CUDA events) */
  double t_orth_s;         /* device time in matvec + orthogonalisation */
  double t_setup_s;        /* wall time (host clock) svk_create spent building this
                              context: hierarchy, patch factors, coarse LU, validation */
} svk_report;

typedef struct svk_ctx svk_ctx;

/* Fill *cfg with the defaults above for a grid of n_elem elements per side. */
int svk_config_default(svk_config* cfg, int32_t n_elem);

/* Grid create + hierarchy build and batched patch setup
 * (a2): builds levels N, N/2, ..., N0, uploads the stencil tables, runs the
 * patch-setup kernel that assembles and inverts the 25 distinct patch matrices
 * of every level in fp64 ("inverting each patch matrix ahead of time", P:260;
 * "25 different patch matrices"), and the minimum-norm level-0
 * pseudo-inverse.  Synchronous.  On error *out = NULL. */
int svk_create(const svk_config* cfg, svk_ctx** out);
int svk_destroy(svk_ctx* ctx);

int svk_num_levels(const svk_ctx* ctx, int32_t* levels);
int svk_level_info(const svk_ctx* ctx, int32_t level, svk_level* out);

/* Problem data on `level`: b (velocity: (f, psi_i) by 3x3 Gauss per element;
 * Dirichlet rows: the boundary value; pressure: 0) and x0 (boundary values,
 * zero elsewhere).  Either pointer may be NULL. */
int svk_set_problem(svk_ctx* ctx, int32_t level, int32_t kind, double* b, double* x0, void* stream);

/* r = b - A x on non-Dirichlet rows, 0 on Dirichlet rows (alg:mg line 3, P:151;
 * kernels "Q2 matrix * Q2 vector", "Q2Q1 matrix * Q2/Q1 vector").
 * r must not alias x or b. */
int svk_residual(svk_ctx* ctx, int32_t level, const double* x, const double* b, double* r, void* stream);

/* y = A x on non-Dirichlet rows, 0 on Dirichlet rows (the interior operator
 * FGMRES iterates with).  y must not alias x. */
int svk_matvec(svk_ctx* ctx, int32_t level, const double* x, double* y, void* stream);

/* nsweeps additive Vanka sweeps (alg:vk):
 *   x <- x + sum_i V_i^T W_i A_i^{-1} V_i (b - A x)
 * with one patch per pressure node and exact patch solves.  Out of place:
 * reads x_in, writes x_out (x_out must not alias x_in or b); for nsweeps > 1
 * the library ping-pongs through its own workspace and the final iterate is
 * in x_out. */
int svk_vanka_sweep(svk_ctx* ctx, int32_t level, const double* x_in, const double* b, double* x_out,
                    int32_t nsweeps, void* stream);

/* r_coarse = P^T r_fine on level-1 with coarse Dirichlet rows set to 0
 * (alg:mg line 4; P = finite-element interpolation).
 * `level` is the FINE level (>= 1). */
int svk_restrict(svk_ctx* ctx, int32_t level, const double* r_fine, double* r_coarse, void* stream);

/* Residual and restriction in one pass (alg:mg lines 3-4; the
 * V-cycle's own kernel, k_residual_strip<MODE 1>): r_coarse = P^T (b - A x) on
 * level-1, Dirichlet rows 0 (reading 9); the fine residual never reaches
 * memory.  x, b: level `level` vectors; r_coarse: level `level`-1 vector, must
 * not alias them.  Asynchronous on `stream`.  Multi-GPU: halos of x and b are
 * refreshed; on the agglomeration level the coarse vector is assembled on every
 * rank (all-gather), on a distributed coarse level only the rank's rows are
 * written.  SVK_ERR_INVALID on level < 1, bad pointers or aliasing. */
int svk_residual_restrict(svk_ctx* ctx, int32_t level, const double* x, const double* b, double* r_coarse,
                          void* stream);

/* x_fine += P e_coarse (alg:mg line 9).  `level` is the FINE level. */
int svk_prolong_add(svk_ctx* ctx, int32_t level, const double* e_coarse, double* x_fine, void* stream);

/* x = A_0^+ b on level 0 (minimum-norm, reading 3); Dirichlet
 * entries of x set to 0. */
int svk_coarse_solve(svk_ctx* ctx, const double* b, double* x, void* stream);

/* One sweep of the CONFIGURED relaxation (svk_config.relax) on `level`:
 * x_out = x_in + correction.  VANKA: identical to svk_vanka_sweep(..., 1, ...);
 * BRAESS_SARAZIN / SCHUR_UZAWA: alg:bs / alg:uz (see enum svk_relax).
 * Layout, ownership and stream semantics as svk_vanka_sweep; x_out must not alias
 * x_in or b.  SVK_ERR_INVALID on a bad level / pointer / aliasing. */
int svk_relax_sweep(svk_ctx* ctx, int32_t level, const double* x_in, const double* b, double* x_out, void* stream);

/* z = M b on the finest level with the CONFIGURED FGMRES preconditioner
 * (svk_config.precond): MG = one V-cycle from zero (as svk_vcycle with x = 0);
 * BLOCK_TRIANGULAR = alg:bt.  b: residual-type vector (Dirichlet entries 0);
 * z: output, fully overwritten, must not alias b.  Asynchronous on `stream`. */
int svk_precond_apply(svk_ctx* ctx, const double* b, double* z, void* stream);

/* One V(nu_pre, nu_post) cycle (alg:mg) on the finest level; x is
 * in/out (a preconditioner application passes x = 0).  b and x must not alias. */
int svk_vcycle(svk_ctx* ctx, const double* b, double* x, void* stream);

/* Flexible GMRES, right-preconditioned by one V-cycle per iteration (P:127,
 * P:649), no restart, stop when the Givens residual estimate <= rtol * ||r0||.
 * x: in = x0 (boundary data in its Dirichlet entries), out = solution.
 * hist (optional, host, maxit+1 doubles): relative residual estimate per
 * iteration.  rep (optional, host) receives the report.  Returns SVK_OK,
 * SVK_NOT_CONVERGED or an error. */
int svk_fgmres(svk_ctx* ctx, const double* b, double* x, double rtol, int32_t maxit, double* hist,
               svk_report* rep, void* stream);

/* End-to-end solve through HOST buffers (pinned or pageable), each in the
 * COMPACT layout [u_x (2N+1)^2, u_y (2N+1)^2, p (N+1)^2] of the finest level:
 * copies b and x0 to the device, runs svk_fgmres, copies x back. */
int svk_solve_host(svk_ctx* ctx, const double* b_host, const double* x0_host, double* x_host, double rtol,
                   int32_t maxit, svk_report* rep, void* stream);

/* Pipelined end-to-end solves of `count` independent problems from HOST buffers
 * (b_host[k], x0_host[k] in, x_host[k] out; compact layout as svk_solve_host;
 * pinned buffers let the copies run asynchronously): problem k is solved on
 * `stream` (svk_fgmres) while the host->device copies of problem
 * k+1 and the device->host copy of problem k-1 run on two library-owned copy
 * streams (two device staging pairs, allocated on first use).  Every problem's
 * copies are made; only their overlap with the solves differs from calling
 * svk_solve_host `count` times, and the results are bitwise the same.  reps
 * (optional, host) receives `count` reports.  Returns the largest per-problem
 * status (SVK_OK or SVK_NOT_CONVERGED) or the first error (remaining problems
 * are not solved).  Multi-GPU: as svk_solve_host, all ranks call together. */
int svk_solve_host_batch(svk_ctx* ctx, int32_t count, const double* const* b_host, const double* const* x0_host,
                         double* const* x_host, double rtol, int32_t maxit, svk_report* reps, void* stream);

/* Introspection for tests: the dense inverse of patch group (cat_x, cat_y),
 * cat in {0: k=0, 1: k=1, 2: 2<=k<=N-2, 3: k=N-1, 4: k=N}, on `level`,
 * copied to host `out` (n*n doubles, row-major, n <= 51); *n receives the
 * number of patch unknowns.  Patch-local order: u_x window points (y outer,
 * x inner; Dirichlet points skipped), then u_y, then p. */
int svk_patch_inverse(svk_ctx* ctx, int32_t level, int32_t cat_x, int32_t cat_y, double* out, int32_t* n);

/* Number of kernel launches issued by this context since creation (for the
 * benchmark's gpu_launches count). */
/* Validation mode.  Every patch of `level` is
 * rebuilt from the stencil on its own (A_i = V_i A V_i^T) and inverted
 * (batched fp64 Gauss-Jordan), and compared with the stored inverse of its
 * group; the generic group's reflection-basis Schur factors (the fused sweep's
 * solve) are applied to the 51 unit vectors and compared with the generic
 * group's inverse.  *max_rel_dev (host, optional) = max |a - b| / max |group
 * inverse| over all of them, *n_patches = (N+1)^2.  Synchronous.  Returns
 * SVK_OK if max_rel_dev <= 1e-12, else SVK_ERR_VALIDATION (message names the
 * deviation); workspace ~170 MB, freed on return. */
int svk_validate_patches(svk_ctx* ctx, int32_t level, double* max_rel_dev, int64_t* n_patches);

/* Device memory held by the context (workspaces, Krylov basis, factors) in
 * bytes, host out-parameter.  With nranks > 1 the vectors of the distributed
 * levels are SLAB-LOCAL: their full pitched layout is reserved as virtual
 * address space but device memory is mapped only for the rank's slab, its halo
 * and a 2-node-row margin (SVK_SLAB_LOCAL=0 allocates them full size), so a
 * rank holds ~1/nranks of each such vector. */
int svk_device_bytes(const svk_ctx* ctx, int64_t* bytes);

int64_t svk_launch_count(const svk_ctx* ctx);

/* Benchmark support.  While profiling is enabled, every full Vanka sweep (non-
 * zero initial guess) on the finest level (the kernels of one sweep step: the
 * boundary-patch kernel and the fused sweep, or the three unfused kernels) is bracketed by
 * CUDA events recorded on the sweep's stream.  svk_sweep_stats synchronises
 * the device, returns the number of bracketed sweeps and their summed device
 * time in milliseconds since the previous call, and resets both. */
int svk_set_profiling(svk_ctx* ctx, int32_t enable);
int svk_sweep_stats(svk_ctx* ctx, int64_t* count, double* total_ms);

/* Row slab of `rank` on a level with N elements per side, for a finest grid
 * n_elem = n_coarse * 2^k split over nranks with the given agglom_rows: node rows
 * [*r0, *r1) on distributed levels (*distributed = 1), or [0, N+1) on replicated
 * ones (*distributed = 0).  Pure function, no GPU needed. */
int svk_partition(int32_t n_elem, int32_t n_coarse, int32_t nranks, int32_t rank, int32_t agglom_rows, int32_t N,
                  int32_t* r0, int32_t* r1, int32_t* distributed);

/* Fill out[128] with a fresh ncclUniqueId (call on rank 0, broadcast the bytes
 * into svk_config.nccl_id on every rank).  SVK_ERR_NCCL if NCCL cannot be loaded. */
int svk_nccl_unique_id(uint8_t* out);

/* Distributed mode: make every rank's copy of a finest-level vector complete
 * (the owned rows of all ranks, all-reduced).  No-op on a single rank. */
int svk_allgather(svk_ctx* ctx, double* v, void* stream);

const char* svk_status_string(int status);
const char* svk_last_error(const svk_ctx* ctx);

#ifdef __cplusplus
}
#endif
#endif /* SVK_H_ */
