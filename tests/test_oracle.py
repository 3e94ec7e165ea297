"""Pins for the CPU oracle (no GPU).  Each test checks the oracle against
something other than itself: the independent NumPy brute force in brute.py,
values printed in the paper (tests/golden/paper_counts.json), closed forms
(manufactured solutions), invariants, or library routines (numpy pinv/lstsq).
"""
import json
import os

import numpy as np
import pytest

import oracle
import svk_inputs
import brute

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "paper_counts.json")))


def rel(a, b):
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


@pytest.fixture(scope="module")
def o8():
    return oracle.Oracle(8)


@pytest.fixture(scope="module")
def o16():
    return oracle.Oracle(16)


# ---------------------------------------------------------------- operator
@pytest.mark.parametrize("N", [2, 4, 8])
def test_operator_matches_exact_kronecker(N):
    """Element-by-element 2D Gauss assembly == exact 1D integration + Kronecker."""
    o = oracle.Oracle(N, n_coarse=N)
    A = o.csr(0).toarray()
    B = brute.full_operator(N)
    assert np.abs(A - B).max() <= 1e-14 * np.abs(B).max()


def test_symmetry_nullspace_one_kernel_vector():
    o = oracle.Oracle(4)
    A = o.csr(0).toarray()
    assert np.abs(A - A.T).max() == 0.0 or np.abs(A - A.T).max() < 1e-15
    d = o.dirichlet(0)
    I = np.flatnonzero(~d)
    AI = A[np.ix_(I, I)]
    s = np.linalg.svd(AI, compute_uv=False)
    assert (s < 1e-10 * s[0]).sum() == 1             # exactly one null vector (reading 3)
    n = np.zeros(A.shape[0])
    n[2 * 81:] = 1.0                                    # constant pressure
    assert np.abs(AI @ n[I]).max() < 1e-14
    # saddle-point structure: zero pressure-pressure block, L block-diagonal over components
    assert np.all(A[2 * 81:, 2 * 81:] == 0)
    assert np.all(A[:81, 81:162] == 0)
    # interior rows of L annihilate constants
    L = A[:81, :81]
    dd = d[:81]
    assert np.abs(L[~dd] @ np.ones(81)).max() < 1e-13


# ---------------------------------------------------------------- patches
@pytest.mark.parametrize("N", [4, 8])
def test_patches_match_paper_definition(N):
    o = oracle.Oracle(N, n_coarse=N)
    for ky in range(N + 1):
        for kx in range(N + 1):
            assert np.array_equal(np.sort(o.patch(0, kx, ky)), np.sort(brute.patch_dofs(N, kx, ky)))


@pytest.mark.parametrize("N", [4, 8, 16, 32, 64])
def test_25_patch_groups(N):
    o = oracle.Oracle(N)
    assert all(o.num_groups(l) == GOLD["patch_groups"]["value"] for l in range(o.levels))
    # groups = per-axis categories {0, 1, 2..N-2, N-1, N} (fig:vkmatrices)
    cat = lambda k: 0 if k == 0 else 1 if k == 1 else 4 if k == N else 3 if k == N - 1 else 2
    seen = {}
    for ky in range(N + 1):
        for kx in range(N + 1):
            g = o.patch_group(o.fine, kx, ky)
            key = (cat(kx), cat(ky))
            assert seen.setdefault(key, g) == g
    assert len(set(seen.values())) == 25


@pytest.mark.parametrize("N", [4, 8, 16])
def test_tab_rwf_counts(N):
    """Patch sizes counted with Dirichlet DOFs reproduce tab:rwf."""
    o = oracle.Oracle(N, n_coarse=N)
    d = o.dirichlet(0)
    l = N - 1
    sizes = []
    for ky in range(N + 1):
        for kx in range(N + 1):
            full = brute.patch_dofs(N, kx, ky, with_dirichlet=True)
            own = o.patch(0, kx, ky)
            assert set(own) == set(full[~d[full]])
            sizes.append(len(full))
    sizes = np.array(sizes)
    poly = lambda c: c[0] + c[1] * l + c[2] * l * l
    assert sizes.sum() == poly(GOLD["form_patch_rhs"]["value"])
    assert (sizes ** 2 + sizes).sum() == poly(GOLD["apply_reads"]["value"])
    assert (2 * sizes ** 2).sum() == poly(GOLD["apply_flops"]["value"])
    assert sorted(set(sizes.tolist())) == [19, 31, 51]
    # unknowns after removing Dirichlet DOFs (reading 7)
    unk = {len(o.patch(0, kx, ky)) for ky in range(N + 1) for kx in range(N + 1)}
    assert unk == ({51, 41, 33, 21, 17, 9} if N >= 4 else unk)


def test_tab_aiperf_reproduces_with_8_byte_doubles():
    """AI column of tab:aiperf at 512^2 from the tab:rwf counts (8 B/double)."""
    N, l = 512, 511
    n, m = (2 * N + 1) ** 2, (N + 1) ** 2
    poly = lambda c: c[0] + c[1] * l + c[2] * l * l
    form = poly(GOLD["form_patch_rhs"]["value"])
    ai = {
        "array_pm": (2 * n + m) / (8 * (2 * (2 * n + m) + 2 * n + m)),
        "array_scalar": (2 * n + m) / (8 * (2 * (2 * n + m))),
        "q2_matvec": (n * n) / (8 * (n * n + n + n)),
        "vanka_form": 0.0,
        "vanka_apply": poly(GOLD["apply_flops"]["value"]) / (8 * (poly(GOLD["apply_reads"]["value"]) + form)),
        "vanka_update": form / (8 * (2 * form)),
    }
    for k, v in GOLD["aiperf_512"]["value"].items():
        decimals = len(repr(v).split(".")[1])           # half a unit in the last printed digit
        assert abs(ai[k] - v) <= 0.5 * 10.0 ** -decimals, (k, ai[k], v)


@pytest.mark.parametrize("N", [4, 8])
def test_weights_multiplicity(N):
    o = oracle.Oracle(N, n_coarse=N, omega=0.8)
    w = o.weights(0)
    d = o.dirichlet(0)
    nl = 2 * N + 1
    for comp in range(2):
        for j in range(1, nl - 1):
            for i in range(1, nl - 1):
                mult = {(0, 0): 9, (1, 0): 6, (0, 1): 6, (1, 1): 4}[(i % 2, j % 2)]
                assert w[comp * nl * nl + j * nl + i] == pytest.approx(0.8 / mult, rel=1e-15)
    assert np.all(w[2 * nl * nl:] == 0.8)
    assert np.all(w[d] == 0)
    # partition of unity: sum_i V_i^T (W_i/omega) V_i = I on non-Dirichlet DOFs
    acc = np.zeros_like(w)
    for ky in range(N + 1):
        for kx in range(N + 1):
            p = o.patch(0, kx, ky)
            acc[p] += w[p] / 0.8
    assert np.allclose(acc[~d], 1.0, rtol=0, atol=1e-15)


# ---------------------------------------------------------------- sweep / residual
@pytest.mark.parametrize("N", [4, 8])
def test_residual_and_sweep_vs_dense_bruteforce(N):
    o = oracle.Oracle(N, n_coarse=N)
    D = brute.Dense(N)
    for seed in (1, 2, 3):
        x = svk_inputs.random_vector(N, seed)
        b = svk_inputs.random_vector(N, seed + 100)
        assert rel(o.residual(0, x, b), D.residual(x, b)) < 1e-13
        xo = o.sweep(0, x, b)
        xd = D.sweep(x, b)
        assert rel(xo - x, xd - x) < 1e-12


def test_sweep_linear_and_zero(o8):
    l = o8.fine
    z = np.zeros(o8.length(l))
    assert np.all(o8.sweep(l, z, z) == 0)
    x = svk_inputs.random_vector(8, 5)
    b = svk_inputs.random_vector(8, 6)
    a = 2.5
    assert rel(o8.sweep(l, a * x, a * b), a * o8.sweep(l, x, b)) < 1e-14
    # Dirichlet entries are never changed
    d = o8.dirichlet(l)
    assert np.array_equal(o8.sweep(l, x, b)[d], x[d])


def test_schur_form_equals_lu(o16):
    """Per patch, the Schur-complement solve (L_w^{-1}, rank-1 pressure) agrees with the
    oracle's LU solve -- an independent algorithm (SURVEY 8(c) patch-solve pin)."""
    A = o16.csr(o16.fine).toarray()
    N = 16
    rng = np.random.default_rng(0)
    for (kx, ky) in [(0, 0), (1, 1), (5, 7), (16, 3), (15, 15)]:
        p = o16.patch(o16.fine, kx, ky)
        Ai = A[np.ix_(p, p)]
        r = rng.standard_normal(len(p))
        nvel = len(p) - 1
        Lw = Ai[:nvel, :nvel]
        bb = Ai[nvel, :nvel]
        c = np.linalg.solve(Lw, bb)
        u0 = np.linalg.solve(Lw, r[:nvel])
        dp = (bb @ u0 - r[nvel]) / (bb @ c)
        sol = np.concatenate([u0 - c * dp, [dp]])
        assert rel(Ai @ sol, r) < 1e-12


# ---------------------------------------------------------------- transfers
def test_prolongation_matches_bruteforce():
    o = oracle.Oracle(16, n_coarse=4)
    for l in (1, 2):
        P = o.prolongation(l).toarray()
        Pb = brute.prolongation(o.N(l - 1))
        assert np.abs(P - Pb).max() == 0.0


def test_galerkin_identity():
    o = oracle.Oracle(16, n_coarse=4)
    for l in (1, 2):
        P = o.prolongation(l).toarray()
        Af, Ac = o.csr(l).toarray(), o.csr(l - 1).toarray()
        If = np.flatnonzero(~o.dirichlet(l))
        Ic = np.flatnonzero(~o.dirichlet(l - 1))
        G = P[np.ix_(If, Ic)].T @ Af[np.ix_(If, If)] @ P[np.ix_(If, Ic)]
        assert np.abs(G - Ac[np.ix_(Ic, Ic)]).max() < 1e-14 * np.abs(Ac).max()


def test_prolongation_reproduces_coarse_polynomials():
    o = oracle.Oracle(8, n_coarse=4)
    Nc, Nf = 4, 8
    f = lambda x, y: 1 + 2 * x - 3 * y + x * x - x * y + 0.5 * y * y + x * x * y * y
    g = lambda x, y: 0.3 + x - 2 * y + 4 * x * y
    def sample(N):
        nl = 2 * N + 1
        xs = np.arange(nl) / (2 * N)
        U = f(xs[None, :], xs[:, None]).ravel()
        ps = np.arange(N + 1) / N
        Pp = g(ps[None, :], ps[:, None]).ravel()
        return np.concatenate([U, -U, Pp])
    ec, ef = sample(Nc), sample(Nf)
    assert np.abs(o.prolong_add(1, ec, np.zeros(o.length(1))) - ef).max() < 1e-13


def test_restrict_is_transpose_with_dirichlet_zeroed():
    o = oracle.Oracle(8, n_coarse=4)
    P = o.prolongation(1).toarray()
    rf = svk_inputs.random_vector(8, 11)
    rc = o.restrict(1, rf)
    ref = P.T @ rf
    ref[o.dirichlet(0)] = 0
    assert rel(rc, ref) < 1e-14


# ---------------------------------------------------------------- coarse / V-cycle
def test_coarse_solve_is_pinv():
    o = oracle.Oracle(4)
    A = o.csr(0).toarray()
    I = np.flatnonzero(~o.dirichlet(0))
    Ap = np.linalg.pinv(A[np.ix_(I, I)])
    for seed in (1, 2):
        b = svk_inputs.random_vector(4, seed)
        b[o.dirichlet(0)] = 0
        x = o.coarse_solve(b)
        assert rel(x[I], Ap @ b[I]) < 1e-12
        assert np.all(x[o.dirichlet(0)] == 0)


@pytest.mark.parametrize("N", [8, 16])
def test_vcycle_vs_dense_mg(N):
    o = oracle.Oracle(N)
    M = brute.DenseMG(N)
    for seed in (1, 2):
        b = svk_inputs.random_vector(N, seed)
        b[o.dirichlet(o.fine)] = 0
        assert rel(o.vcycle(b), M.vcycle(b)) < 1e-12
        x0 = svk_inputs.random_vector(N, seed + 7)
        assert rel(o.vcycle(b, x0) - x0, M.vcycle(b, x0.copy()) - x0) < 1e-12


def test_vcycle_fixed_point_and_linearity(o16):
    l = o16.fine
    A = o16.csr(l).toarray()
    d = o16.dirichlet(l)
    I = np.flatnonzero(~d)
    b, x0 = o16.problem(oracle.MMS_PAPER)
    rhs = b[I] - A[np.ix_(I, np.flatnonzero(d))] @ x0[d]
    xs = x0.copy()
    xs[I] = np.linalg.lstsq(A[np.ix_(I, I)], rhs, rcond=None)[0]
    out = o16.vcycle(b, xs)
    assert np.abs(out - xs).max() < 1e-10 * np.abs(xs).max()
    z = np.zeros_like(b)
    assert np.all(o16.vcycle(z) == 0)
    r = svk_inputs.random_vector(16, 3)
    r[d] = 0
    assert rel(o16.vcycle(3 * r), 3 * o16.vcycle(r)) < 1e-13


# ---------------------------------------------------------------- FGMRES
@pytest.mark.parametrize("k", [3, 8, 15])
def test_fgmres_matches_least_squares_definition(o16, k):
    """x_k = x0 + Z_k y, y = argmin ||r0 - A Z_k y||, Z_k = M V_k, V_k an orthonormal
    (CGS2) basis of the Krylov space of A M -- the definition of right-preconditioned
    (F)GMRES with a fixed linear preconditioner."""
    l = o16.fine
    b, x0 = o16.problem(oracle.MMS_PAPER)
    r0 = o16.residual(l, x0, b)
    V = [r0 / np.linalg.norm(r0)]
    Z = []
    for j in range(k):
        Z.append(o16.vcycle(V[j]))
        w = o16.matvec(l, Z[j])
        for _ in range(2):  # CGS2
            Vm = np.array(V)
            w = w - Vm.T @ (Vm @ w)
        V.append(w / np.linalg.norm(w))
    AZ = np.array([o16.matvec(l, z) for z in Z]).T
    y = np.linalg.lstsq(AZ, r0, rcond=None)[0]
    x_def = x0 + np.array(Z).T @ y
    x, its, hist, tr, st = o16.fgmres(b, x0, rtol=0.0, maxit=k)
    assert its == k
    assert rel(x - x0, x_def - x0) < 1e-9
    assert abs(hist[-1] - np.linalg.norm(r0 - AZ @ y) / np.linalg.norm(r0)) < 1e-9 * max(hist[-1], 1e-30) + 1e-14


@pytest.mark.parametrize("kind,N", [(oracle.MMS_PAPER, 8), (oracle.MMS_PAPER, 16), (oracle.MMS_PAPER, 32),
                                    (oracle.MMS_INSPACE, 16)])
def test_manufactured_solution_nodally_exact(kind, N):
    """The Q2-Q1 solution of the paper's MMS is exact at every DOF point on
    uniform grids; the in-space MMS lies in the FE space.  Pins assembly, sign (reading 1),
    boundary data (reading 2), RHS quadrature and the whole solver."""
    o = oracle.Oracle(N)
    b, x0 = o.problem(kind)
    x, its, hist, tr, st = o.fgmres(b, x0, rtol=1e-12, maxit=60)
    assert st == 0
    ex = o.exact(kind)
    ux, uy, p = o.split(x, o.fine)
    eux, euy, ep = o.split(ex, o.fine)
    assert np.abs(ux - eux).max() < 1e-10
    assert np.abs(uy - euy).max() < 1e-10
    assert np.abs((p - p.mean()) - (ep - ep.mean())).max() < 1e-8
    assert ep[-1, -1] == pytest.approx(GOLD["mms_pressure_at_1_1"]["value"]) or kind != oracle.MMS_PAPER


def test_iteration_counts_oracle_internal():
    """Regression of the oracle's FGMRES+V(1,1)-Vanka counts (omega=0.8, tol 1e-10).
    Oracle-internal (the paper prints no counts): guards against silent drift."""
    its = {}
    for N in (16, 32, 64):
        o = oracle.Oracle(N)
        b, x0 = o.problem(oracle.MMS_PAPER)
        its[N] = o.fgmres(b, x0)[1]
    assert its == {16: 18, 32: 19, 64: 19}


# ---------------------------------------------------------------- sampled (full-size) oracle
@pytest.mark.parametrize("N", [4, 8, 16])
def test_sampled_sweep_and_residual_equal_global_oracle(N):
    """The local-box evaluation used for full-size parity equals the global oracle."""
    o = oracle.Oracle(N, n_coarse=4)
    l = o.fine
    x = svk_inputs.random_vector(N, 21)
    b = svk_inputs.random_vector(N, 22)
    idx = np.arange(o.length(l), dtype=np.int64)
    xs = o.sweep(l, x, b)
    rs = o.residual(l, x, b)
    assert rel(oracle.sweep_sample(N, x, b, idx) - x, xs - x) < 1e-12
    assert rel(oracle.residual_sample(N, x, b, idx), rs) < 1e-13
    xs2 = oracle.Oracle(N, weighting=oracle.WEIGHT_SCALAR, omega=0.5).sweep(l, x, b)
    assert rel(oracle.sweep_sample(N, x, b, idx, omega=0.5, weighting=oracle.WEIGHT_SCALAR) - x, xs2 - x) < 1e-12


@pytest.mark.parametrize("N", [8, 16])
def test_sampled_transfers_equal_global_oracle(N):
    """The local residual+restriction and prolongation samplers used for full-size
    parity equal the global oracle (explicit P / P^T) on every DOF."""
    o = oracle.Oracle(N, n_coarse=4)
    l = o.fine
    x = svk_inputs.random_vector(N, 31)
    b = svk_inputs.random_vector(N, 32)
    rc = o.restrict(l, o.residual(l, x, b))
    idxc = np.arange(o.length(l - 1), dtype=np.int64)
    assert rel(oracle.restrict_residual_sample(N, x, b, idxc), rc) < 1e-13
    ec = svk_inputs.random_vector(N // 2, 33)
    ec[o.dirichlet(l - 1)] = 0.0
    xf = svk_inputs.random_vector(N, 34)
    idxf = np.arange(o.length(l), dtype=np.int64)
    assert rel(oracle.prolong_sample(N, ec, xf, idxf) - xf, o.prolong_add(l, ec, xf) - xf) < 1e-14


def test_degenerate_cases_single_level_and_zero_rhs():
    """Degenerate cases of the method: with a single level (N = N0) the V-cycle is
    the exact minimum-norm solve, so FGMRES with that exact preconditioner
    converges in one iteration; a zero right-hand side with zero initial guess
    needs none."""
    o = oracle.Oracle(4, n_coarse=4)
    b, x0 = o.problem(oracle.MMS_PAPER)
    x, its, hist, tr, st = o.fgmres(b, x0, rtol=1e-10, maxit=10)
    assert st == 0 and its == 1 and tr < 1e-12
    z = np.zeros_like(b)
    x, its, hist, tr, st = o.fgmres(z, z, rtol=1e-10, maxit=10)
    assert st == 0 and its == 0 and np.all(x == 0)


@pytest.mark.parametrize("nu", [0.37, 7.5])
def test_viscosity_operator_and_sweep_vs_bruteforce(nu):
    """nu != 1: L = nu (M (x) K + K (x) M) while B is unchanged -- the assembled
    operator and one Vanka sweep against the brute force built with the same nu."""
    N = 8
    o = oracle.Oracle(N, n_coarse=N, nu=nu)
    B = brute.full_operator(N, nu)
    A = o.csr(0).toarray()
    assert np.abs(A - B).max() <= 1e-14 * np.abs(B).max()
    D = brute.Dense(N, nu=nu)
    x = svk_inputs.random_vector(N, 71)
    b = svk_inputs.random_vector(N, 72)
    assert rel(o.sweep(0, x, b) - x, D.sweep(x, b) - x) < 1e-12
    # sensitivity: the nu = 1 operator differs
    assert np.abs(brute.full_operator(N, 1.0) - B).max() > 1e-3 * np.abs(B).max()


@pytest.mark.parametrize("nu1,nu2,omega", [(2, 2, 0.7), (0, 1, 0.8), (1, 0, 0.8), (3, 1, 0.6)])
def test_vcycle_smoothing_counts_vs_dense_mg(nu1, nu2, omega):
    """V(nu1, nu2) (alg:mg) with other sweep counts and weights against
    the dense brute-force multigrid with the same counts; another count differs."""
    N = 16
    o = oracle.Oracle(N, omega=omega, nu1=nu1, nu2=nu2)
    M = brute.DenseMG(N, omega=omega, nu1=nu1, nu2=nu2)
    b = svk_inputs.random_vector(N, 81)
    b[o.dirichlet(o.fine)] = 0
    want = M.vcycle(b)
    assert rel(o.vcycle(b), want) < 1e-12
    assert rel(brute.DenseMG(N, omega=omega, nu1=nu1 + 1, nu2=nu2).vcycle(b), want) > 1e-6
