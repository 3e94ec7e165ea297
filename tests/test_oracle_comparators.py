"""Pins for the oracle's Braess-Sarazin and Schur-Uzawa relaxations (SURVEY 8(f)
NEXT-1; alg:bs P:236-241, alg:uz P:313-320).  No GPU.

Each check uses something other than the oracle's own formula:
  * the dense operator of brute.py (exact 1D integration + Kronecker products),
  * the limits the paper's derivations fix: with an exact inner solve, inexact
    Braess-Sarazin (eq:bsfact) IS the original under-relaxed solve of
    [[tD, B^T], [B, 0]], and Schur-Uzawa IS the solve of the block
    lower-triangular system eq:uzblock (whose sign it pins, DESIGN reading 19),
  * invariants (fixed point of the exact solution, linearity, Dirichlet rows).
"""
import numpy as np
import pytest

import brute
import oracle
import svk_inputs


def rel(a, b):
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


def dense_parts(N, t=1.0):
    """(A, free velocity mask, B, D) from the brute-force dense operator."""
    A = brute.full_operator(N)
    d = brute.dirichlet(N)
    nvel = 2 * (2 * N + 1) ** 2
    fu = ~d[:nvel]
    B = A[nvel:, :nvel][:, fu]            # pressure rows, free velocity columns
    D = np.diag(A[:nvel, :nvel])[fu]      # diag(L) on free velocity DOFs
    return A, d, fu, B, D


def residual_dense(A, d, x, b):
    xx = x.copy()
    r = b - A @ xx
    r[d] = 0.0
    return r


def consistent(A, d, x, b, N):
    """b with its pressure part shifted so that sum(r_p) = 0: S is singular (constant
    pressure, reading 3) and the Jacobi limits exist only for consistent data."""
    b = b.copy()
    npp = (N + 1) ** 2
    b[-npp:] -= residual_dense(A, d, x, b)[-npp:].mean()
    return b


def demean_p(v, N):
    v = v.copy()
    npp = (N + 1) ** 2
    v[-npp:] -= v[-npp:].mean()
    return v


@pytest.mark.parametrize("N", [4, 8])
def test_schur_complement_equals_dense_product(N):
    o = oracle.Oracle(N, n_coarse=N)
    o.set_relax(oracle.RELAX_BS, t=2.0)
    _, _, _, B, D = dense_parts(N)
    S = -(B / D) @ B.T / 2.0
    assert rel(o.schur(0).toarray(), S) < 1e-13


@pytest.mark.parametrize("N", [4, 8])
def test_bs_exact_inner_solve_is_original_braess_sarazin(N):
    """nj -> infinity: x_out - x = omega_BS [[tD, B^T],[B, 0]]^+ r (modulo the constant pressure)."""
    t, wbs = 1.5, 0.9
    o = oracle.Oracle(N, n_coarse=N)
    o.set_relax(oracle.RELAX_BS, t=t, omega_r=wbs, omega_j=0.9, nj=4000)
    A, d, fu, B, D = dense_parts(N)
    nvel = fu.size
    K = np.block([[np.diag(t * D), B.T], [B, np.zeros((B.shape[0], B.shape[0]))]])
    for seed in (1, 2):
        x = svk_inputs.random_vector(N, seed)
        b = consistent(A, d, x, svk_inputs.random_vector(N, seed + 50), N)
        r = residual_dense(A, d, x, b)
        rr = np.concatenate([r[:nvel][fu], r[nvel:]])
        dd = np.linalg.lstsq(K, rr, rcond=None)[0]
        want = np.zeros_like(x)
        want[:nvel][fu] = wbs * dd[: fu.sum()]
        want[nvel:] = wbs * dd[fu.sum():]
        got = o.relax_sweep(0, x, b) - x
        assert rel(demean_p(got, N), demean_p(want, N)) < 1e-9


@pytest.mark.parametrize("N", [4, 8])
def test_su_exact_inner_solve_solves_block_lower_triangular_system(N):
    """eq:uzblock: t D du = r_u and S dp = r_p - B du, S = -(1/t) B D^-1 B^T."""
    t = 1.25
    o = oracle.Oracle(N, n_coarse=N)
    o.set_relax(oracle.RELAX_SU, t=t, omega_j=0.9, nj=4000)
    A, d, fu, B, D = dense_parts(N)
    nvel = fu.size
    S = -(B / D) @ B.T / t
    x = svk_inputs.random_vector(N, 7)
    b = consistent(A, d, x, svk_inputs.random_vector(N, 8), N)
    r = residual_dense(A, d, x, b)
    delta = o.relax_sweep(0, x, b) - x
    du, dp = delta[:nvel][fu], delta[nvel:]
    assert rel(t * D * du, r[:nvel][fu]) < 1e-13
    assert np.all(delta[:nvel][~fu] == 0)
    assert rel(S @ dp, r[nvel:] - B @ du) < 1e-9
    # the paper's literal alg:uz sign (S dp = B du - r_p) would give the opposite
    assert rel(S @ dp, B @ du - r[nvel:]) > 1.0


@pytest.mark.parametrize("kind", [oracle.RELAX_BS, oracle.RELAX_SU])
def test_comparator_fixed_point_linearity_dirichlet(kind):
    N = 8
    o = oracle.Oracle(N, n_coarse=N)
    o.set_relax(kind, t=1.0, omega_r=1.0, omega_j=0.8 if kind == oracle.RELAX_BS else 0.4,
                nj=3 if kind == oracle.RELAX_BS else 1)
    A = brute.full_operator(N)
    dmask = brute.dirichlet(N)
    xs = svk_inputs.random_vector(N, 3)
    b = A @ xs
    b[dmask] = xs[dmask]
    assert rel(o.relax_sweep(0, xs, b), xs) < 1e-13          # exact solution is a fixed point
    x = svk_inputs.random_vector(N, 4)
    b = svk_inputs.random_vector(N, 5)
    a = -1.75
    assert rel(o.relax_sweep(0, a * x, a * b) - a * x, a * (o.relax_sweep(0, x, b) - x)) < 1e-13
    assert np.array_equal(o.relax_sweep(0, x, b)[dmask], x[dmask])


def test_comparator_iteration_counts_oracle_internal():
    """FGMRES + V(1,1) with BS (t=1, omega_BS=1, omega_J=0.8, 3 Jacobi) and SU
    (t=1, omega_J=0.4, 1 Jacobi), tol 1e-10, paper MMS.  Oracle-internal
    regression (the paper prints curves, no counts); the discrete solution is the
    manufactured one (nodal exactness), whatever the relaxation."""
    its = {}
    for name, kind, kw in (("bs", oracle.RELAX_BS, dict(t=1, omega_r=1, omega_j=0.8, nj=3)),
                           ("su", oracle.RELAX_SU, dict(t=1, omega_j=0.4, nj=1))):
        o = oracle.Oracle(16)
        o.set_relax(kind, **kw)
        b, x0 = o.problem(oracle.MMS_PAPER)
        x, k, _, tr, st = o.fgmres(b, x0, rtol=1e-10, maxit=300)
        assert st == 0 and tr < 1e-9
        ex = o.exact(oracle.MMS_PAPER)
        nv = (2 * 16 + 1) ** 2
        assert np.abs(x[: 2 * nv] - ex[: 2 * nv]).max() < 1e-9
        its[name] = k
    assert its == {"bs": 14, "su": 31}


# ------------------------------------------------- block-triangular preconditioner (alg:bt)
def q1_mass_1d(N):
    """1D Q1 mass matrix by exact polynomial integration (brute.Q1 bases)."""
    h = 1.0 / N
    me = np.array([[brute._int01(a * b) * h for b in brute.Q1] for a in brute.Q1])
    m = np.zeros((N + 1, N + 1))
    for e in range(N):
        m[e:e + 2, e:e + 2] += me
    return m


@pytest.mark.parametrize("N", [4, 8])
def test_pressure_mass_matrix_is_q1_kronecker(N):
    o = oracle.Oracle(N, n_coarse=4)
    o.set_precond(oracle.PRECOND_BT)
    m = q1_mass_1d(N)
    assert rel(o.mass(o.fine).toarray(), np.kron(m, m)) < 1e-14


@pytest.mark.parametrize("N", [8, 16])
def test_bt_many_cycles_is_exact_upper_block_triangular_solve(N):
    """alg:bt with converged block solves = [[L, B^T],[0, -M]]^{-1} r (eq:schuruzawablock,
    P:343-357) on the interior system; dense brute-force L, B and Q1 mass."""
    o = oracle.Oracle(N)
    o.set_precond(oracle.PRECOND_BT, cycles=60, nu=3, omega_u=1.0, omega_p=0.6)
    A = brute.full_operator(N)
    d = brute.dirichlet(N)
    nvel = 2 * (2 * N + 1) ** 2
    fu = ~d[:nvel]
    m = q1_mass_1d(N)
    M = np.kron(m, m)
    L = A[:nvel, :nvel][np.ix_(fu, fu)]
    BT = A[:nvel, nvel:][fu]
    K = np.block([[L, BT], [np.zeros((M.shape[0], L.shape[0])), -M]])
    r = svk_inputs.random_vector(N, 11)
    r[d] = 0.0
    z = o.precond_apply(r)
    want = np.linalg.solve(K, np.concatenate([r[:nvel][fu], r[nvel:]]))
    assert np.all(z[:nvel][~fu] == 0)
    assert rel(np.concatenate([z[:nvel][fu], z[nvel:]]), want) < 1e-11


def test_bt_linear_and_fgmres_oracle_internal():
    o = oracle.Oracle(16)
    o.set_precond(oracle.PRECOND_BT)
    r = svk_inputs.random_vector(16, 12)
    r[o.dirichlet(o.fine)] = 0.0
    assert rel(o.precond_apply(-2.0 * r), -2.0 * o.precond_apply(r)) < 1e-14
    b, x0 = o.problem(oracle.MMS_PAPER)
    x, k, _, tr, st = o.fgmres(b, x0, rtol=1e-10, maxit=200)
    assert st == 0 and tr < 1e-9
    ex = o.exact(oracle.MMS_PAPER)
    nv = (2 * 16 + 1) ** 2
    assert np.abs(x[: 2 * nv] - ex[: 2 * nv]).max() < 1e-9
    assert k == 18  # oracle-internal regression (3 V(3,3) per block, omega 1.0 / 0.6)
