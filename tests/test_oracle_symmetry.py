"""Pins (no GPU) for the coefficient identities the B200 sweep kernels exploit.

k_factor_setup and tools/gen_solve.py load each distinct stencil / patch-solve
value once and apply it at every position where it occurs.
That is exact only if the discrete operator has these symmetries; here they are
checked on the oracle's explicitly assembled CSR matrix (O1), which
shares nothing with the CUDA path:

* generic patch (A_i = V_i A V_i^T): the velocity block is the same 25x25
  Lw for both components with no u_x-u_y coupling, Lw is symmetric and invariant
  under swapping the two axes of the 5x5 window, and b_y = swap(b_x);
* hence B = S T Lw^-1 T^T S (the reflection-basis inverse the kernels apply) is
  block diagonal EE/EO/OE/OO, symmetric and swap invariant;
* the Laplacian rows at interior lattice points depend only on (|drow|, |dcol|),
  the (odd row, even column) stencil is the transpose of the (even row, odd
  column) one, and the two B rows of an interior pressure node are transposes.
"""
import numpy as np
import pytest

import oracle
import brute

N = 16


@pytest.fixture(scope="module")
def A():
    return oracle.Oracle(N, n_coarse=N).csr(0).toarray()


def swap_perm():
    # window index oy*5+ox -> ox*5+oy
    return np.array([(q % 5) * 5 + q // 5 for q in range(25)])


def generic_patch(A, kx=8, ky=8):
    d = brute.patch_dofs(N, kx, ky)  # [u_x window (row-major, x fastest), u_y window, p_k]
    assert len(d) == 51
    return A[np.ix_(d, d)]


def test_generic_patch_structure(A):
    Ai = generic_patch(A)
    Lx, Ly, Cxy = Ai[:25, :25], Ai[25:50, 25:50], Ai[:25, 25:50]
    bx, by = Ai[50, :25], Ai[50, 25:50]
    s = np.abs(Lx).max()
    assert np.abs(Lx - Ly).max() <= 1e-15 * s
    assert np.abs(Cxy).max() == 0.0
    assert np.abs(Lx - Lx.T).max() <= 1e-15 * s
    P = swap_perm()
    assert np.abs(Lx[np.ix_(P, P)] - Lx).max() <= 1e-15 * s
    assert np.abs(by - bx[P]).max() <= 1e-15 * np.abs(bx).max()
    assert Ai[50, 50] == 0.0


def test_reflection_basis_inverse_is_symmetric_and_swap_invariant(A):
    Ai = generic_patch(A)
    Lw = Ai[:25, :25]
    T5 = np.array([[1, 0, 0, 0, 1], [0, 1, 0, 1, 0], [0, 0, 1, 0, 0], [1, 0, 0, 0, -1], [0, 1, 0, -1, 0]], float)
    S5 = np.array([0.5, 0.5, 1.0, 0.5, 0.5])
    T = np.kron(T5, T5)          # (ty,tx) <- (vy,vx)
    S = np.diag(np.kron(S5, S5))
    B = S @ T @ np.linalg.inv(Lw) @ T.T @ S
    s = np.abs(B).max()
    even = np.arange(5) < 3
    par_y, par_x = np.repeat(even, 5), np.tile(even, 5)
    cross = (par_y[:, None] != par_y[None, :]) | (par_x[:, None] != par_x[None, :])
    assert np.abs(B[cross]).max() <= 1e-13 * s          # block diagonal
    assert np.abs(B - B.T).max() <= 1e-13 * s           # symmetric
    P = swap_perm()                                     # swap commutes with T (same T5 per axis)
    assert np.abs(B[np.ix_(P, P)] - B).max() <= 1e-13 * s
    # and it is the velocity inverse: T^-1 S^-1 B S^-1 T^-T = Lw^-1
    Ti = np.linalg.inv(T)
    Si = np.linalg.inv(S)
    assert np.abs(Ti @ Si @ B @ Si @ Ti.T - np.linalg.inv(Lw)).max() <= 1e-12 * np.abs(np.linalg.inv(Lw)).max()
    # Schur vectors: c_y = swap(c_x)
    bx, by = Ai[50, :25], Ai[50, 25:50]
    cx, cy = np.linalg.solve(Lw, bx), np.linalg.solve(Lw, by)
    assert np.abs(cy - cx[P]).max() <= 1e-13 * np.abs(cx).max()


def _stencil(A, comp, i, j):
    """5x5 Laplacian coefficients of lattice point (i, j), component comp, offsets -2..2"""
    nl = 2 * N + 1
    nv = nl * nl
    row = A[comp * nv + j * nl + i]
    out = np.zeros((5, 5))
    for db in range(-2, 3):
        for da in range(-2, 3):
            out[db + 2, da + 2] = row[comp * nv + (j + db) * nl + (i + da)]
    return out


def test_laplacian_stencil_symmetries(A):
    # interior points of the four parity classes (row parity, column parity)
    st = {(py, px): _stencil(A, 0, 10 + px, 10 + py) for py in (0, 1) for px in (0, 1)}
    s = max(np.abs(v).max() for v in st.values())
    for (py, px), L in st.items():
        assert np.abs(L - L[::-1, :]).max() <= 1e-15 * s  # reflection in y
        assert np.abs(L - L[:, ::-1]).max() <= 1e-15 * s  # reflection in x
        if py == px:
            assert np.abs(L - L.T).max() <= 1e-15 * s
        # u_y has the same stencil
        i, j = 10 + px, 10 + py
        assert np.abs(_stencil(A, 1, i, j) - L).max() <= 1e-15 * s
    assert np.abs(st[(0, 1)] - st[(1, 0)].T).max() <= 1e-15 * s


def test_interior_pressure_rows_are_transposes(A):
    nl = 2 * N + 1
    nv = nl * nl
    kx = ky = 8
    row = A[2 * nv + ky * (N + 1) + kx]
    wx = np.zeros((5, 5))
    wy = np.zeros((5, 5))
    for oy in range(5):
        for ox in range(5):
            g = (2 * ky - 2 + oy) * nl + (2 * kx - 2 + ox)
            wx[oy, ox] = row[g]
            wy[oy, ox] = row[nv + g]
    assert np.abs(wy - wx.T).max() <= 1e-15 * np.abs(wx).max()
    # and nothing outside the 5x5 window
    assert np.count_nonzero(row[:2 * nv]) == np.count_nonzero(wx) + np.count_nonzero(wy)
