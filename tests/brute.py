"""Independent dense NumPy brute force for tiny grids (N <= 16).

Used only to pin the oracle.  It shares no code with oracle/oracle.cpp and
derives everything a different way:
  * 1D element matrices by EXACT polynomial integration (numpy.polynomial) of
    Lagrange bases built from their roots, instead of 2D Gauss quadrature;
  * the 2D operator as Kronecker products of assembled 1D matrices
    (L = nu (M (x) K + K (x) M), B_x = -C (x) G, B_y = -G (x) C) instead of
    element-by-element 2D assembly;
  * patches via explicit 0/1 restriction matrices V_i and numpy.linalg.inv;
  * interpolation as Kronecker products of 1D Lagrange-evaluation matrices;
  * the coarse solve as numpy.linalg.pinv.
Sign convention b(v,q) = -int q div v (reading 1).
"""
from __future__ import annotations

import numpy as np
from numpy.polynomial import Polynomial as Poly


def lagrange(nodes):
    out = []
    for a, xa in enumerate(nodes):
        others = [x for b, x in enumerate(nodes) if b != a]
        p = Poly.fromroots(others)
        out.append(p / p(xa))
    return out


Q2 = lagrange([0.0, 0.5, 1.0])
Q1 = lagrange([0.0, 1.0])


def _int01(p: Poly) -> float:
    P = p.integ()
    return float(P(1.0) - P(0.0))


def element_1d(h: float):
    """K_e (3x3), M_e (3x3), G_e (2x3) = int phi_c psi_a', C_e (2x3) = int phi_c psi_a."""
    K = np.array([[_int01(a.deriv() * b.deriv()) / h for b in Q2] for a in Q2])
    M = np.array([[_int01(a * b) * h for b in Q2] for a in Q2])
    G = np.array([[_int01(c * a.deriv()) for a in Q2] for c in Q1])
    Cm = np.array([[_int01(c * a) * h for a in Q2] for c in Q1])
    return K, M, G, Cm


def global_1d(N: int):
    h = 1.0 / N
    Ke, Me, Ge, Ce = element_1d(h)
    nl = 2 * N + 1
    K = np.zeros((nl, nl)); M = np.zeros((nl, nl))
    G = np.zeros((N + 1, nl)); Cm = np.zeros((N + 1, nl))
    for e in range(N):
        v = [2 * e, 2 * e + 1, 2 * e + 2]
        p = [e, e + 1]
        K[np.ix_(v, v)] += Ke
        M[np.ix_(v, v)] += Me
        G[np.ix_(p, v)] += Ge
        Cm[np.ix_(p, v)] += Ce
    return K, M, G, Cm


def full_operator(N: int, nu: float = 1.0) -> np.ndarray:
    K, M, G, Cm = global_1d(N)
    L = nu * (np.kron(M, K) + np.kron(K, M))   # row index j*(2N+1)+i: first factor acts on y
    Bx = -np.kron(Cm, G)
    By = -np.kron(G, Cm)
    nv, npp = L.shape[0], Bx.shape[0]
    A = np.zeros((2 * nv + npp, 2 * nv + npp))
    A[:nv, :nv] = L
    A[nv:2 * nv, nv:2 * nv] = L
    A[2 * nv:, :nv] = Bx
    A[2 * nv:, nv:2 * nv] = By
    A[:nv, 2 * nv:] = Bx.T
    A[nv:2 * nv, 2 * nv:] = By.T
    return A


def dirichlet(N: int) -> np.ndarray:
    nl = 2 * N + 1
    i = np.arange(nl)
    edge = (i == 0) | (i == nl - 1)
    lat = (edge[None, :] | edge[:, None]).ravel()
    return np.concatenate([lat, lat, np.zeros((N + 1) ** 2, bool)])


def patch_dofs(N: int, kx: int, ky: int, with_dirichlet: bool = False):
    nl = 2 * N + 1
    nv = nl * nl
    d = dirichlet(N)
    out = []
    for comp in range(2):
        for j in range(2 * ky - 2, 2 * ky + 3):
            for i in range(2 * kx - 2, 2 * kx + 3):
                if 0 <= i < nl and 0 <= j < nl:
                    g = comp * nv + j * nl + i
                    if with_dirichlet or not d[g]:
                        out.append(g)
    out.append(2 * nv + ky * (N + 1) + kx)
    return np.array(out, dtype=np.int64)


class Dense:
    """Dense Stokes level + Vanka operator for tiny N."""

    def __init__(self, N: int, nu: float = 1.0, omega: float = 0.8, weighting: str = "mult"):
        self.N, self.nu, self.omega = N, nu, omega
        self.A = full_operator(N, nu)
        self.dir = dirichlet(N)
        self.n = self.A.shape[0]
        self.patches = [patch_dofs(N, kx, ky) for ky in range(N + 1) for kx in range(N + 1)]
        mult = np.zeros(self.n)
        for p in self.patches:
            mult[p] += 1
        self.mult = mult
        w = np.where(mult > 0, omega / np.maximum(mult, 1), 0.0) if weighting == "mult" else np.full(self.n, omega)
        S = np.zeros((self.n, self.n))
        for p in self.patches:
            # V_i A V_i^T and V_i^T (.) V_i written as index extraction / scatter
            Ai = self.A[np.ix_(p, p)]
            S[np.ix_(p, p)] += np.diag(w[p]) @ np.linalg.inv(Ai)
        self.S = S          # sum_i V_i^T W_i A_i^{-1} V_i
        self.mask = (~self.dir).astype(float)

    def residual(self, x, b):
        return self.mask * (b - self.A @ x)

    def sweep(self, x, b):
        return x + self.S @ self.residual(x, b)

    def interior_matrix(self):
        I = np.flatnonzero(~self.dir)
        return I, self.A[np.ix_(I, I)]


def interp_1d(Nc: int):
    """(P2: (4Nc+1)x(2Nc+1), P1: (2Nc+1)x(Nc+1)) coarse Lagrange bases at fine points."""
    Nf = 2 * Nc
    P2 = np.zeros((2 * Nf + 1, 2 * Nc + 1))
    for i in range(2 * Nf + 1):
        x = i / (2 * Nf)
        e = min(int(np.floor(x * Nc)), Nc - 1)
        t = x * Nc - e
        for a in range(3):
            P2[i, 2 * e + a] = Q2[a](t)
    P1 = np.zeros((Nf + 1, Nc + 1))
    for k in range(Nf + 1):
        x = k / Nf
        e = min(int(np.floor(x * Nc)), Nc - 1)
        t = x * Nc - e
        for c in range(2):
            P1[k, e + c] = Q1[c](t)
    P2[np.abs(P2) < 1e-15] = 0.0
    P1[np.abs(P1) < 1e-15] = 0.0
    return P2, P1


def prolongation(Nc: int) -> np.ndarray:
    P2, P1 = interp_1d(Nc)
    V = np.kron(P2, P2)
    Pp = np.kron(P1, P1)
    nf, nc = V.shape
    P = np.zeros((2 * nf + Pp.shape[0], 2 * nc + Pp.shape[1]))
    P[:nf, :nc] = V
    P[nf:2 * nf, nc:2 * nc] = V
    P[2 * nf:, 2 * nc:] = Pp
    return P


class DenseMG:
    """Dense V(1,1) per alg:mg on brute-force components."""

    def __init__(self, N: int, N0: int = 4, nu: float = 1.0, omega: float = 0.8, nu1: int = 1, nu2: int = 1):
        self.nu1, self.nu2 = nu1, nu2
        self.levels = []
        n = N0
        while n <= N:
            self.levels.append(Dense(n, nu, omega))
            n *= 2
        self.P = [None] + [prolongation(self.levels[l - 1].N) for l in range(1, len(self.levels))]
        I, A0 = self.levels[0].interior_matrix()
        self.I0, self.A0pinv = I, np.linalg.pinv(A0)

    def coarse(self, b):
        x = np.zeros_like(b)
        x[self.I0] = self.A0pinv @ b[self.I0]
        return x

    def mg(self, l, b, x):
        if l == 0:
            return self.coarse(b)
        Lv = self.levels[l]
        for _ in range(self.nu1):
            x = Lv.sweep(x, b)
        r = Lv.residual(x, b)
        rc = self.P[l].T @ r
        rc[self.levels[l - 1].dir] = 0.0
        ec = self.coarse(rc) if l == 1 else self.mg(l - 1, rc, np.zeros_like(rc))
        x = x + self.P[l] @ ec
        for _ in range(self.nu2):
            x = Lv.sweep(x, b)
        return x

    def vcycle(self, b, x=None):
        x = np.zeros_like(b) if x is None else x
        return self.mg(len(self.levels) - 1, b, x)
