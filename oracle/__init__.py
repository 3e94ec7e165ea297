"""CPU oracle for the Vanka / V-cycle / FGMRES hot path (arXiv 2401.06277).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` leg may import this
package.  The product path (``paper_2401_06277_b200``) never imports it and
shares no code with it.

The arithmetic lives in ``oracle/oracle.cpp`` (plain C++17 + OpenMP, fp64);
this module only compiles it with g++ and marshals numpy arrays through ctypes.
Vector layout (compact, per level with N elements per side):
``[u_x ((2N+1)^2, x fastest), u_y ((2N+1)^2), p ((N+1)^2)]``.
Level 0 is the coarsest (alg:mg).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.cpp")
_LIB = os.path.join(_HERE, "liboracle.so")
_lock = threading.Lock()
_lib = None

MMS_ZERO, MMS_PAPER, MMS_INSPACE, CAVITY = 0, 1, 2, 3
RELAX_VANKA, RELAX_BS, RELAX_SU = 0, 1, 2
PRECOND_MG, PRECOND_BT = 0, 1
WEIGHT_MULT, WEIGHT_SCALAR = 0, 1


def build(force: bool = False) -> str:
    """Compile oracle.cpp into liboracle.so (g++, -O2, OpenMP)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + ".tmp%d" % os.getpid()
        cmd = ["g++", "-O2", "-std=c++17", "-fopenmp", "-shared", "-fPIC", _SRC, "-o", tmp]
        subprocess.run(cmd, check=True)
        os.replace(tmp, _LIB)
    return _LIB


def _load():
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        build()
        lib = C.CDLL(_LIB)
        P, I, I64, D = C.c_void_p, C.c_int, C.c_int64, C.c_double
        sig = {
            "orc_create": (P, [I, I, D, D, I, I, I, I]),
            "orc_destroy": (None, [P]),
            "orc_num_levels": (I, [P]),
            "orc_level_len": (I64, [P, I]),
            "orc_level_n": (I, [P, I]),
            "orc_num_groups": (I, [P, I]),
            "orc_nnz": (I64, [P, I]),
            "orc_max_threads": (I, []),
            "orc_csr": (None, [P, I, P, P, P]),
            "orc_dirichlet": (None, [P, I, P]),
            "orc_weights": (None, [P, I, P]),
            "orc_patch": (I, [P, I, I, I, P]),
            "orc_patch_group": (I, [P, I, I, I]),
            "orc_total_patch_dofs": (I64, [P, I]),
            "orc_problem": (None, [P, I, I, P, P]),
            "orc_exact": (None, [P, I, I, P]),
            "orc_matvec": (None, [P, I, P, P]),
            "orc_residual": (None, [P, I, P, P, P]),
            "orc_vanka_sweep": (None, [P, I, P, P, P]),
            "orc_restrict": (None, [P, I, P, P]),
            "orc_prolong_add": (None, [P, I, P, P]),
            "orc_prolongation_csr": (None, [P, I, P, P, P]),
            "orc_prolongation_nnz": (I64, [P, I]),
            "orc_coarse_solve": (None, [P, P, P]),
            "orc_vcycle": (None, [P, P, P]),
            "orc_fgmres": (I, [P, P, P, D, I, P, P, P]),
            "orc_sweep_sample": (None, [I, D, D, I, P, P, P, I64, P]),
            "orc_residual_sample": (None, [I, D, P, P, P, I64, P]),
            "orc_restrict_residual_sample": (None, [I, D, P, P, P, I64, P]),
            "orc_prolong_sample": (None, [I, P, P, P, I64, P]),
            "orc_set_relax": (I, [P, I, D, D, D, I]),
            "orc_relax_sweep": (None, [P, I, P, P, P]),
            "orc_schur_nnz": (I64, [P, I]),
            "orc_schur_csr": (None, [P, I, P, P, P]),
            "orc_set_precond": (I, [P, I, I, I, D, D]),
            "orc_precond_apply": (None, [P, P, P]),
            "orc_mass_nnz": (I64, [P, I]),
            "orc_mass_csr": (None, [P, I, P, P, P]),
        }
        for name, (res, args) in sig.items():
            f = getattr(lib, name)
            f.restype = res
            f.argtypes = args
        _lib = lib
        return lib


def _ptr(a: np.ndarray):
    assert a.flags["C_CONTIGUOUS"]
    return a.ctypes.data_as(C.c_void_p)


def _f64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)


def max_threads() -> int:
    return int(_load().orc_max_threads())


def sweep_sample(N: int, x, b, idx, nu: float = 1.0, omega: float = 0.8, weighting: int = WEIGHT_MULT):
    """Vanka-sweep output at DOFs `idx` of a level with N elements per side, computed
    from locally assembled element boxes (no global assembly; usable at 4096^2)."""
    lib = _load()
    x, b = _f64(x), _f64(b)
    idx = np.ascontiguousarray(idx, dtype=np.int64)
    out = np.zeros(len(idx))
    lib.orc_sweep_sample(N, nu, omega, weighting, _ptr(x), _ptr(b), _ptr(idx), len(idx), _ptr(out))
    return out


def residual_sample(N: int, x, b, idx, nu: float = 1.0):
    """(b - A x) at DOFs `idx` (0 on Dirichlet rows), from locally assembled boxes."""
    lib = _load()
    x, b = _f64(x), _f64(b)
    idx = np.ascontiguousarray(idx, dtype=np.int64)
    out = np.zeros(len(idx))
    lib.orc_residual_sample(N, nu, _ptr(x), _ptr(b), _ptr(idx), len(idx), _ptr(out))
    return out


def restrict_residual_sample(Nf: int, x, b, idx, nu: float = 1.0):
    """(P^T (b - A x)) at coarse DOFs `idx` (coarse level Nf/2, Dirichlet rows 0) of a
    fine level with Nf elements, from locally assembled boxes (usable at 4096^2)."""
    lib = _load()
    x, b = _f64(x), _f64(b)
    idx = np.ascontiguousarray(idx, dtype=np.int64)
    out = np.zeros(len(idx))
    lib.orc_restrict_residual_sample(Nf, nu, _ptr(x), _ptr(b), _ptr(idx), len(idx), _ptr(out))
    return out


def prolong_sample(Nf: int, ec, xf, idx):
    """(x_f + P e_c) at fine DOFs `idx` of a fine level with Nf elements."""
    lib = _load()
    ec, xf = _f64(ec), _f64(xf)
    idx = np.ascontiguousarray(idx, dtype=np.int64)
    out = np.zeros(len(idx))
    lib.orc_prolong_sample(Nf, _ptr(ec), _ptr(xf), _ptr(idx), len(idx), _ptr(out))
    return out


class Oracle:
    """Hierarchy N_fine, N_fine/2, ..., n_coarse assembled element by element."""

    def __init__(self, n_elem: int, n_coarse: int = 4, nu: float = 1.0, omega: float = 0.8,
                 weighting: int = WEIGHT_MULT, nu1: int = 1, nu2: int = 1, coarse_mode: int = 0):
        self._lib = _load()
        self._h = self._lib.orc_create(n_elem, n_coarse, nu, omega, weighting, nu1, nu2, coarse_mode)
        if not self._h:
            raise ValueError("oracle: bad configuration (N=%d, N0=%d)" % (n_elem, n_coarse))
        self.n_elem, self.n_coarse, self.nu, self.omega = n_elem, n_coarse, nu, omega
        self.levels = int(self._lib.orc_num_levels(self._h))

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            self._lib.orc_destroy(h)
            self._h = None

    # ---- sizes / layout -------------------------------------------------
    def N(self, level: int) -> int:
        return int(self._lib.orc_level_n(self._h, level))

    def length(self, level: int) -> int:
        return int(self._lib.orc_level_len(self._h, level))

    @property
    def fine(self) -> int:
        return self.levels - 1

    def split(self, v: np.ndarray, level: int):
        """(ux, uy, p) views shaped (2N+1, 2N+1), (2N+1, 2N+1), (N+1, N+1) [row = y]."""
        N = self.N(level)
        nl, nv = 2 * N + 1, (2 * N + 1) ** 2
        return (v[:nv].reshape(nl, nl), v[nv:2 * nv].reshape(nl, nl), v[2 * nv:].reshape(N + 1, N + 1))

    # ---- structure ------------------------------------------------------
    def csr(self, level: int):
        import scipy.sparse as sp
        n = self.length(level)
        nnz = int(self._lib.orc_nnz(self._h, level))
        rp = np.zeros(n + 1, np.int64)
        col = np.zeros(nnz, np.int32)
        val = np.zeros(nnz, np.float64)
        self._lib.orc_csr(self._h, level, _ptr(rp), _ptr(col), _ptr(val))
        return sp.csr_matrix((val, col, rp), shape=(n, n))

    def prolongation(self, level: int):
        import scipy.sparse as sp
        nf, nc = self.length(level), self.length(level - 1)
        nnz = int(self._lib.orc_prolongation_nnz(self._h, level))
        rp = np.zeros(nf + 1, np.int64)
        col = np.zeros(nnz, np.int32)
        val = np.zeros(nnz, np.float64)
        self._lib.orc_prolongation_csr(self._h, level, _ptr(rp), _ptr(col), _ptr(val))
        return sp.csr_matrix((val, col, rp), shape=(nf, nc))

    def dirichlet(self, level: int) -> np.ndarray:
        out = np.zeros(self.length(level), np.uint8)
        self._lib.orc_dirichlet(self._h, level, _ptr(out))
        return out.astype(bool)

    def weights(self, level: int) -> np.ndarray:
        out = np.zeros(self.length(level))
        self._lib.orc_weights(self._h, level, _ptr(out))
        return out

    def patch(self, level: int, kx: int, ky: int) -> np.ndarray:
        buf = np.zeros(64, np.int64)
        n = self._lib.orc_patch(self._h, level, kx, ky, _ptr(buf))
        return buf[:n].copy()

    def patch_group(self, level: int, kx: int, ky: int) -> int:
        return int(self._lib.orc_patch_group(self._h, level, kx, ky))

    def num_groups(self, level: int) -> int:
        return int(self._lib.orc_num_groups(self._h, level))

    def total_patch_dofs(self, level: int) -> int:
        return int(self._lib.orc_total_patch_dofs(self._h, level))

    # ---- problem data ---------------------------------------------------
    def problem(self, kind: int, level: int | None = None):
        level = self.fine if level is None else level
        n = self.length(level)
        b, x0 = np.zeros(n), np.zeros(n)
        self._lib.orc_problem(self._h, level, kind, _ptr(b), _ptr(x0))
        return b, x0

    def exact(self, kind: int, level: int | None = None) -> np.ndarray:
        level = self.fine if level is None else level
        out = np.zeros(self.length(level))
        self._lib.orc_exact(self._h, level, kind, _ptr(out))
        return out

    # ---- operations -----------------------------------------------------
    def matvec(self, level: int, x) -> np.ndarray:
        x = _f64(x)
        y = np.zeros_like(x)
        self._lib.orc_matvec(self._h, level, _ptr(x), _ptr(y))
        return y

    def residual(self, level: int, x, b) -> np.ndarray:
        x, b = _f64(x), _f64(b)
        r = np.zeros_like(x)
        self._lib.orc_residual(self._h, level, _ptr(x), _ptr(b), _ptr(r))
        return r

    def sweep(self, level: int, x, b, nsweeps: int = 1) -> np.ndarray:
        x, b = _f64(x).copy(), _f64(b)
        out = np.zeros_like(x)
        for _ in range(nsweeps):
            self._lib.orc_vanka_sweep(self._h, level, _ptr(x), _ptr(b), _ptr(out))
            x, out = out, x
        return x

    def set_relax(self, kind: int, t: float = 1.0, omega_r: float = 1.0, omega_j: float = 0.8, nj: int = 3):
        """V-cycle relaxation: RELAX_VANKA (alg:vk), RELAX_BS (inexact Braess-Sarazin,
        alg:bs; omega_r = omega_BS) or RELAX_SU (Schur-Uzawa, alg:uz; omega_r unused);
        t scales D = diag(L); omega_j, nj: weighted Jacobi on S = -(1/t) B D^-1 B^T."""
        if self._lib.orc_set_relax(self._h, kind, t, omega_r, omega_j, nj) != 0:
            raise ValueError("oracle: bad relaxation parameters")
        self.relax_kind = kind

    def relax_sweep(self, level: int, x, b) -> np.ndarray:
        """One sweep of the configured relaxation (Vanka by default)."""
        x, b = _f64(x), _f64(b)
        out = np.zeros_like(x)
        self._lib.orc_relax_sweep(self._h, level, _ptr(x), _ptr(b), _ptr(out))
        return out

    def schur(self, level: int):
        """S = -(1/t) B D^{-1} B^T on level `level` (after set_relax with BS or SU)."""
        import scipy.sparse as sp
        n = (self.N(level) + 1) ** 2
        nnz = int(self._lib.orc_schur_nnz(self._h, level))
        rp = np.zeros(n + 1, np.int64)
        col = np.zeros(nnz, np.int32)
        val = np.zeros(nnz, np.float64)
        self._lib.orc_schur_csr(self._h, level, _ptr(rp), _ptr(col), _ptr(val))
        return sp.csr_matrix((val, col, rp), shape=(n, n))

    def set_precond(self, kind: int, cycles: int = 3, nu: int = 3, omega_u: float = 1.0, omega_p: float = 0.6):
        """FGMRES preconditioner: PRECOND_MG (monolithic V-cycle) or PRECOND_BT (block-triangular,
        alg:bt: `cycles` V(nu,nu) cycles of weighted Jacobi on M (omega_p) then on L (omega_u))."""
        if self._lib.orc_set_precond(self._h, kind, cycles, nu, omega_u, omega_p) != 0:
            raise ValueError("oracle: bad preconditioner parameters")

    def precond_apply(self, r) -> np.ndarray:
        r = _f64(r)
        z = np.zeros_like(r)
        self._lib.orc_precond_apply(self._h, _ptr(r), _ptr(z))
        return z

    def mass(self, level: int):
        """Q1 pressure mass matrix (after set_precond(PRECOND_BT))."""
        import scipy.sparse as sp
        n = (self.N(level) + 1) ** 2
        nnz = int(self._lib.orc_mass_nnz(self._h, level))
        rp = np.zeros(n + 1, np.int64)
        col = np.zeros(nnz, np.int32)
        val = np.zeros(nnz, np.float64)
        self._lib.orc_mass_csr(self._h, level, _ptr(rp), _ptr(col), _ptr(val))
        return sp.csr_matrix((val, col, rp), shape=(n, n))

    def restrict(self, level: int, rf) -> np.ndarray:
        rf = _f64(rf)
        rc = np.zeros(self.length(level - 1))
        self._lib.orc_restrict(self._h, level, _ptr(rf), _ptr(rc))
        return rc

    def prolong_add(self, level: int, ec, xf) -> np.ndarray:
        ec, xf = _f64(ec), _f64(xf).copy()
        self._lib.orc_prolong_add(self._h, level, _ptr(ec), _ptr(xf))
        return xf

    def coarse_solve(self, b) -> np.ndarray:
        b = _f64(b)
        x = np.zeros_like(b)
        self._lib.orc_coarse_solve(self._h, _ptr(b), _ptr(x))
        return x

    def vcycle(self, b, x=None) -> np.ndarray:
        b = _f64(b)
        x = np.zeros_like(b) if x is None else _f64(x).copy()
        self._lib.orc_vcycle(self._h, _ptr(b), _ptr(x))
        return x

    def fgmres(self, b, x0, rtol: float = 1e-10, maxit: int = 200):
        """Returns (x, iterations, history[0..its], true_rel, status)."""
        b, x = _f64(b), _f64(x0).copy()
        hist = np.zeros(maxit + 1)
        tr = C.c_double(0.0)
        st = C.c_int(0)
        its = self._lib.orc_fgmres(self._h, _ptr(b), _ptr(x), rtol, maxit, _ptr(hist), C.byref(tr), C.byref(st))
        return x, int(its), hist[: its + 1].copy(), float(tr.value), int(st.value)
