"""GPU parity of the comparator relaxations: inexact
Braess-Sarazin (alg:bs) and Schur-Uzawa (alg:uz) through the C ABI
(svk_relax_sweep, svk_vcycle, svk_fgmres) against the CPU oracle on the same
seeded inputs.  Tolerances as for Vanka: 1e-12 relative in the 2-norm of the
correction per sweep / V-cycle, FGMRES iterations within +-1.  Sizes span every
level of the hierarchy (N = 4 ... 256), i.e. the tiny-level S classes, the seven
boundary-distance classes per axis and ragged CUDA blocks."""
import numpy as np
from parity_util import rel
import pytest

import oracle
import svk_inputs

pytestmark = pytest.mark.gpu

KINDS = {"bs": (oracle.RELAX_BS, dict(t=1.0, omega_r=1.0, omega_j=0.8, nj=3)),
         "su": (oracle.RELAX_SU, dict(t=1.0, omega_j=0.4, nj=1))}




def make(N, kind, **over):
    from paper_2401_06277_b200 import Solver
    k, kw = KINDS[kind]
    kw = dict(kw, **over)
    O = oracle.Oracle(N)
    O.set_relax(k, **kw)
    S = Solver(N, relax=kind, relax_t=kw["t"], relax_omega=kw.get("omega_r", 1.0), jacobi_omega=kw["omega_j"],
               jacobi_sweeps=kw["nj"])
    return S, O


def to_np(S, v, level):
    return S.to_compact(v, level).cpu().numpy()


@pytest.mark.parametrize("kind", ["bs", "su"])
@pytest.mark.parametrize("N", [8, 16, 64, 256])
def test_relax_sweep_parity(gpu, kind, N):
    S, O = make(N, kind)
    for l in range(S.levels):
        n = S.info[l].N
        for seed in (1, 2):
            x = svk_inputs.random_vector(n, seed)
            b = svk_inputs.random_vector(n, seed + 30)
            xo = O.relax_sweep(l, x, b)
            xg = to_np(S, S.relax_sweep(l, S.from_compact(x, l), S.from_compact(b, l)), l)
            assert rel(xg - x, xo - x) < 1e-12, (kind, N, l, seed)


@pytest.mark.parametrize("kind", ["bs", "su"])
def test_relax_parameters_parity(gpu, kind):
    """t, omega_BS, the Jacobi weight and sweep count (including 0 sweeps) reach the kernels."""
    for over in (dict(t=1.7, omega_j=0.6, nj=5), dict(t=0.5, nj=0), dict(nj=2, omega_r=0.7)):
        if kind == "su":
            over.pop("omega_r", None)
        S, O = make(16, kind, **over)
        x = svk_inputs.random_vector(16, 3)
        b = svk_inputs.random_vector(16, 4)
        xo = O.relax_sweep(O.fine, x, b)
        xg = to_np(S, S.relax_sweep(S.fine, S.from_compact(x), S.from_compact(b)), S.fine)
        assert rel(xg - x, xo - x) < 1e-12, over


@pytest.mark.parametrize("kind", ["bs", "su"])
@pytest.mark.parametrize("N", [16, 64])
def test_vcycle_parity(gpu, kind, N):
    S, O = make(N, kind)
    b = svk_inputs.random_vector(N, 9)
    b[O.dirichlet(O.fine)] = 0.0
    xo = O.vcycle(b)
    xg = to_np(S, S.vcycle(S.from_compact(b)), S.fine)
    assert rel(xg, xo) < 1e-12


@pytest.mark.parametrize("kind,N", [("bs", 16), ("bs", 64), ("su", 16), ("su", 64), ("su", 128)])
def test_fgmres_iterations(gpu, kind, N):
    """SU at 128^2 needs 72 iterations: also the regression test of FGMRES beyond 64
    basis vectors (the coefficient-scaling launch once covered only 64)."""
    S, O = make(N, kind)
    bg, x0 = S.set_problem("mms_paper")
    rep, _ = S.fgmres(bg, x0, rtol=1e-10, maxit=300)
    bo, x0o = O.problem(oracle.MMS_PAPER)
    _, its, _, _, st = O.fgmres(bo, x0o, rtol=1e-10, maxit=300)
    assert st == 0 and rep["converged"] == 1
    assert abs(rep["iterations"] - its) <= 1, (rep["iterations"], its)
    ex = O.exact(oracle.MMS_PAPER)
    nv = (2 * N + 1) ** 2
    assert np.abs(to_np(S, x0, S.fine)[: 2 * nv] - ex[: 2 * nv]).max() < 1e-8


def test_vanka_sweep_unchanged_by_relax_choice(gpu):
    """svk_vanka_sweep stays the Vanka sweep whatever svk_config.relax says."""
    S, _ = make(16, "bs")
    O = oracle.Oracle(16)
    x = svk_inputs.random_vector(16, 5)
    b = svk_inputs.random_vector(16, 6)
    xg = to_np(S, S.sweep(S.fine, S.from_compact(x), S.from_compact(b)), S.fine)
    assert rel(xg - x, O.sweep(O.fine, x, b) - x) < 1e-12


def test_comparators_single_gpu_only(gpu):
    from paper_2401_06277_b200 import Solver, SvkError
    with pytest.raises(SvkError):
        Solver(64, rank=0, nranks=2, transport="emulated", relax="bs")


# --------------------------------------------- block-triangular preconditioner (alg:bt)
@pytest.mark.parametrize("N", [8, 16, 64, 256])
def test_bt_precond_apply_parity(gpu, N):
    from paper_2401_06277_b200 import Solver
    O = oracle.Oracle(N)
    O.set_precond(oracle.PRECOND_BT)
    S = Solver(N, precond="bt")
    for seed in (1, 2):
        r = svk_inputs.random_vector(N, seed)
        r[O.dirichlet(O.fine)] = 0.0
        zo = O.precond_apply(r)
        zg = to_np(S, S.precond_apply(S.from_compact(r)), S.fine)
        assert rel(zg, zo) < 1e-12, (N, seed)


def test_bt_parameters_parity(gpu):
    from paper_2401_06277_b200 import Solver
    O = oracle.Oracle(32)
    O.set_precond(oracle.PRECOND_BT, cycles=2, nu=1, omega_u=0.7, omega_p=0.5)
    S = Solver(32, precond="bt", bt_cycles=2, bt_nu=1, bt_omega_u=0.7, bt_omega_p=0.5)
    r = svk_inputs.random_vector(32, 3)
    r[O.dirichlet(O.fine)] = 0.0
    assert rel(to_np(S, S.precond_apply(S.from_compact(r)), S.fine), O.precond_apply(r)) < 1e-12


@pytest.mark.parametrize("N", [16, 64])
def test_bt_fgmres_iterations(gpu, N):
    from paper_2401_06277_b200 import Solver
    O = oracle.Oracle(N)
    O.set_precond(oracle.PRECOND_BT)
    S = Solver(N, precond="bt")
    bg, x0 = S.set_problem("mms_paper")
    rep, _ = S.fgmres(bg, x0, rtol=1e-10, maxit=200)
    bo, x0o = O.problem(oracle.MMS_PAPER)
    _, its, _, _, st = O.fgmres(bo, x0o, rtol=1e-10, maxit=200)
    assert st == 0 and rep["converged"] == 1
    assert abs(rep["iterations"] - its) <= 1, (rep["iterations"], its)


def test_precond_apply_mg_is_vcycle(gpu):
    from paper_2401_06277_b200 import Solver
    S = Solver(16)
    O = oracle.Oracle(16)
    r = svk_inputs.random_vector(16, 4)
    r[O.dirichlet(O.fine)] = 0.0
    assert rel(to_np(S, S.precond_apply(S.from_compact(r)), S.fine), O.vcycle(r)) < 1e-12
