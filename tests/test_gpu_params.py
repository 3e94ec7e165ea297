"""Parity away from the default parameters: viscosity nu != 1 (the stencils and the
patch factors scale with it: L = nu (M (x) K + K (x) M)), V(2,2) cycles
(alg:mg nu1 = nu2 = 2) and another Vanka weight, each against the oracle
built with the same parameters.  1e-12 relative as everywhere (north_star)."""
import numpy as np
from parity_util import rel
import pytest

import oracle
import svk_inputs

pytestmark = pytest.mark.gpu




@pytest.mark.parametrize("nu", [0.01, 7.5])
@pytest.mark.parametrize("N", [16, 64])
def test_viscosity_sweep_residual_vcycle(gpu, nu, N):
    from paper_2401_06277_b200 import Solver
    S, O = Solver(N, nu=nu), oracle.Oracle(N, nu=nu)
    l = S.fine
    x = svk_inputs.random_vector(N, 31)
    b = svk_inputs.random_vector(N, 32)
    rg = S.to_compact(S.residual(l, S.from_compact(x), S.from_compact(b))).cpu().numpy()
    assert rel(rg, O.residual(l, x, b)) < 1e-12
    xg = S.to_compact(S.sweep(l, S.from_compact(x), S.from_compact(b))).cpu().numpy()
    assert rel(xg - x, O.sweep(l, x, b) - x) < 1e-12
    bb = b.copy()
    bb[O.dirichlet(l)] = 0.0
    vg = S.to_compact(S.vcycle(S.from_compact(bb))).cpu().numpy()
    assert rel(vg, O.vcycle(bb)) < 1e-12


@pytest.mark.parametrize("N", [32, 128])
def test_v22_and_weight(gpu, N):
    from paper_2401_06277_b200 import Solver
    S = Solver(N, nu_pre=2, nu_post=2, omega=0.7)
    O = oracle.Oracle(N, nu1=2, nu2=2, omega=0.7)
    b = svk_inputs.random_vector(N, 41)
    b[O.dirichlet(O.fine)] = 0.0
    x0 = svk_inputs.random_vector(N, 42)
    vg = S.to_compact(S.vcycle(S.from_compact(b), S.from_compact(x0))).cpu().numpy()
    vo = O.vcycle(b, x0)
    assert rel(vg - x0, vo - x0) < 1e-12
    bg, xg0 = S.set_problem("mms_paper")
    rep, _ = S.fgmres(bg, xg0, rtol=1e-10, maxit=100)
    bo, x0o = O.problem(oracle.MMS_PAPER)
    its_o = O.fgmres(bo, x0o, rtol=1e-10, maxit=100)[1]
    assert abs(rep["iterations"] - its_o) <= 1, (rep["iterations"], its_o)


@pytest.mark.parametrize("N", [48, 96, 384])
def test_coarsest_six(gpu, N):
    """hierarchy with N0 = 6 (N = 6 * 2^k): 49 / 97 / 385 node columns, ragged against
    the strip width (60 node columns) and the chunking"""
    from paper_2401_06277_b200 import Solver
    S, O = Solver(N, n_coarse=6), oracle.Oracle(N, n_coarse=6)
    l = S.fine
    x = svk_inputs.random_vector(N, 51)
    b = svk_inputs.random_vector(N, 52)
    xg = S.to_compact(S.sweep(l, S.from_compact(x), S.from_compact(b))).cpu().numpy()
    assert rel(xg - x, O.sweep(l, x, b) - x) < 1e-12
    bb = b.copy()
    bb[O.dirichlet(l)] = 0.0
    vg = S.to_compact(S.vcycle(S.from_compact(bb))).cpu().numpy()
    assert rel(vg, O.vcycle(bb)) < 1e-12
    if N <= 96:
        bg, xg0 = S.set_problem("mms_paper")
        rep, _ = S.fgmres(bg, xg0, rtol=1e-10, maxit=100)
        bo, x0o = O.problem(oracle.MMS_PAPER)
        its_o = O.fgmres(bo, x0o, rtol=1e-10, maxit=100)[1]
        assert abs(rep["iterations"] - its_o) <= 1, (rep["iterations"], its_o)
