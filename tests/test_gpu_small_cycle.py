"""The V-cycle's coarse levels in one cluster launch (csrc/small_cycle.cuh) against
the per-kernel recursion (SVK_SMALL_N=0) and the oracle: same alg:mg steps,
the same operators, so the two agree to rounding; the one-launch form replaces the
13 launches of the levels <= 16^2."""
import os

import numpy as np
import pytest

import oracle
import svk_inputs
from parity_util import rel

pytestmark = pytest.mark.gpu


def _solver(N, small, **kw):
    from paper_2401_06277_b200 import Solver
    old = os.environ.get("SVK_SMALL_N")
    os.environ["SVK_SMALL_N"] = str(small)
    try:
        return Solver(N, **kw)
    finally:
        if old is None:
            del os.environ["SVK_SMALL_N"]
        else:
            os.environ["SVK_SMALL_N"] = old


@pytest.mark.parametrize("N", [32, 64])
@pytest.mark.parametrize("kw,okw", [({}, {}), ({"coarse": "sweeps3"}, {"coarse_mode": 1}),
                                     ({"weighting": "scalar", "omega": 0.15},
                                      {"weighting": oracle.WEIGHT_SCALAR, "omega": 0.15})])
def test_small_cycle_matches_per_kernel_recursion_and_oracle(gpu, N, kw, okw):
    import torch
    A, B = _solver(N, 16, **kw), _solver(N, 0, **kw)
    O = oracle.Oracle(N, **okw)
    b = svk_inputs.random_vector(N, 7)
    b[O.dirichlet(O.fine)] = 0.0
    za = A.to_compact(A.vcycle(A.from_compact(b))).cpu().numpy()
    zb = B.to_compact(B.vcycle(B.from_compact(b))).cpu().numpy()
    zo = O.vcycle(b)
    assert rel(za, zb) <= 1e-13
    assert rel(za, zo) <= 1e-12
    # the levels <= 16^2 (3 of them) run in one launch instead of 13
    n0 = A.launch_count
    A.vcycle(A.from_compact(b))
    torch.cuda.synchronize()
    la = A.launch_count - n0
    n0 = B.launch_count
    B.vcycle(B.from_compact(b))
    torch.cuda.synchronize()
    lb = B.launch_count - n0
    assert la < lb


def test_small_cycle_fgmres_iterations(gpu):
    A, B = _solver(128, 16), _solver(128, 0)
    for S in (A, B):
        bb, x0 = S.set_problem("mms_paper")
        rep, _ = S.fgmres(bb, x0, rtol=1e-10, maxit=60)
        S.its = rep["iterations"]
    assert abs(A.its - B.its) <= 1


def test_small_cycle_launch_failure_falls_back(gpu):
    # a cluster size the device cannot launch (32 > 16): the first launch fails, the
    # context switches to the per-kernel recursion, results unchanged
    old = os.environ.get("SVK_SMALL_CLUSTER")
    os.environ["SVK_SMALL_CLUSTER"] = "32"
    try:
        A = _solver(64, 16)
    finally:
        if old is None:
            del os.environ["SVK_SMALL_CLUSTER"]
        else:
            os.environ["SVK_SMALL_CLUSTER"] = old
    B = _solver(64, 0)
    O = oracle.Oracle(64)
    b = svk_inputs.random_vector(64, 11)
    b[O.dirichlet(O.fine)] = 0.0
    za = A.to_compact(A.vcycle(A.from_compact(b))).cpu().numpy()
    zb = B.to_compact(B.vcycle(B.from_compact(b))).cpu().numpy()
    assert np.array_equal(za, zb)


@pytest.mark.parametrize("nu", [(0, 1), (1, 0), (3, 1)])
def test_small_cycle_smoothing_counts(gpu, nu):
    # V(nu1, nu2) with the coarse levels in one launch, against the per-kernel path
    # and the oracle (alg:mg with nu1 pre- and nu2 post-smoothing sweeps)
    N = 64
    A = _solver(N, 16, nu_pre=nu[0], nu_post=nu[1])
    B = _solver(N, 0, nu_pre=nu[0], nu_post=nu[1])
    O = oracle.Oracle(N, nu1=nu[0], nu2=nu[1])
    b = svk_inputs.random_vector(N, 13)
    b[O.dirichlet(O.fine)] = 0.0
    za = A.to_compact(A.vcycle(A.from_compact(b))).cpu().numpy()
    zb = B.to_compact(B.vcycle(B.from_compact(b))).cpu().numpy()
    assert rel(za, zb) <= 1e-13
    assert rel(za, O.vcycle(b)) <= 1e-12
