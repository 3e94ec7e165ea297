"""Parity of every libsvk call (through the C ABI) against the CPU oracle on the
same seeded inputs.  Tolerances follow BASELINE.json north_star: 1e-12 relative
(in the 2-norm of the correction) per sweep / residual / transfer / V-cycle,
FGMRES iteration counts within +-1.  Sizes span several tiles and ragged tails
(N+1 = 17, 65, 129, 257 node columns vs the kernels' strip widths).
"""
import numpy as np
from parity_util import rel
import pytest

import oracle
import svk_inputs

pytestmark = pytest.mark.gpu

IMPLS = ["fused", "unfused", "simple"]  # simple: per-patch stored inverses (NEXT-3)




_orc = {}
_gpu = {}


def get_oracle(N, **kw):
    key = (N, tuple(sorted(kw.items())))
    if key not in _orc:
        _orc[key] = oracle.Oracle(N, **kw)
    return _orc[key]


def get_solver(N, **kw):
    from paper_2401_06277_b200 import Solver
    key = (N, tuple(sorted(kw.items())))
    if key not in _gpu:
        _gpu[key] = Solver(N, **kw)
    return _gpu[key]


def to_np(S, v, level):
    return S.to_compact(v, level).cpu().numpy()


@pytest.mark.parametrize("N", [8, 16, 64, 256])
def test_set_problem_parity(gpu, N):
    S, O = get_solver(N), get_oracle(N)
    for kind, name in [(oracle.MMS_PAPER, "mms_paper"), (oracle.MMS_INSPACE, "mms_inspace"), (oracle.CAVITY, "cavity")]:
        b, x0 = S.set_problem(name)
        bo, x0o = O.problem(kind)
        assert rel(to_np(S, b, S.fine), bo) < 1e-13
        assert rel(to_np(S, x0, S.fine), x0o) < 1e-14 or np.linalg.norm(x0o) == 0


@pytest.mark.parametrize("N", [4, 16, 64, 256])
def test_residual_and_matvec_parity(gpu, N):
    S, O = get_solver(N), get_oracle(N)
    for l in range(S.levels):
        n = S.info[l].N
        for seed in (1, 2):
            x = svk_inputs.random_vector(n, seed)
            b = svk_inputs.random_vector(n, seed + 50)
            r = S.residual(l, S.from_compact(x, l), S.from_compact(b, l))
            assert rel(to_np(S, r, l), O.residual(l, x, b)) < 1e-13
            y = S.matvec(l, S.from_compact(x, l))
            assert rel(to_np(S, y, l), O.matvec(l, x)) < 1e-13


@pytest.mark.parametrize("impl", IMPLS)
@pytest.mark.parametrize("N", [4, 8, 16, 64, 256])
def test_sweep_parity(gpu, impl, N):
    S, O = get_solver(N, sweep=impl), get_oracle(N)
    for l in range(S.levels):
        n = S.info[l].N
        for seed in (1, 2, 3):
            x = svk_inputs.random_vector(n, seed)
            b = svk_inputs.random_vector(n, seed + 10)
            xo = O.sweep(l, x, b)
            xg = to_np(S, S.sweep(l, S.from_compact(x, l), S.from_compact(b, l)), l)
            assert rel(xg - x, xo - x) < 1e-12, (l, seed)


@pytest.mark.parametrize("impl", IMPLS)
def test_multi_sweep_and_weighting_modes(gpu, impl):
    N = 32
    for weighting, wcode in (("mult", oracle.WEIGHT_MULT), ("scalar", oracle.WEIGHT_SCALAR)):
        S = get_solver(N, sweep=impl, weighting=weighting, omega=0.6)
        O = get_oracle(N, weighting=wcode, omega=0.6)
        x = svk_inputs.random_vector(N, 7)
        b = svk_inputs.random_vector(N, 8)
        for ns in (1, 2, 3):
            xo = O.sweep(S.fine, x, b, nsweeps=ns)
            xg = to_np(S, S.sweep(S.fine, S.from_compact(x), S.from_compact(b), nsweeps=ns), S.fine)
            assert rel(xg - x, xo - x) < 1e-12, (weighting, ns)


@pytest.mark.parametrize("N", [16, 64, 256])
def test_transfer_parity(gpu, N):
    S, O = get_solver(N), get_oracle(N)
    for l in range(1, S.levels):
        nf, nc = S.info[l].N, S.info[l - 1].N
        rf = svk_inputs.random_vector(nf, 3)
        rc = to_np(S, S.restrict(l, S.from_compact(rf, l)), l - 1)
        assert rel(rc, O.restrict(l, rf)) < 1e-13
        ec = svk_inputs.random_vector(nc, 4)
        ec[O.dirichlet(l - 1)] = 0.0
        xf = svk_inputs.random_vector(nf, 5)
        out = to_np(S, S.prolong_add(l, S.from_compact(ec, l - 1), S.from_compact(xf, l)), l)
        ref = O.prolong_add(l, ec, xf)
        assert rel(out - xf, ref - xf) < 1e-13


@pytest.mark.parametrize("N", [16, 64, 256])
def test_residual_restrict_parity(gpu, N):
    """The V-cycle's fused residual + restriction (svk_residual_restrict) on every
    level against the oracle's explicit P^T (b - A x)."""
    S, O = get_solver(N), get_oracle(N)
    for l in range(1, S.levels):
        n = S.info[l].N
        x = svk_inputs.random_vector(n, 41)
        b = svk_inputs.random_vector(n, 42)
        rc = to_np(S, S.residual_restrict(l, S.from_compact(x, l), S.from_compact(b, l)), l - 1)
        assert rel(rc, O.restrict(l, O.residual(l, x, b))) < 1e-13, l


def test_coarse_solve_parity(gpu):
    S, O = get_solver(16), get_oracle(16)
    for seed in (1, 2, 3):
        b = svk_inputs.random_vector(4, seed)
        b[O.dirichlet(0)] = 0.0
        xg = to_np(S, S.coarse_solve(S.from_compact(b, 0)), 0)
        assert rel(xg, O.coarse_solve(b)) < 1e-12


def test_patch_inverses_match_oracle_patch_matrices(gpu):
    N = 16
    S, O = get_solver(N), get_oracle(N)
    A = O.csr(O.fine).toarray()
    rep = {0: 0, 1: 1, 2: 2, 3: N - 1, 4: N}
    for cy in range(5):
        for cx in range(5):
            p = O.patch(O.fine, rep[cx], rep[cy])  # oracle order: u_x window, u_y window, p (same as the ABI's)
            Ai = A[np.ix_(p, p)]
            inv = S.patch_inverse(S.fine, cx, cy)
            assert inv.shape == Ai.shape
            assert np.abs(inv @ Ai - np.eye(len(p))).max() < 1e-10


@pytest.mark.parametrize("impl", IMPLS)
@pytest.mark.parametrize("N", [8, 16, 64, 256])
def test_vcycle_parity(gpu, impl, N):
    S, O = get_solver(N, sweep=impl), get_oracle(N)
    for seed in (1, 2):
        b = svk_inputs.random_vector(N, seed)
        b[O.dirichlet(O.fine)] = 0.0
        xo = O.vcycle(b)
        xg = to_np(S, S.vcycle(S.from_compact(b)), S.fine)
        assert rel(xg, xo) < 1e-12
        x0 = svk_inputs.random_vector(N, seed + 20)
        xo = O.vcycle(b, x0)
        xg = to_np(S, S.vcycle(S.from_compact(b), S.from_compact(x0)), S.fine)
        assert rel(xg - x0, xo - x0) < 1e-12


def test_vcycle_coarse_sweeps3_parity(gpu):
    N = 32
    S = get_solver(N, coarse="sweeps3")
    O = get_oracle(N, coarse_mode=1)
    b = svk_inputs.random_vector(N, 9)
    b[O.dirichlet(O.fine)] = 0.0
    assert rel(to_np(S, S.vcycle(S.from_compact(b)), S.fine), O.vcycle(b)) < 1e-12


@pytest.mark.parametrize("impl", IMPLS)
@pytest.mark.parametrize("N,kind", [(16, "mms_paper"), (64, "mms_paper"), (128, "cavity"), (256, "mms_paper")])
def test_fgmres_iterations_and_solution(gpu, impl, N, kind):
    S, O = get_solver(N, sweep=impl), get_oracle(N)
    kcode = {"mms_paper": oracle.MMS_PAPER, "cavity": oracle.CAVITY}[kind]
    b, x0 = S.set_problem(kind)
    rep, hist = S.fgmres(b, x0, rtol=1e-10, maxit=100)
    bo, x0o = O.problem(kcode)
    xo, its, ho, tro, st = O.fgmres(bo, x0o, rtol=1e-10, maxit=100)
    assert rep["converged"] == 1 and st == 0
    assert abs(rep["iterations"] - its) <= 1
    assert rep["rel_residual"] < 1e-9
    xg = to_np(S, x0, S.fine)
    ux, uy, p = O.split(xg, O.fine)
    oux, ouy, op = O.split(xo, O.fine)
    scale = max(np.abs(oux).max(), np.abs(ouy).max(), 1e-30)
    assert np.abs(ux - oux).max() < 1e-8 * scale + 1e-12
    assert np.abs(uy - ouy).max() < 1e-8 * scale + 1e-12
    assert np.abs((p - p.mean()) - (op - op.mean())).max() < 1e-6 * max(np.abs(op).max(), 1.0)
    # history agrees while well above roundoff
    k = min(len(hist), len(ho))
    m = ho[:k] > 1e-6
    assert np.all(np.abs(hist[:k][m] - ho[:k][m]) <= 1e-6 * ho[:k][m])


@pytest.mark.parametrize("N,kind", [(64, "mms_paper"), (256, "cavity")])
def test_fgmres_orth_modes(gpu, N, kind):
    """ADAPTIVE (one Gram-Schmidt pass unless it cancels; reading 18) and CGS2
    reach the oracle's (MGS) iteration count and solution."""
    O = get_oracle(N)
    kcode = {"mms_paper": oracle.MMS_PAPER, "cavity": oracle.CAVITY}[kind]
    bo, x0o = O.problem(kcode)
    xo, its, ho, _, _ = O.fgmres(bo, x0o, rtol=1e-10, maxit=100)
    hists = {}
    for orth in ("adaptive", "cgs2"):
        S = get_solver(N, orth=orth)
        b, x = S.set_problem(kind)
        rep, hist = S.fgmres(b, x, rtol=1e-10, maxit=100)
        assert rep["converged"] == 1 and abs(rep["iterations"] - its) <= 1
        if orth == "cgs2":
            assert rep["n_reorth"] == rep["iterations"]
        else:
            assert 0 <= rep["n_reorth"] <= rep["iterations"]
        xg = to_np(S, x, S.fine)
        nv = (2 * N + 1) ** 2
        assert np.abs(xg[:2 * nv] - xo[:2 * nv]).max() < 1e-8 * max(np.abs(xo[:2 * nv]).max(), 1.0)
        k = min(len(hist), len(ho))
        m = ho[:k] > 1e-6
        assert np.all(np.abs(hist[:k][m] - ho[:k][m]) <= 1e-6 * ho[:k][m])
        hists[orth] = hist


@pytest.mark.parametrize("N", [64, 512])
def test_mms_nodal_exactness_gpu(gpu, N):
    """Closed-form pin at any size: the converged solution equals the paper's
    manufactured solution at every DOF point."""
    S = get_solver(N)
    b, x = S.set_problem("mms_paper")
    rep, _ = S.fgmres(b, x, rtol=1e-11, maxit=100)
    assert rep["converged"] == 1
    O = oracle.Oracle(4)  # exact nodal values come from the closed form only
    nl = 2 * N + 1
    xs = np.arange(nl) / (2 * N)
    X, Y = np.meshgrid(xs, xs)
    eux = X * (1 - X) * (2 * X - 1) * (6 * Y ** 2 - 6 * Y + 1)
    euy = Y * (Y - 1) * (2 * Y - 1) * (6 * X ** 2 - 6 * X + 1)
    ps = np.arange(N + 1) / N
    PX, PY = np.meshgrid(ps, ps)
    ep = PX ** 2 - 3 * PY ** 2 + 8.0 / 3.0 * PX * PY
    ux, uy, p = [t.cpu().numpy() for t in S.planes(x)]
    assert np.abs(ux - eux).max() < 1e-9
    assert np.abs(uy - euy).max() < 1e-9
    assert np.abs((p - p.mean()) - (ep - ep.mean())).max() < 1e-6
    del O


def test_solve_host_e2e(gpu):
    N = 64
    S, O = get_solver(N), get_oracle(N)
    bo, x0o = O.problem(oracle.MMS_PAPER)
    x, rep = S.solve_host(bo, x0o, rtol=1e-10, maxit=100)
    xo, its, _, _, _ = O.fgmres(bo, x0o)
    assert abs(rep["iterations"] - its) <= 1 and rep["converged"] == 1
    ux, uy, p = O.split(x, O.fine)
    oux, ouy, op = O.split(xo, O.fine)
    assert np.abs(ux - oux).max() < 1e-8


def test_errors_are_loud(gpu):
    from paper_2401_06277_b200 import SvkError
    S = get_solver(16)
    x = S.new_vector()
    with pytest.raises(SvkError):
        S.sweep(S.fine, x, x, out=x)                 # aliasing
    with pytest.raises(SvkError):
        S.residual(S.fine, x[:-1].clone(), x)        # wrong length
    with pytest.raises(SvkError):
        S.restrict(0, S.new_vector(0))               # no coarser level


def test_host_arrays_and_arguments_are_checked(gpu):
    """svk_solve_host reads / writes 2(2N+1)^2+(N+1)^2 doubles: the binding rejects
    short, wrongly typed, non-contiguous or read-only arrays, and the C entry point
    itself rejects maxit < 1, a NaN rtol and an aliased output."""
    import ctypes as C
    from paper_2401_06277_b200 import SvkError
    from paper_2401_06277_b200.svk import Report
    N = 16
    S = get_solver(N)
    n = 2 * (2 * N + 1) ** 2 + (N + 1) ** 2
    ok = np.zeros(n)
    for bad in (np.zeros(n - 1), np.zeros(n, np.float32), np.zeros(2 * n)[::2]):
        with pytest.raises(SvkError):
            S.solve_host(bad, ok)
        with pytest.raises(SvkError):
            S.solve_host(ok, bad)
    ro = np.zeros(n)
    ro.flags.writeable = False
    with pytest.raises(SvkError):
        S.solve_host(ok, ok, x_host=ro)
    with pytest.raises(SvkError):
        S.solve_host(ok, ok.copy(), x_host=ok)
    p = ok.ctypes.data_as(C.c_void_p)
    out = np.zeros(n)
    q = out.ctypes.data_as(C.c_void_p)
    rep = Report()
    for rtol, maxit in ((1e-10, 0), (1e-10, -5), (float("nan"), 10), (-1.0, 10)):
        assert S.lib.svk_solve_host(S._h, p, p, q, rtol, maxit, C.byref(rep), None) < 0
    assert S.lib.svk_solve_host(S._h, p, p, p, 1e-10, 10, C.byref(rep), None) < 0


@pytest.mark.parametrize("N,kind", [(64, "mms_paper"), (256, "cavity")])
def test_low_memory_krylov_matches_fgmres(gpu, N, kind):
    """krylov_store_z = 0 (right-preconditioned GMRES with the fixed V-cycle, one
    z buffer, x = x0 + M sum y_j V_j): the same iterates as FGMRES up to rounding,
    so the oracle's iteration count and solution, with half the Krylov memory."""
    from paper_2401_06277_b200 import Solver
    O = get_oracle(N)
    kcode = {"mms_paper": oracle.MMS_PAPER, "cavity": oracle.CAVITY}[kind]
    bo, x0o = O.problem(kcode)
    xo, its, ho, _, _ = O.fgmres(bo, x0o, rtol=1e-10, maxit=100)
    out = {}
    for low in (False, True):
        S = Solver(N, low_memory=low)
        b, x = S.set_problem(kind)
        rep, hist = S.fgmres(b, x, rtol=1e-10, maxit=100)
        out[low] = (rep, hist, to_np(S, x, S.fine), S.device_bytes)
        S.close()
    (r0, h0, x0g, m0), (r1, h1, x1g, m1) = out[False], out[True]
    assert r1["converged"] == 1 and r1["iterations"] == r0["iterations"] and abs(r1["iterations"] - its) <= 1
    assert np.all(np.abs(h1 - h0) <= 1e-9 * np.maximum(h0, 1e-12))
    assert r1["rel_residual"] < 1e-9
    nv = (2 * N + 1) ** 2
    scale = max(np.abs(xo[:2 * nv]).max(), 1.0)
    assert np.abs(x1g[:2 * nv] - xo[:2 * nv]).max() < 1e-8 * scale
    assert np.abs(x1g[:2 * nv] - x0g[:2 * nv]).max() < 1e-9 * scale
    assert m1 < m0


def test_degenerate_cases_single_level_and_zero_rhs(gpu):
    """As the oracle pin: N = N0 (one level: the V-cycle is the exact min-norm solve)
    converges in one FGMRES iteration to the oracle's solution; b = 0, x0 = 0 needs
    none and returns x = 0."""
    from paper_2401_06277_b200 import Solver
    S, O = Solver(4, n_coarse=4), oracle.Oracle(4, n_coarse=4)
    b, x = S.set_problem("mms_paper")
    rep, hist = S.fgmres(b, x, rtol=1e-10, maxit=10)
    bo, x0o = O.problem(oracle.MMS_PAPER)
    xo, its, _, _, _ = O.fgmres(bo, x0o, rtol=1e-10, maxit=10)
    assert rep["converged"] == 1 and rep["iterations"] == its == 1
    xg = to_np(S, x, S.fine)
    nv = 9 * 9
    assert np.abs(xg[:2 * nv] - xo[:2 * nv]).max() < 1e-12
    z = S.new_vector()
    xz = S.new_vector()
    rep, hist = S.fgmres(z, xz, rtol=1e-10, maxit=10)
    assert rep["converged"] == 1 and rep["iterations"] == 0 and float(xz.abs().max()) == 0.0


def test_not_converged_is_reported_and_matches_oracle_history(gpu):
    """maxit below the needed count: SVK_NOT_CONVERGED (status 1, non-fatal), the
    report filled, and the truncated residual history equal to the oracle's."""
    N = 64
    S, O = get_solver(N), get_oracle(N)
    b, x = S.set_problem("mms_paper")
    rep, hist = S.fgmres(b, x, rtol=1e-10, maxit=5)
    assert rep["status"] == 1 and rep["converged"] == 0 and rep["iterations"] == 5 and len(hist) == 6
    bo, x0o = O.problem(oracle.MMS_PAPER)
    xo, its, ho, tro, st = O.fgmres(bo, x0o, rtol=1e-10, maxit=5)
    assert st == 1 and its == 5
    assert np.all(np.abs(hist - ho) <= 1e-9 * ho)
    assert abs(rep["rel_residual"] - tro) <= 1e-8 * tro
