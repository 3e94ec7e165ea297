"""Parity at BASELINE.json's full size (4096^2, configs[2]) in the launch
configuration bench.py times (fused sweep, default hierarchy): sampled outputs
the oracle computes one by one from locally assembled element boxes
(oracle.sweep_sample / residual_sample), plus the closed-form nodal exactness
of the converged FGMRES solution, which holds at any size."""
import json
import os

import numpy as np
import pytest

import oracle
import svk_inputs

pytestmark = pytest.mark.gpu

N = 4096


@pytest.fixture(scope="module")
def solver(gpu):
    from paper_2401_06277_b200 import Solver
    return Solver(N)


def structured_samples(Nn):
    """DOFs at the places a tiled kernel gets wrong: domain edges, strip edges (60-node
    strips of 2-warp CTAs, 120-node strips of 4-warp ones), chunk rows (64-69 node
    rows per CTA at this size), plus pressure nodes there."""
    lat = 2 * Nn + 1
    nv = lat * lat
    node_cols = [0, 1, 2, Nn - 2, Nn - 1, Nn] + [c + d for c in (60, 120, 240, 1200) for d in (-2, -1, 0, 1, 2)]
    node_rows = [0, 1, 2, Nn - 2, Nn - 1, Nn] + [r + d for r in (64, 69, 128, 138, 2000) for d in (-1, 0, 1)]
    cols = sorted({i for k in node_cols for i in (2 * k - 1, 2 * k, 2 * k + 1) if 1 <= i <= lat - 2})
    rows = sorted({j for k in node_rows for j in (2 * k - 1, 2 * k, 2 * k + 1) if 1 <= j <= lat - 2})
    out = []
    for j in rows:
        for i in cols:
            out += [j * lat + i, nv + j * lat + i]
    for ky in node_rows:
        for kx in node_cols:
            out.append(2 * nv + ky * (Nn + 1) + kx)
    return np.array(sorted(set(out)), dtype=np.int64)


def test_fullsize_sweep_and_residual_sampled(solver):
    S = solver
    x = svk_inputs.random_vector(N, 101)
    b = svk_inputs.random_vector(N, 102)
    xd, bd = S.from_compact(x), S.from_compact(b)
    xg = S.to_compact(S.sweep(S.fine, xd, bd)).cpu().numpy()
    rg = S.to_compact(S.residual(S.fine, xd, bd)).cpu().numpy()
    idx = np.union1d(svk_inputs.random_sample_indices(N, 103, 400), structured_samples(N))
    xo = oracle.sweep_sample(N, x, b, idx)
    ro = oracle.residual_sample(N, x, b, idx)
    d_g, d_o = xg[idx] - x[idx], xo - x[idx]
    assert np.abs(d_g - d_o).max() <= 1e-12 * np.abs(d_o).max()
    assert np.abs(rg[idx] - ro).max() <= 1e-13 * np.abs(ro).max()


def test_fullsize_residual_restrict_and_prolong_sampled(solver):
    """The transfer kernels at 4096^2 in the V-cycle's launch configuration:
    r_c = P^T (b - A x) (fused residual + restriction) sampled on the 2048^2
    level, and x_f + P e_c sampled on the fine level, against the oracle's local
    samplers (oracle.restrict_residual_sample / prolong_sample)."""
    S = solver
    Nc = N // 2
    x = svk_inputs.random_vector(N, 111)
    b = svk_inputs.random_vector(N, 112)
    rc = S.to_compact(S.residual_restrict(S.fine, S.from_compact(x), S.from_compact(b)), S.fine - 1).cpu().numpy()
    idxc = np.union1d(svk_inputs.random_sample_indices(Nc, 113, 400), structured_samples(Nc))
    ro = oracle.restrict_residual_sample(N, x, b, idxc)
    assert np.abs(rc[idxc] - ro).max() <= 1e-12 * np.abs(ro).max()
    del rc
    ec = svk_inputs.random_vector(Nc, 114)
    latc = 2 * Nc + 1
    for comp in range(2):  # coarse Dirichlet entries of a correction are 0
        pl = ec[comp * latc * latc:(comp + 1) * latc * latc].reshape(latc, latc)
        pl[0, :] = pl[-1, :] = pl[:, 0] = pl[:, -1] = 0.0
    xg = S.to_compact(S.prolong_add(S.fine, S.from_compact(ec, S.fine - 1), S.from_compact(x)), S.fine).cpu().numpy()
    idx = np.union1d(svk_inputs.random_sample_indices(N, 115, 400), structured_samples(N))
    po = oracle.prolong_sample(N, ec, x, idx)
    d_g, d_o = xg[idx] - x[idx], po - x[idx]
    assert np.abs(d_g - d_o).max() <= 1e-13 * np.abs(d_o).max()


def test_fullsize_mms_nodal_exactness(solver):
    S = solver
    b, x = S.set_problem("mms_paper")
    rep, hist = S.fgmres(b, x, rtol=1e-10, maxit=60)
    # the oracle's own 4096^2 solve (tests/golden/oracle_iterations_large.json: 19 iterations)
    gold = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "oracle_iterations_large.json")))
    assert rep["converged"] == 1 and abs(rep["iterations"] - gold["fgmres_iterations"]["mms_paper_4096"]) <= 1
    ux, uy, p = S.planes(x)
    lat = 2 * N + 1
    xs = np.arange(lat) / (2 * N)
    err_u = 0.0
    for j0 in range(0, lat, 1024):  # row blocks keep host memory small
        ys = xs[j0:j0 + 1024][:, None]
        X = xs[None, :]
        eux = X * (1 - X) * (2 * X - 1) * (6 * ys ** 2 - 6 * ys + 1)
        euy = ys * (ys - 1) * (2 * ys - 1) * (6 * X ** 2 - 6 * X + 1)
        err_u = max(err_u, np.abs(ux[j0:j0 + 1024].cpu().numpy() - eux).max(),
                    np.abs(uy[j0:j0 + 1024].cpu().numpy() - euy).max())
    ps = np.arange(N + 1) / N
    PX, PY = np.meshgrid(ps, ps)
    ep = PX ** 2 - 3 * PY ** 2 + 8.0 / 3.0 * PX * PY
    pn = p.cpu().numpy()
    err_p = np.abs((pn - pn.mean()) - (ep - ep.mean())).max()
    # discretisation is nodally exact; the remaining error is the 1e-10 solver tolerance
    assert err_u < 1e-8 and err_p < 1e-5, (err_u, err_p)
