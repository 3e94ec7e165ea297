"""Multi-GPU row-slab path on ONE device:
p logical ranks run in p host threads through the EMULATED transport (same
partition, halo exchanges, agglomeration and all-reduces as NCCL; only the
byte mover differs).  Every distributed result is compared with the CPU
oracle (the parity bar of test_gpu_parity.py) and with the single-rank GPU
path.  SVK_POISON_HALO=1 fills every row beyond a rank's halo with NaN after
each exchange, so a kernel that reads outside its halo fails the test.
"""
import itertools
import threading

import numpy as np
from parity_util import rel
import pytest

import oracle
import svk_inputs

pytestmark = pytest.mark.gpu

_group = itertools.count(1000)




def run_ranks(P, fn, timeout=300):
    """fn(rank) in P threads, each on its own CUDA stream; returns the results."""
    import torch
    out, errs = [None] * P, []

    def body(r):
        try:
            torch.cuda.set_device(0)
            st = torch.cuda.Stream()
            with torch.cuda.stream(st):
                out[r] = fn(r)
                st.synchronize()
        except BaseException as e:  # noqa: BLE001 - reported below
            errs.append((r, e))

    th = [threading.Thread(target=body, args=(r,), daemon=True) for r in range(P)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout)
    assert not any(t.is_alive() for t in th), "a rank hung (barrier mismatch)"
    if errs:
        raise errs[0][1]
    return out


def make_solvers(P, N, agglom, **kw):
    from paper_2401_06277_b200 import Solver
    g = next(_group)
    return [Solver(N, rank=r, nranks=P, transport="emulated", agglom_rows=agglom, emul_group=g, **kw)
            for r in range(P)]


def owned_compact(S, v, level=None):
    """compact vector with the rows outside this rank's slab set to NaN"""
    level = S.fine if level is None else level
    r0, r1, d = S.owned_rows(level)
    ux, uy, p = [t.cpu().numpy().copy() for t in S.planes(v, level)]
    if d:
        lat = ux.shape[0]
        for a in (ux, uy):
            a[:2 * r0] = np.nan
            a[min(2 * r1, lat):] = np.nan
        p[:r0] = np.nan
        p[r1:] = np.nan
    return np.concatenate([ux.ravel(), uy.ravel(), p.ravel()])


def merge(parts):
    """combine per-rank compact vectors (NaN outside the owned rows)"""
    out = np.full_like(parts[0], np.nan)
    for q in parts:
        m = ~np.isnan(q)
        assert not np.any(m & ~np.isnan(out)), "overlapping slabs"
        out[m] = q[m]
    assert not np.any(np.isnan(out)), "rows owned by no rank"
    return out


CASES = [(2, 64, 8), (3, 64, 4), (4, 64, 4), (2, 128, 16)]


@pytest.fixture
def poison(monkeypatch):
    monkeypatch.setenv("SVK_POISON_HALO", "1")


@pytest.mark.parametrize("P,N,agg", CASES)
def test_partition_matches_levels(gpu, P, N, agg):
    from paper_2401_06277_b200 import svk
    Ss = make_solvers(P, N, agg)
    for S in Ss:
        for l in range(S.levels):
            li = S.info[l]
            r0, r1, d = svk.partition(N, 4, P, S.rank, agg, li.N)
            assert (li.row0, li.row1, bool(li.distributed)) == (r0, r1, d)
            assert li.halo_rows == (4 if d else 0)
        assert S.info[S.fine].distributed
    for S in Ss:
        S.close()


@pytest.mark.parametrize("P,N,agg", CASES)
def test_dist_residual_and_sweep(gpu, poison, P, N, agg):
    O = oracle.Oracle(N)
    Ss = make_solvers(P, N, agg)
    L = Ss[0].fine
    x = svk_inputs.random_vector(N, 11)
    b, _ = O.problem(oracle.MMS_PAPER)
    ref_r = O.residual(L, x, b)
    ref_s = O.sweep(L, x, b)
    ref_s3 = O.sweep(L, O.sweep(L, ref_s, b), b)

    def fn(r):
        S = Ss[r]
        xg, bg = S.from_compact(x), S.from_compact(b)
        rr = S.residual(L, xg, bg)
        xs = S.sweep(L, xg, bg)
        xs3 = S.sweep(L, xg, bg, nsweeps=3)
        return owned_compact(S, rr), owned_compact(S, xs), owned_compact(S, xs3)

    res = run_ranks(P, fn)
    assert rel(merge([q[0] for q in res]), ref_r) < 1e-13
    assert rel(merge([q[1] for q in res]) - x, ref_s - x) < 1e-12
    assert rel(merge([q[2] for q in res]) - x, ref_s3 - x) < 1e-12
    for S in Ss:
        S.close()


@pytest.mark.parametrize("P,N,agg,coarse", [c + ("exact",) for c in CASES] + [(2, 64, 8, "sweeps3")])
def test_dist_vcycle(gpu, poison, P, N, agg, coarse):
    O = oracle.Oracle(N, coarse_mode=1 if coarse == "sweeps3" else 0)
    Ss = make_solvers(P, N, agg, coarse=coarse)
    b = svk_inputs.random_vector(N, 5)
    b[O.dirichlet(O.fine)] = 0.0
    x0 = svk_inputs.random_vector(N, 25)
    ref, ref0 = O.vcycle(b), O.vcycle(b, x0)

    def fn(r):
        S = Ss[r]
        x = S.vcycle(S.from_compact(b))
        y = S.vcycle(S.from_compact(b), S.from_compact(x0))
        return owned_compact(S, x), owned_compact(S, y), bool(S.torch.isnan(x).any())

    res = run_ranks(P, fn)
    assert all(q[2] for q in res)  # the poison is live: rows beyond each halo hold NaN
    assert rel(merge([q[0] for q in res]), ref) < 1e-12
    assert rel(merge([q[1] for q in res]) - x0, ref0 - x0) < 1e-12
    for S in Ss:
        S.close()


@pytest.mark.parametrize("P,N,agg", CASES + [(2, 64, 64), (8, 512, 32)])
def test_dist_fgmres_vs_oracle_and_single(gpu, poison, P, N, agg):
    from paper_2401_06277_b200 import Solver
    O = oracle.Oracle(N)
    bo, x0o = O.problem(oracle.MMS_PAPER)
    xo, its, ho, _, st = O.fgmres(bo, x0o, rtol=1e-10, maxit=100)
    S1 = Solver(N)
    b1, x1 = S1.set_problem("mms_paper")
    rep1, hist1 = S1.fgmres(b1, x1, rtol=1e-10, maxit=100)
    x1c = S1.to_compact(x1).cpu().numpy()
    Ss = make_solvers(P, N, agg)

    def fn(r):
        S = Ss[r]
        b, x = S.set_problem("mms_paper")
        rep, hist = S.fgmres(b, x, rtol=1e-10, maxit=100)
        part = owned_compact(S, x)
        S.allgather(x)
        return rep, hist, part, S.to_compact(x).cpu().numpy()

    res = run_ranks(P, fn)
    for rep, hist, _, full in res:
        assert rep["converged"] == 1 and rep["status"] == 0
        assert rep["iterations"] == res[0][0]["iterations"]
        assert abs(rep["iterations"] - its) <= 1
        assert abs(rep["iterations"] - rep1["iterations"]) <= 1
        assert rep["rel_residual"] < 1e-9
        np.testing.assert_array_equal(hist, res[0][1])  # identical on every rank
        if rep["iterations"] == rep1["iterations"]:
            assert np.all(np.abs(hist - hist1) <= 1e-8 * np.maximum(hist1, 1e-12))
    xd = merge([q[2] for q in res]) if Ss[0].owned_rows()[2] else res[0][2]
    for q in res:  # allgather assembles the same full vector everywhere
        assert np.array_equal(q[3], xd)
    nv = (2 * N + 1) ** 2
    scale = max(np.abs(xo[:2 * nv]).max(), 1.0)
    assert np.abs(xd[:2 * nv] - xo[:2 * nv]).max() < 1e-8 * scale
    assert np.abs(xd[:2 * nv] - x1c[:2 * nv]).max() < 1e-8 * scale
    pd, po = xd[2 * nv:], xo[2 * nv:]
    assert np.abs((pd - pd.mean()) - (po - po.mean())).max() < 1e-6 * max(np.abs(po).max(), 1.0)
    S1.close()
    for S in Ss:
        S.close()


def test_dist_solve_host(gpu, poison):
    P, N, agg = 2, 64, 8
    O = oracle.Oracle(N)
    bo, x0o = O.problem(oracle.CAVITY)
    xo, its, _, _, _ = O.fgmres(bo, x0o, rtol=1e-10, maxit=100)
    Ss = make_solvers(P, N, agg)
    res = run_ranks(P, lambda r: Ss[r].solve_host(bo, x0o, rtol=1e-10, maxit=100))
    for x, rep in res:
        assert rep["converged"] == 1 and abs(rep["iterations"] - its) <= 1
        nv = (2 * N + 1) ** 2
        assert np.abs(x[:2 * nv] - xo[:2 * nv]).max() < 1e-8
    assert np.array_equal(res[0][0], res[1][0])
    for S in Ss:
        S.close()


def test_dist_solve_host_batch(gpu, poison):
    # svk_solve_host_batch on 2 emulated ranks: every rank assembles every solution,
    # bitwise the per-problem svk_solve_host results
    P, N, agg = 2, 64, 8
    O = oracle.Oracle(N)
    probs = [O.problem(oracle.CAVITY), O.problem(oracle.MMS_PAPER)]
    Ss = make_solvers(P, N, agg)
    single = run_ranks(P, lambda r: [Ss[r].solve_host(b, x0, rtol=1e-10, maxit=100) for b, x0 in probs])
    batch = run_ranks(P, lambda r: Ss[r].solve_host_batch([p[0] for p in probs], [p[1] for p in probs],
                                                          rtol=1e-10, maxit=100))
    for r in range(P):
        xs, reps, st = batch[r]
        assert st == 0
        for (x1, r1), x2, r2 in zip(single[r], xs, reps):
            assert np.array_equal(x1, x2) and r1["iterations"] == r2["iterations"]
    assert all(np.array_equal(a, b) for a, b in zip(batch[0][0], batch[1][0]))
    for S in Ss:
        S.close()


def test_dist_config_errors(gpu):
    from paper_2401_06277_b200 import Solver, SvkError
    with pytest.raises(SvkError):
        Solver(64, rank=0, nranks=2, transport="none")
    with pytest.raises(SvkError):
        Solver(64, rank=2, nranks=2, transport="emulated")
    with pytest.raises(SvkError):
        Solver(64, rank=0, nranks=2, transport="emulated", agglom_rows=2)
    with pytest.raises(SvkError):
        Solver(64, rank=0, nranks=2, transport="emulated", sweep="unfused")


@pytest.mark.parametrize("P", [2, 4])
def test_slab_local_memory_per_rank(gpu, P):
    """Distributed-level workspaces and the Krylov basis are slab-local: each rank
    maps ~1/P of every such vector (plus halo, margin and page rounding), so a
    rank's device memory is ~1/P of the single-GPU footprint (the replicated
    coarse levels are small).  SVK_SLAB_LOCAL=0 would map them full size."""
    from paper_2401_06277_b200 import Solver
    N, its = 2048, 4
    S1 = Solver(N)
    b, x = S1.set_problem("mms_paper")
    S1.fgmres(b, x, rtol=0.0, maxit=its)   # allocates its + 1 basis pairs
    full = S1.device_bytes
    S1.close()
    del S1, b, x
    Ss = make_solvers(P, N, 64)

    def fn(r):
        S = Ss[r]
        b, x = S.set_problem("mms_paper")
        S.fgmres(b, x, rtol=0.0, maxit=its)
        return S.device_bytes

    per_rank = run_ranks(P, fn)
    for nb in per_rank:
        assert nb < full * (1.0 / P + 0.12), (nb, full, P)
    assert sum(per_rank) < full * 1.25
    for S in Ss:
        S.close()
