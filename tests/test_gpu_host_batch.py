"""svk_solve_host_batch (include/svk.h): the pipelined host-buffer solves give
bitwise the results of one svk_solve_host call per problem (the copies of problems
k+1 / k-1 only overlap the solve of problem k), with per-problem reports; argument
errors are rejected before any work."""
import numpy as np
import pytest

from paper_2401_06277_b200 import Solver, SvkError

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("N", [32, 128])
def test_batch_equals_single_solves(gpu, N):
    import torch
    S = Solver(N)
    probs = []
    for kind in ("mms_paper", "cavity", "mms_inspace"):
        b, x0 = S.set_problem(kind)
        probs.append((S.to_compact(b).cpu().numpy().copy(), S.to_compact(x0).cpu().numpy().copy()))
    g = np.random.default_rng(3)
    probs.append((probs[0][0] + 1e-3 * g.standard_normal(probs[0][0].size), probs[0][1].copy()))
    singles = [S.solve_host(b, x0, rtol=1e-10, maxit=80) for b, x0 in probs]
    pinned = [(torch.from_numpy(b).pin_memory().numpy(), torch.from_numpy(x0).pin_memory().numpy()) for b, x0 in probs]
    xs, reps, st = S.solve_host_batch([p[0] for p in pinned], [p[1] for p in pinned], rtol=1e-10, maxit=80)
    assert st == max(r["status"] for _, r in singles)
    assert reps[0]["converged"] == 1
    for (x1, r1), x2, r2 in zip(singles, xs, reps):
        assert np.array_equal(x1, x2)
        assert r1["iterations"] == r2["iterations"] and r1["converged"] == r2["converged"]
        assert r1["rel_residual"] == r2["rel_residual"]


def test_batch_argument_errors(gpu):
    S = Solver(16)
    b, x0 = S.set_problem("mms_paper")
    bh, x0h = S.to_compact(b).cpu().numpy(), S.to_compact(x0).cpu().numpy()
    with pytest.raises(SvkError):
        S.solve_host_batch([bh], [x0h, x0h])
    with pytest.raises(SvkError):
        S.solve_host_batch([bh], [x0h], x_hosts=[bh])       # aliasing
    with pytest.raises(SvkError):
        S.solve_host_batch([bh[:-1]], [x0h])                # wrong length
