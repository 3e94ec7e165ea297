"""The GPU path is deterministic (owner-computes accumulation in a fixed
order, no atomics, fixed reduction trees): repeating a sweep, a V-cycle, the
Gram-Schmidt reductions and a whole FGMRES solve gives bitwise identical results,
also across the strip kernels' chunking of the grid into waves."""
import numpy as np
import pytest

import svk_inputs

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("N", [64, 512])
def test_bitwise_repeatable(gpu, N):
    import torch
    from paper_2401_06277_b200 import Solver
    S = Solver(N)
    x = S.from_compact(svk_inputs.random_vector(N, 61))
    b = S.from_compact(svk_inputs.random_vector(N, 62))
    s1 = S.sweep(S.fine, x, b).clone()
    s2 = S.sweep(S.fine, x, b).clone()
    assert torch.equal(s1, s2)
    v1 = S.vcycle(b).clone()
    v2 = S.vcycle(b).clone()
    assert torch.equal(v1, v2)
    bg, x0 = S.set_problem("mms_paper")
    xa, xb = x0.clone(), x0.clone()
    ra, ha = S.fgmres(bg, xa, rtol=1e-10, maxit=60)
    rb, hb = S.fgmres(bg, xb, rtol=1e-10, maxit=60)
    assert ra["iterations"] == rb["iterations"]
    assert np.array_equal(ha, hb)
    assert torch.equal(xa, xb)
