"""FGMRES iteration parity against the oracle at the benchmarked sizes
(north_star: "an FGMRES+V(Vanka) time-to-solution agreeing with the oracle's
iteration count"; BASELINE.json configs[1] = the 1024^2 lid-driven cavity).

The GPU solve runs first (default launch configuration, as bench.py times it)
and its context is freed; the oracle then solves the same problem in its own
process (tests/oracle_solve.py, address space capped) on the host cores.
Checked: iterations within +-1, 25 patch groups on every oracle level, the
residual history while it is well above roundoff, and the solution at 20,000
seeded sample positions (pressure modulo the constant, reading 3).

Always run: 1024^2 cavity and MMS.  SVK_LARGE_ORACLE=2048,4096 adds MMS runs
at those sizes (the 4096^2 oracle needs ~150 GB of host memory and ~15 min).
"""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))
CASES = [(1024, "cavity"), (1024, "mms_paper")]
if os.environ.get("SVK_LARGE_ORACLE"):
    CASES += [(int(n), "mms_paper") for n in os.environ["SVK_LARGE_ORACLE"].split(",")]


@pytest.mark.parametrize("N,kind", CASES)
def test_fgmres_iteration_parity_at_size(gpu, tmp_path, N, kind):
    import torch
    from paper_2401_06277_b200 import Solver
    S = Solver(N)
    levels = S.levels
    b, x = S.set_problem(kind)
    rep, hist = S.fgmres(b, x, rtol=1e-10, maxit=100)
    xc = S.to_compact(x).cpu().numpy()
    S.close()
    del S, b, x
    torch.cuda.empty_cache()
    assert rep["converged"] == 1

    out = str(tmp_path / "oracle.npz")
    mem_gb = 180 if N >= 4096 else 120
    r = subprocess.run([sys.executable, os.path.join(HERE, "oracle_solve.py"), str(N), kind, out, str(mem_gb)],
                       capture_output=True, text=True, timeout=7200)
    assert r.returncode == 0, r.stderr[-3000:]
    info = json.loads(r.stdout.strip().splitlines()[-1])
    d = np.load(out)
    its = int(d["its"])
    info.update(gpu_iterations=rep["iterations"], gpu_rel_residual=rep["rel_residual"], gpu_t_total_s=rep["t_total_s"])
    rec = os.path.join(os.path.dirname(HERE), "gpurun_out")
    if os.path.isdir(rec):
        with open(os.path.join(rec, "iteration_parity.jsonl"), "a") as f:
            f.write(json.dumps(info) + "\n")

    assert int(d["status"]) == 0
    assert list(d["groups"]) == [25] * levels
    assert abs(rep["iterations"] - its) <= 1, info
    ho = d["hist"]
    k = min(len(hist), len(ho))
    m = ho[:k] > 1e-6
    assert np.all(np.abs(hist[:k][m] - ho[:k][m]) <= 1e-6 * ho[:k][m])
    idx, xs = d["idx"], d["xs"]
    nvel = 2 * (2 * N + 1) ** 2
    vel = idx < nvel
    g = xc[idx]
    scale = max(np.abs(xs[vel]).max(), 1e-30)
    assert np.abs(g[vel] - xs[vel]).max() < 1e-8 * scale + 1e-12
    gp = g[~vel] - xc[nvel:].mean()
    op = xs[~vel] - float(d["p_mean"])
    assert np.abs(gp - op).max() < 1e-6 * max(np.abs(op).max(), 1.0)
