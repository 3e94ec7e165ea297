"""The launch-time switches leave results unchanged: the V-cycle and an FGMRES solve
with programmatic dependent launch off (SVK_PDL=0) and with other strip chunkings
(SVK_CHUNK_ROWS) match the oracle like the default configuration.  The switches
are read once per process, so each configuration runs in a subprocess."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = r"""
import json, sys
import numpy as np
import oracle, svk_inputs
from paper_2401_06277_b200 import Solver
N = int(sys.argv[1])
S, O = Solver(N), oracle.Oracle(N)
l = S.fine
b = svk_inputs.random_vector(N, 3)
b[O.dirichlet(l)] = 0.0
vg = S.to_compact(S.vcycle(S.from_compact(b))).cpu().numpy()
vo = O.vcycle(b)
x = svk_inputs.random_vector(N, 4)
sg = S.to_compact(S.sweep(l, S.from_compact(x), S.from_compact(b))).cpu().numpy()
so = O.sweep(l, x, b)
bg, x0 = S.set_problem("mms_paper")
rep, _ = S.fgmres(bg, x0, rtol=1e-10, maxit=100)
rel = lambda a, c: float(np.linalg.norm(a - c) / np.linalg.norm(c))
print(json.dumps({"vcycle": rel(vg, vo), "sweep": rel(sg - x, so - x), "its": rep["iterations"]}))
"""


def run(env_extra, N):
    env = dict(os.environ, PYTHONPATH=ROOT, **env_extra)
    out = subprocess.run([sys.executable, "-c", SCRIPT, str(N)], cwd=ROOT, env=env, capture_output=True, text=True,
                         timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    return json.loads(out.stdout.strip().splitlines()[-1])


@pytest.mark.parametrize("env_extra", [{"SVK_PDL": "0"}, {"SVK_CHUNK_ROWS": "8"}, {"SVK_CHUNK_ROWS": "1000"},
                                       {"SVK_GRAPHS": "0"}])
def test_launch_switches_keep_parity(gpu, env_extra):
    N = 128
    r = run(env_extra, N)
    assert r["vcycle"] < 1e-12, r
    assert r["sweep"] < 1e-12, r
    import oracle
    O = oracle.Oracle(N)
    bo, x0o = O.problem(oracle.MMS_PAPER)
    its_o = O.fgmres(bo, x0o, rtol=1e-10, maxit=100)[1]
    assert abs(r["its"] - its_o) <= 1, (r, its_o)


GRAPH_SCRIPT = r"""
import json, sys
import numpy as np
import torch
from paper_2401_06277_b200 import Solver
N = int(sys.argv[1])
S = Solver(N)
b, x0 = S.set_problem("mms_paper")
S.set_profiling(True)
S.sweep_stats()
out = []
for rep_i in range(2):  # the second solve replays the captured graphs
    x = x0.clone()
    l0 = S.launch_count
    rep, hist = S.fgmres(b, x, rtol=1e-10, maxit=100)
    torch.cuda.synchronize()
    nsw, ms = S.sweep_stats()
    out.append({"its": rep["iterations"], "hist": hist.tolist(), "x": float(x.double().abs().sum()),
                "xhash": float((x * torch.arange(x.numel(), device=x.device, dtype=x.dtype).remainder(97)).sum()),
                "launches": S.launch_count - l0, "nsw": nsw, "sweep_ms": ms})
print(json.dumps(out))
"""


def test_graph_replay_is_bitwise_identical_to_direct_launches(gpu):
    """The FGMRES preconditioner V-cycle replayed from captured CUDA graphs gives
    bitwise the same iterates as direct launches (fixed reduction orders), and
    the graph path still reports its kernel count and the timed finest sweeps."""
    res = {}
    for g in ("0", "1"):
        env = dict(os.environ, PYTHONPATH=ROOT, SVK_GRAPHS=g)
        out = subprocess.run([sys.executable, "-c", GRAPH_SCRIPT, "256"], cwd=ROOT, env=env, capture_output=True,
                             text=True, timeout=600)
        assert out.returncode == 0, out.stderr[-2000:]
        res[g] = json.loads(out.stdout.strip().splitlines()[-1])
    for k in range(2):
        a, c = res["0"][k], res["1"][k]
        assert a["its"] == c["its"] and a["hist"] == c["hist"] and a["x"] == c["x"] and a["xhash"] == c["xhash"]
        assert a["launches"] == c["launches"] > 0
        assert a["nsw"] == c["nsw"] == a["its"] and c["sweep_ms"] > 0
