"""Run one oracle FGMRES solve in its own process (test infrastructure).

    python tests/oracle_solve.py N KIND OUT.npz [MEM_GB]

KIND is mms_paper or cavity.  Writes iterations, residual history, true
relative residual, the setup / solve seconds and the solution at the sample
indices svk_inputs.random_sample_indices(N, 777, 20000) plus the whole
pressure plane's mean (pressures compare modulo the constant).  MEM_GB caps the
process's address space (RLIMIT_AS) so a too-large grid fails with an
allocation error instead of exhausting the host.
"""
import json
import os
import resource
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402


def main():
    N, kind, out = int(sys.argv[1]), sys.argv[2], sys.argv[3]
    if len(sys.argv) > 4:
        lim = int(float(sys.argv[4]) * 2 ** 30)
        resource.setrlimit(resource.RLIMIT_AS, (lim, lim))
    import oracle
    import svk_inputs
    code = {"mms_paper": oracle.MMS_PAPER, "cavity": oracle.CAVITY}[kind]
    t0 = time.perf_counter()
    o = oracle.Oracle(N)
    t1 = time.perf_counter()
    b, x0 = o.problem(code)
    x, its, hist, tr, st = o.fgmres(b, x0, rtol=1e-10, maxit=100)
    t2 = time.perf_counter()
    idx = svk_inputs.random_sample_indices(N, 777, 20000)
    nv = (2 * N + 1) ** 2
    np.savez(out, its=its, hist=hist, true_rel=tr, status=st, idx=idx, xs=x[idx], p_mean=x[2 * nv:].mean(),
             groups=np.array([o.num_groups(l) for l in range(o.levels)]))
    print(json.dumps({"N": N, "kind": kind, "iterations": its, "status": st, "true_rel": tr,
                      "setup_s": t1 - t0, "solve_s": t2 - t1, "threads": oracle.max_threads(),
                      "maxrss_gb": resource.getrusage(resource.RUSAGE_SELF).ru_maxrss / 2 ** 20}))


if __name__ == "__main__":
    main()
