"""Per-size device times (development aid; results -> profiles/r2_sizes.json):
fused sweep, V-cycle, and FGMRES+V(1,1)-Vanka solves (paper MMS and lid-driven
cavity); at 8192^2 the solve runs in the low-memory Krylov mode (only the
Arnoldi basis kept), the only way its basis fits one B200."""
import json
import sys

import torch

from paper_2401_06277_b200 import Solver
from tools.perf_probe import ev_time

out = []
for N in [int(a) for a in sys.argv[1:]] or [1024, 2048, 4096, 8192]:
    S = Solver(N)
    b, x0 = S.set_problem("mms_paper")
    x = torch.randn_like(b)
    o = S.new_vector()
    ts = ev_time(lambda: S.sweep(S.fine, x, b, out=o), reps=10)
    tv = ev_time(lambda: S.vcycle(b, o), reps=5)
    nodes, dofs = (N + 1) ** 2, 2 * (2 * N + 1) ** 2 + (N + 1) ** 2
    rec = {"N": N, "dofs": dofs, "sweep_ms": ts * 1e3, "sweep_gdof_s": dofs / ts / 1e9,
           "sweep_tflops_alg": 1316 * nodes / ts / 1e12, "vcycle_ms": tv * 1e3}
    del x, o
    if N > 4096:  # the FGMRES basis of 8192^2 needs the low-memory mode on one GPU
        del S, b, x0
        torch.cuda.empty_cache()
        S = Solver(N, low_memory=True)
        rec["solve_mode"] = "low-memory Krylov (krylov_store_z = 0)"
    if True:
        for kind in ("mms_paper",) if N > 4096 else ("mms_paper", "cavity"):
            b, x0 = S.set_problem(kind)
            xs = S.new_vector()
            best = None
            for _ in range(3):
                xs.copy_(x0)
                st, en = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                st.record()
                rep, _ = S.fgmres(b, xs, rtol=1e-10, maxit=60)
                en.record()
                torch.cuda.synchronize()
                t = st.elapsed_time(en) * 1e-3
                best = t if best is None else min(best, t)
            rec[kind] = {"iterations": rep["iterations"], "rel_residual": rep["rel_residual"], "time_to_solve_s": best,
                         "mdof_s": dofs / best / 1e6}
    print(json.dumps(rec), flush=True)
    out.append(rec)
    del S
    torch.cuda.empty_cache()
json.dump(out, open("gpurun_out/sizes.json", "w"), indent=1)
