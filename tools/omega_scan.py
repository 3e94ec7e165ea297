"""FGMRES + V(1,1)-Vanka iteration counts and solve times vs the Vanka weight omega
(reading 6: W_i = omega diag(1/mult)) at several N (development aid)."""
import sys
import time

import torch

from paper_2401_06277_b200 import Solver

for N in [int(a) for a in sys.argv[1].split(",")]:
    for om in [float(a) for a in sys.argv[2].split(",")]:
        S = Solver(N, omega=om)
        out = []
        for kind in ("mms_paper", "cavity"):
            b, x0 = S.set_problem(kind)
            rep, _ = S.fgmres(b, x0, rtol=1e-10, maxit=80)
            b, x0 = S.set_problem(kind)
            torch.cuda.synchronize()
            t = time.perf_counter()
            rep, _ = S.fgmres(b, x0, rtol=1e-10, maxit=80)
            out.append("%s its %d %.1f ms" % (kind, rep["iterations"], 1e3 * (time.perf_counter() - t)))
        print("N=%d omega=%.3f: %s" % (N, om, "; ".join(out)), flush=True)
        S.close()
