"""Per-iteration accounting of the FGMRES solve (development aid): device time of
solves capped at k iterations (rtol 0) against the V-cycle / orthogonalisation
times the report attributes, to expose per-iteration gaps (host sync, launches)."""
import sys

import torch

from paper_2401_06277_b200 import Solver

N = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
S = Solver(N)
b, x0 = S.set_problem("mms_paper")
x = S.new_vector()
for k in (1, 5, 10, 15, 19):
    res = []
    for rep in range(3):
        x.copy_(x0)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        r, _ = S.fgmres(b, x, rtol=0.0, maxit=k)
        e1.record()
        torch.cuda.synchronize()
        res.append((e0.elapsed_time(e1), 1e3 * r["t_vcycle_s"], 1e3 * r["t_orth_s"], r["n_reorth"]))
    t, tv, to, nr = min(res)
    print("k=%2d total %8.2f ms  vcycle %7.2f  orth %7.2f  other %6.2f  reorth %d" % (k, t, tv, to, t - tv - to, nr))
