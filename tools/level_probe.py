"""Per-level device time of the V-cycle building blocks (development aid)."""
import sys

import torch

from paper_2401_06277_b200 import Solver


def t_ev(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


N = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
S = Solver(N)
print("level N sweep_ms residual_ms restrict_ms prolong_ms")
tot = [0, 0, 0, 0]
for l in range(S.levels - 1, 0, -1):
    x = torch.randn(S.info[l].vec_len, dtype=torch.float64, device="cuda")
    b = torch.randn_like(x)
    o = torch.empty_like(x)
    xc = torch.zeros(S.info[l - 1].vec_len, dtype=torch.float64, device="cuda")
    ts = t_ev(lambda: S.sweep(l, x, b, out=o))
    tr = t_ev(lambda: S.residual(l, x, b, out=o))
    tq = t_ev(lambda: S.restrict(l, x, out=xc))
    tp = t_ev(lambda: S.prolong_add(l, xc, o))
    for k, v in enumerate((ts, tr, tq, tp)):
        tot[k] += v
    print(l, S.info[l].N, "%.4f %.4f %.4f %.4f" % (ts, tr, tq, tp))
print("sum", " ".join("%.3f" % v for v in tot))
bz = torch.zeros(S.info[0].vec_len, dtype=torch.float64, device="cuda")
print("coarse %.4f ms" % t_ev(lambda: S.coarse_solve(bz)))
b, x0 = S.set_problem("mms_paper")
z = S.new_vector()
print("vcycle %.3f ms" % t_ev(lambda: S.vcycle(b, z)))
print("matvec %.3f ms" % t_ev(lambda: S.matvec(S.fine, b, out=z)))
