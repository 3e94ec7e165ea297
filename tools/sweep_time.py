"""Device time of one fused sweep (x random) and one V-cycle at N (development aid)."""
import sys

import torch

from paper_2401_06277_b200 import Solver
from tools.perf_probe import ev_time

N = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
S = Solver(N)
b, x = S.set_problem("mms_paper")
x = torch.randn_like(b)
out = S.new_vector()
t = ev_time(lambda: S.sweep(S.fine, x, b, out=out), reps=20)
nodes = (N + 1) ** 2
tv = ev_time(lambda: S.vcycle(b, out), reps=10)
print(f"N={N} sweep {t*1e3:.3f} ms ({216*nodes/t/1e9:.0f} GB/s alg, {1316*nodes/t/1e12:.2f} TF alg)  vcycle {tv*1e3:.3f} ms", flush=True)
r = S.new_vector()
tr = ev_time(lambda: S.residual(S.fine, x, b, out=r), reps=20)
tm = ev_time(lambda: S.matvec(S.fine, x, out=r), reps=20)
print(f"N={N} residual {tr*1e3:.3f} ms ({216*nodes/tr/1e9:.0f} GB/s alg)  matvec {tm*1e3:.3f} ms ({144*nodes/tm/1e9:.0f} GB/s alg)", flush=True)
