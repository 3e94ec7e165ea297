"""Device time of V-cycles at N (development aid for the x = 0 sweep variants; SVK_LEAN env)."""
import sys

import torch

from paper_2401_06277_b200 import Solver
from tools.perf_probe import ev_time

N = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
S = Solver(N)
b, x = S.set_problem("mms_paper")
out = S.new_vector()
tv = ev_time(lambda: S.vcycle(b, out), reps=10)
print(f"N={N} vcycle {tv*1e3:.3f} ms", flush=True)
