"""One V-cycle (or FGMRES solve) bracketed by cudaProfilerStart/Stop for an ncu launch list:
    ncu --profile-from-start off --metrics gpu__time_duration.sum --csv python tools/ncu_vcycle.py 4096 [vcycle|fgmres] [vanka|bs|su]
"""
import sys

import torch

from paper_2401_06277_b200 import Solver

N = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
what = sys.argv[2] if len(sys.argv) > 2 else "vcycle"
relax = sys.argv[3] if len(sys.argv) > 3 else "vanka"
S = Solver(N, relax=relax)
b, x0 = S.set_problem("mms_paper")
z = S.new_vector()
for _ in range(2):
    S.vcycle(b, z)
torch.cuda.synchronize()
torch.cuda.profiler.start()
if what == "vcycle":
    S.vcycle(b, z)
else:
    S.fgmres(b, x0, rtol=1e-10, maxit=100)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
