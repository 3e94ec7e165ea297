"""Per-launch device times (ncu, serialised) of one FGMRES-preconditioner V-cycle
(x = 0 on entry) at N, grouped by kernel and level order (development aid):
    ncu --profile-from-start off --metrics gpu__time_duration.sum --csv python tools/vcycle_launches.py 4096
"""
import sys

import torch

from paper_2401_06277_b200 import Solver

N = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
S = Solver(N)
b, _ = S.set_problem("mms_paper")
z = S.new_vector()
for _ in range(2):
    S.precond_apply(b, z)
torch.cuda.synchronize()
torch.cuda.profiler.start()
S.precond_apply(b, z)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
