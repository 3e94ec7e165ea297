"""Per-phase times of the one-launch coarse V-cycle (development aid):
SVK_GRAPHS=0 SVK_DEBUG_SMALL=2 SVK_SMALL_N=16 python tools/sc_stamps.py 1024"""
import sys

import torch

from paper_2401_06277_b200 import Solver

N = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
S = Solver(N)
b, _ = S.set_problem("mms_paper")
z = S.new_vector()
for _ in range(3):
    S.precond_apply(b, z)
torch.cuda.synchronize()
