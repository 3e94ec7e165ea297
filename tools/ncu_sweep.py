"""Drive a few fused sweeps for an ncu capture (development aid)."""
import sys

import torch

from paper_2401_06277_b200 import Solver

N = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
impl = sys.argv[2] if len(sys.argv) > 2 else "fused"
S = Solver(N, sweep=impl)
b, x = S.set_problem("mms_paper")
x = torch.randn_like(b)
out = S.new_vector()
for _ in range(3):
    S.sweep(S.fine, x, b, out=out)
torch.cuda.synchronize()
print("ok")
