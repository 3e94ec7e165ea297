"""Tiny fused sweep for sanitizer / debugging runs."""
import sys

import torch

from paper_2401_06277_b200 import Solver

N = int(sys.argv[1]) if len(sys.argv) > 1 else 16
S = Solver(N)
b, x = S.set_problem("mms_paper")
x = torch.randn_like(b)
out = S.sweep(S.fine, x, b)
torch.cuda.synchronize()
print("ok", float(out.abs().sum()))
