"""Device time of one V-cycle (svk_vcycle from zero) at size N, CUDA events
(development aid; SVK_LIBRARY selects a library variant for A/B runs)."""
import sys

import torch

from paper_2401_06277_b200 import Solver

N = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
S = Solver(N)
b, _ = S.set_problem("mms_paper")
x = S.new_vector()
for _ in range(3):
    S.vcycle(b, x)
torch.cuda.synchronize()
a, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
best = 1e9
for rep in range(3):
    a.record()
    for _ in range(10):
        S.vcycle(b, x)
    e.record()
    torch.cuda.synchronize()
    best = min(best, a.elapsed_time(e) / 10)
print("N=%d vcycle %.3f ms" % (N, best))
