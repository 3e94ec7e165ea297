"""svk_solve_host_batch vs svk_solve_host at N (development aid): wall time per
step and the per-problem solve times the reports carry."""
import sys
import time

import numpy as np
import torch

from paper_2401_06277_b200 import Solver

N = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
K = int(sys.argv[2]) if len(sys.argv) > 2 else 8
S = Solver(N)
b, x0 = S.set_problem("mms_paper")
bh = S.to_compact(b).cpu().pin_memory().numpy()
x0h = S.to_compact(x0).cpu().pin_memory().numpy()
xh = torch.empty(bh.size, dtype=torch.float64).pin_memory().numpy()
S.solve_host(bh, x0h, x_host=xh)
t = time.perf_counter()
_, r = S.solve_host(bh, x0h, x_host=xh)
print("single: %.1f ms wall, solve t_total %.1f ms" % (1e3 * (time.perf_counter() - t), 1e3 * r["t_total_s"]))
bl = [torch.from_numpy(bh.copy()).pin_memory().numpy() for _ in range(K)]
x0l = [torch.from_numpy(x0h.copy()).pin_memory().numpy() for _ in range(K)]
xl = [torch.empty(bh.size, dtype=torch.float64).pin_memory().numpy() for _ in range(K)]
for rep in range(2):
    t = time.perf_counter()
    _, reps, st = S.solve_host_batch(bl, x0l, x_hosts=xl)
    w = time.perf_counter() - t
    print("batch K=%d: %.1f ms wall per step; solve t_total per problem: %s" % (
        K, 1e3 * w / K, " ".join("%.1f" % (1e3 * q["t_total_s"]) for q in reps)))

# interference: a device-resident solve while 1D pinned H2D copies run on another stream
bd, x0d = S.set_problem("mms_paper")
host = torch.empty(300 * 2 ** 20, dtype=torch.float64).pin_memory()  # 2.4 GB
dev = torch.empty_like(host, device="cuda")
cs = torch.cuda.Stream()
cs2 = torch.cuda.Stream()
hout = torch.empty(150 * 2 ** 20, dtype=torch.float64).pin_memory()  # 1.2 GB
dsrc = torch.zeros_like(hout, device="cuda")
for label, copy in (("no copies", 0), ("concurrent 1D H2D", 1), ("concurrent 1D D2H", 2), ("both", 3)):
    x = x0d.clone()
    torch.cuda.synchronize()
    if copy & 1:
        with torch.cuda.stream(cs):
            for _ in range(3):
                dev.copy_(host, non_blocking=True)
    if copy & 2:
        with torch.cuda.stream(cs2):
            for _ in range(6):
                hout.copy_(dsrc, non_blocking=True)
    rep, _ = S.fgmres(bd, x, rtol=1e-10, maxit=60)
    torch.cuda.synchronize()
    print("%s: solve t_total %.1f ms" % (label, 1e3 * rep["t_total_s"]))
