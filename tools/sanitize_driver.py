"""Exercise every kernel of the default hot path once at a small size for
compute-sanitizer (racecheck / synccheck / memcheck / initcheck):
fused sweep (k_boundary_patches + k_vanka_fused), residual and mat-vec strips,
a V-cycle (k_vanka_zero, k_residual_strip<0,1>, k_prolong, coarse solve) and a
few FGMRES iterations (Krylov kernels).

    compute-sanitizer --tool racecheck python tools/sanitize_driver.py 64
"""
import sys

import torch

from paper_2401_06277_b200 import Solver

N = int(sys.argv[1]) if len(sys.argv) > 1 else 64
S = Solver(N)
b, x0 = S.set_problem("mms_paper")
g = torch.Generator(device="cuda").manual_seed(5)
x = x0 + 0.1 * torch.randn(x0.shape, dtype=torch.float64, device="cuda", generator=g)
out = S.sweep(S.fine, S.from_compact(S.to_compact(x)), b)
r = S.residual(S.fine, out, b)
y = S.matvec(S.fine, out)
z = S.vcycle(b)
xx = x0.clone()
rep, _ = S.fgmres(b, xx, rtol=1e-10, maxit=4)
torch.cuda.synchronize()
print("ok N=%d sweep %.6e res %.6e mv %.6e vc %.6e its %d" % (N, float(out.abs().sum()), float(r.abs().sum()),
                                                               float(y.abs().sum()), float(z.abs().sum()),
                                                               rep["iterations"]))
