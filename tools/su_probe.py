"""Development probe: SU / BS V-cycle parity and FGMRES at mid sizes."""
import numpy as np, torch, sys
import oracle, svk_inputs
from paper_2401_06277_b200 import Solver
kind = sys.argv[1] if len(sys.argv) > 1 else "su"
ok = {"su": (2, dict(t=1, omega_j=0.4, nj=1)), "bs": (1, dict(t=1, omega_r=1, omega_j=0.8, nj=3))}[kind]
for N in (64, 128, 256):
    S = Solver(N, relax=kind)
    O = oracle.Oracle(N); O.set_relax(ok[0], **ok[1])
    b = svk_inputs.random_vector(N, 9); b[O.dirichlet(O.fine)] = 0
    xo = O.vcycle(b)
    xg = S.to_compact(S.vcycle(S.from_compact(b))).cpu().numpy()
    print(N, "vcycle rel", np.linalg.norm(xg - xo) / np.linalg.norm(xo), np.isfinite(xg).all(), flush=True)
    x2 = xo.copy()
    for l in range(S.levels):
        n = S.info[l].N
        x = svk_inputs.random_vector(n, 1); bb = svk_inputs.random_vector(n, 2)
        a = O.relax_sweep(l, x, bb); g = S.to_compact(S.relax_sweep(l, S.from_compact(x, l), S.from_compact(bb, l)), l).cpu().numpy()
        print("   level", l, n, np.linalg.norm((g - x) - (a - x)) / np.linalg.norm(a - x), flush=True)
    bg, x0 = S.set_problem("mms_paper")
    try:
        rep, h = S.fgmres(bg, x0, rtol=1e-10, maxit=200)
        print(N, rep["iterations"], rep["rel_residual"], flush=True)
    except Exception as e:
        print(N, "ERR", e, flush=True)
    del S; torch.cuda.empty_cache()
