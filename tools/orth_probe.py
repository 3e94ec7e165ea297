"""FGMRES orthogonalisation modes at full size: iterations, second passes, times."""
import sys
import time

import torch

from paper_2401_06277_b200 import Solver


def main():
    N = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
    for kind in ("mms_paper", "cavity"):
        for orth in ("adaptive", "cgs2"):
            S = Solver(N, orth=orth)
            b, x0 = S.set_problem(kind)
            x = S.new_vector()
            for rep_i in range(2):
                x.copy_(x0)
                torch.cuda.synchronize()
                t0 = time.perf_counter()
                rep, hist = S.fgmres(b, x, rtol=1e-10, maxit=100)
                torch.cuda.synchronize()
                t = time.perf_counter() - t0
            print(f"{kind:9s} {orth:8s} N={N} its={rep['iterations']} reorth={rep['n_reorth']} "
                  f"rel={rep['rel_residual']:.2e} wall={t:.3f}s vcyc={rep['t_vcycle_s']:.3f}s "
                  f"orth={rep['t_orth_s']:.3f}s", flush=True)
            del S, b, x0, x
            torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
