"""Quick device-time probe of the sweep / V-cycle / FGMRES (development aid)."""
import sys
import time

import torch

from paper_2401_06277_b200 import Solver


def ev_time(fn, reps=10, warm=3):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps * 1e-3


def main():
    N = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
    for impl in ("fused", "unfused"):
        S = Solver(N, sweep=impl)
        b, x = S.set_problem("mms_paper")
        x = torch.randn_like(b)
        out = S.new_vector()
        t = ev_time(lambda: S.sweep(S.fine, x, b, out=out))
        nodes = (N + 1) ** 2
        dofs = 2 * (2 * N + 1) ** 2 + nodes
        print(f"{impl:8s} N={N} sweep {t*1e3:.3f} ms  {dofs/t/1e9:.2f} GDOF/s  {216*nodes/t/1e9:.0f} GB/s(alg)", flush=True)
        bz = b.clone()
        tv = ev_time(lambda: S.vcycle(bz, out), reps=5)
        print(f"{impl:8s} vcycle {tv*1e3:.3f} ms", flush=True)
        b, x0 = S.set_problem("mms_paper")
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        rep, hist = S.fgmres(b, x0, rtol=1e-10, maxit=60)
        torch.cuda.synchronize()
        print(f"{impl:8s} fgmres its={rep['iterations']} rel={rep['rel_residual']:.2e} wall={time.perf_counter()-t0:.3f}s "
              f"vcyc={rep['t_vcycle_s']:.3f}s orth={rep['t_orth_s']:.3f}s", flush=True)
        del S
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
