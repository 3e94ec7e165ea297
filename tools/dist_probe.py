"""p emulated ranks of one FGMRES solve on one GPU (development aid for the
multi-GPU path): python tools/dist_probe.py P N AGGLOM.  A rank that fails
prints its error and ends the process at once (the others would wait at the
next emulated barrier)."""
import os
import sys
import threading
import traceback

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "tests"))
os.environ.setdefault("SVK_POISON_HALO", "1")
import test_gpu_dist as T  # noqa: E402

P, N, agg = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
Ss = T.make_solvers(P, N, agg)
out = [None] * P


def body(r):
    import torch
    try:
        torch.cuda.set_device(0)
        st = torch.cuda.Stream()
        with torch.cuda.stream(st):
            S = Ss[r]
            b, x = S.set_problem("mms_paper")
            rep, hist = S.fgmres(b, x, rtol=1e-10, maxit=100)
            st.synchronize()
            out[r] = rep["iterations"]
    except BaseException:
        sys.stderr.write("rank %d failed:\n%s" % (r, traceback.format_exc()))
        sys.stderr.flush()
        os._exit(1)


th = [threading.Thread(target=body, args=(r,), daemon=True) for r in range(P)]
for t in th:
    t.start()
for t in th:
    t.join()
print(out, "device bytes per rank", [S.device_bytes for S in Ss])
