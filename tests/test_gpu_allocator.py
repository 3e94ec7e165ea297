"""svk_config.alloc_fn / free_fn (include/svk.h): the context's vector workspaces
come from the caller's allocator (here torch's caching allocator), the solve is
bitwise the one of the default cudaMalloc context, and svk_destroy hands every
block back.  Also svk_report.t_setup_s."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

N = 128


def solve(S):
    b, x = S.set_problem("mms_paper")
    rep, hist = S.fgmres(b, x, rtol=1e-10, maxit=40)
    S.torch.cuda.synchronize()
    return rep, hist, x.cpu().numpy()


def test_torch_allocator_matches_cuda_and_returns_blocks(gpu):
    import torch
    from paper_2401_06277_b200 import Solver
    ref = Solver(N)
    rep0, hist0, x0 = solve(ref)
    bytes0 = ref.device_bytes
    ref.close()

    torch.cuda.synchronize()
    base = torch.cuda.memory_allocated(gpu)
    S = Solver(N, allocator="torch")
    after_create = torch.cuda.memory_allocated(gpu)
    assert after_create > base   # level workspaces now live in torch's pool
    rep1, hist1, x1 = solve(S)
    # the Krylov basis (allocated lazily by the first solve) also comes from torch
    grown = torch.cuda.memory_allocated(gpu) - base
    assert S.device_bytes == bytes0
    assert S.device_bytes <= grown <= S.device_bytes + 16 * 2 ** 20
    assert rep1["iterations"] == rep0["iterations"] and rep1["converged"] == 1
    assert np.array_equal(x0, x1) and np.array_equal(np.asarray(hist0), np.asarray(hist1))
    del x1
    S.close()
    torch.cuda.synchronize()
    # every block svk took went back (the only tensors left are the test's own)
    assert torch.cuda.memory_allocated(gpu) <= base + 2 ** 20


def test_allocator_failure_is_reported(gpu):
    import ctypes as C
    from paper_2401_06277_b200 import svk
    lib = svk.load_library()
    calls = []
    alloc = svk.ALLOC_FN(lambda n, d, u: calls.append(n) or None)   # always fails
    free = svk.FREE_FN(lambda p, n, d, u: None)
    c = svk.Config()
    lib.svk_config_default(C.byref(c), 32)
    c.alloc_fn, c.free_fn = C.cast(alloc, C.c_void_p), C.cast(free, C.c_void_p)
    h = C.c_void_p()
    st = lib.svk_create(C.byref(c), C.byref(h))
    assert st == -2 and calls   # SVK_ERR_CUDA after the first refused block
    assert not h.value


def test_report_carries_setup_time(gpu):
    from paper_2401_06277_b200 import Solver
    S = Solver(64)
    rep, _, _ = solve(S)
    assert 0.0 < rep["t_setup_s"] < 60.0
    assert rep["t_total_s"] > 0.0


def test_guarded_workspaces_no_out_of_bounds_access(gpu):
    # Every vector workspace of the context (level vectors, boundary-patch and
    # coarse-cycle buffers, Krylov basis) comes from an allocator that surrounds
    # the block with 64 KB guard zones of NaN: an out-of-bounds write changes a
    # guard (checked at free), an out-of-bounds read pulls a NaN into the result
    # (the solve must still match the plain context bitwise).  This stands in for
    # compute-sanitizer memcheck, which the GPU pool does not allow.
    import ctypes as C

    import torch
    from paper_2401_06277_b200 import Solver
    from paper_2401_06277_b200.svk import ALLOC_FN, FREE_FN
    G = 1 << 16
    live, bad = {}, []

    def _alloc(nbytes, device, user):
        t = torch.full(((int(nbytes) + 2 * G + 7) // 8,), float("nan"), dtype=torch.float64, device=gpu)
        p = t.data_ptr() + G
        live[p] = (t, int(nbytes))
        return p

    def _free(ptr, nbytes, device, user):
        t, n = live.pop(ptr)
        torch.cuda.synchronize()
        g0, g1 = t[: G // 8], t[(G + n + 7) // 8:]
        if not (bool(torch.isnan(g0).all()) and bool(torch.isnan(g1).all())):
            bad.append(n)

    cbs = (ALLOC_FN(_alloc), FREE_FN(_free))
    for n in (32, 64, 128):
        ref = Solver(n)
        rep0, hist0, x0 = solve(ref)
        ref.close()
        S = Solver(n, allocator=cbs)
        S.vcycle(S.set_problem("mms_paper")[0])
        rep1, hist1, x1 = solve(S)
        S.close()
        assert not live and not bad, (n, bad)
        assert rep1["iterations"] == rep0["iterations"]
        assert np.array_equal(x0, x1)
