"""Host-side multi-rank logic on CPU (no GPU): the row-slab partition that
libsvk computes (svk_partition, a pure function exported by the C ABI) and the
NCCL-id bootstrap over torch.distributed, run with world_size 2 on `gloo`.

The partition rules checked here are the ones SURVEY 8(e) states: slabs of
node rows cover [0, N+1) disjointly; slabs nest across the distributed levels
(a coarse slab is the halved fine slab); every distributed slab holds at least
`agglom_rows` rows on the coarsest distributed level (so a rank's 4-row halo
always comes from its direct neighbour); coarser levels are replicated.
"""
import os
import socket

import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2401_06277_b200 import svk


def levels(n_elem, n_coarse=4):
    N, out = n_coarse, []
    while N <= n_elem:
        out.append(N)
        N *= 2
    return out


@pytest.mark.parametrize("n_elem,P,agg", [(64, 2, 8), (64, 3, 4), (64, 4, 4), (4096, 8, 64), (4096, 2, 64),
                                          (128, 2, 64), (1024, 5, 16), (6 * 256, 3, 64)])
def test_partition_rules(n_elem, P, agg):
    n_coarse = 6 if n_elem % 3 == 0 else 4
    Ns = levels(n_elem, n_coarse)
    dist_levels = [N for N in Ns[1:] if N >= agg * P] if P > 1 else []
    for N in Ns:
        slabs = [svk.partition(n_elem, n_coarse, P, r, agg, N) for r in range(P)]
        d = N in dist_levels
        assert all(s[2] == d for s in slabs)
        if not d:
            assert all((s[0], s[1]) == (0, N + 1) for s in slabs)
            continue
        assert slabs[0][0] == 0 and slabs[-1][1] == N + 1
        for a, b in zip(slabs, slabs[1:]):
            assert a[1] == b[0]
        rows = [s[1] - s[0] for s in slabs]
        assert min(rows) >= agg * (N // dist_levels[0]) >= 4
        if N != dist_levels[0]:  # nested: the coarse slab is the halved fine slab
            coarse = [svk.partition(n_elem, n_coarse, P, r, agg, N // 2) for r in range(P)]
            for f, c in zip(slabs, coarse):
                assert f[0] == 2 * c[0]
                assert f[1] == (N + 1 if c[1] == N // 2 + 1 else 2 * c[1])
    if dist_levels:
        Nla = dist_levels[0]
        rows = [svk.partition(n_elem, n_coarse, P, r, agg, Nla) for r in range(P)]
        assert min(s[1] - s[0] for s in rows) >= agg


def test_partition_errors():
    with pytest.raises(svk.SvkError):
        svk.partition(64, 4, 2, 2, 8, 64)      # rank out of range
    with pytest.raises(svk.SvkError):
        svk.partition(64, 4, 2, 0, 2, 64)      # agglom_rows below the halo depth
    with pytest.raises(svk.SvkError):
        svk.partition(64, 4, 2, 0, 8, 48)      # not a level of the hierarchy
    with pytest.raises(svk.SvkError):
        svk.partition(96, 4, 2, 0, 8, 96)      # n_elem not n_coarse * 2^k


def test_nccl_unique_id_shape():
    a, b = svk.nccl_unique_id(), svk.nccl_unique_id()
    assert len(a) == 128 and len(b) == 128 and a != b


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        nid = svk.nccl_id_broadcast()
        n_elem, agg = 256, 16
        mine = {N: svk.partition(n_elem, 4, world, rank, agg, N) for N in levels(n_elem)}
        allp = [None] * world
        dist.all_gather_object(allp, mine)
        ids = [None] * world
        dist.all_gather_object(ids, nid)
        q.put((rank, ids, allp))
    finally:
        dist.destroy_process_group()


def test_gloo_bootstrap_world2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    out = [q.get(timeout=120) for _ in ps]
    for p in ps:
        p.join(60)
        assert p.exitcode == 0
    for rank, ids, allp in out:
        assert len(ids[0]) == 128 and ids[0] == ids[1]  # every rank got rank 0's id
        for N, (r0, r1, d) in allp[0].items():
            s1 = allp[1][N]
            if d:
                assert r0 == 0 and r1 == s1[0] and s1[1] == N + 1
            else:
                assert (r0, r1) == (0, N + 1) == (s1[0], s1[1])
