"""Multi-rank (N > 1) path on CPU: gloo, world_size 2.

bench.py's N-GPU step: every rank builds the same plan with (rank, nranks), applies it to its
owned Morton range of leaves (rows outside the range are zero), and one all-reduce of `out`
assembles the result.  Here the device apply is replaced by the oracle evaluated on exactly the
rows each rank owns (the ownership comes from the library's host-only plan), so the test checks
what the multi-rank path relies on:
  * the owned leaf ranges of the ranks partition the leaves (every row owned exactly once),
  * owned ranges are contiguous in Morton order and balanced by points,
  * the all-reduce of the rank-local outputs equals the single-rank result bit for bit.
"""
import os
import socket

import numpy as np
import pytest

import oracle
import synth

torch = pytest.importorskip("torch")
fda = pytest.importorskip("paper_1311_5202_b200.fda")


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        p = synth.make_problem("x", k=3.0, nu=6)
        csr = p.correction(seed=3)
        phi = synth.random_phi(p.N, 4)
        opt = fda.fda_options_default(host_only=1, rank=rank, nranks=world, leaf_size=30)
        h = fda.fda_plan_create(p.x, p.n, p.w, p.k, p.alpha, p.eps, opt)
        st = fda.fda_plan_stats(h)
        lop, lev, ijk = fda.fda_plan_export_leaves(h, p.N)
        fda.fda_plan_destroy(h)
        lb, le = st["owned_leaf_begin"], st["owned_leaf_end"]
        rows = np.nonzero((lop >= lb) & (lop < le))[0].astype(np.int64)
        assert rows.shape[0] == st["owned_end"] - st["owned_begin"]
        out = np.zeros(p.N, dtype=np.complex128)
        if rows.shape[0]:
            out[rows] = oracle.apply_rows(p.x, p.n, p.w, p.k, p.alpha, phi, rows=rows, csr=csr)
        t = torch.from_numpy(out.view(np.float64).copy())
        dist.all_reduce(t)                       # the assembly bench.py does over NCCL
        cnt = torch.zeros(p.N, dtype=torch.int64)
        cnt[torch.from_numpy(rows)] = 1
        dist.all_reduce(cnt)
        rng = torch.tensor([lb, le, st["owned_begin"], st["owned_end"]], dtype=torch.int64)
        allr = [torch.zeros_like(rng) for _ in range(world)]
        dist.all_gather(allr, rng)
        if rank == 0:
            full = oracle.apply_rows(p.x, p.n, p.w, p.k, p.alpha, phi, csr=csr)
            q.put({"equal": bool(np.array_equal(t.numpy().view(np.complex128), full)),
                   "cnt_ok": bool(torch.all(cnt == 1)), "ranges": [r.tolist() for r in allr], "N": p.N,
                   "nleaves": int(lev.shape[0])})
    finally:
        dist.destroy_process_group()


def test_two_rank_partition_and_assembly():
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.SimpleQueue()
    port = _free_port()
    mp.spawn(_worker, args=(2, port, q), nprocs=2, join=True)
    res = q.get()
    assert res["cnt_ok"], "every row owned by exactly one rank"
    assert res["equal"], "all-reduce of rank-local rows equals the single-rank result"
    (lb0, le0, pb0, pe0), (lb1, le1, pb1, pe1) = res["ranges"]
    assert lb0 == 0 and le0 == lb1 and le1 == res["nleaves"]       # contiguous Morton leaf ranges
    assert pb0 == 0 and pe0 == pb1 and pe1 == res["N"]
    assert abs(pe0 - res["N"] / 2) <= 60                            # balanced by points (leaf <= N_p)
