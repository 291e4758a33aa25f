"""Multi-rank (N > 1) host logic on CPU: gloo, world_size 2 and 4.

Every rank builds the library's host-only plan with (rank, nranks) and exports its ownership and its
expansion-exchange lists.  Checked against an independent computation from the exported tree and M2L
pairs (fda_plan_export_leaves / fda_plan_export_m2l), with the lists of all ranks gathered over gloo:
  * the ranks' owned leaf ranges are contiguous in Morton order and partition the leaves;
  * what rank q sends to rank r is, entry for entry and in order, what r expects from q;
  * rank r receives exactly the source cubes its M2L reads (pairs whose target cube holds points of r)
    that hold points of another rank, and it receives such a cube from every other rank holding points
    of it, and from no rank that holds none (the partial sums of DESIGN.md §7b).
"""
import os
import socket

import numpy as np
import pytest

import synth

torch = pytest.importorskip("torch")
fda = pytest.importorskip("paper_1311_5202_b200.fda")


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _cube_ranks(lev, ijk, ranges):
    """(level, cube ijk) -> set of ranks whose owned leaves lie in the cube (from the exported leaves)."""
    owner = {}
    for q, (lb, le) in enumerate(ranges):
        for t in range(lb, le):
            for l in range(int(lev[t]) + 1):
                key = (l,) + tuple(int(v) >> (int(lev[t]) - l) for v in ijk[t])
                owner.setdefault(key, set()).add(q)
    return owner


def _worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        p = synth.make_problem("x", k=20.0, nu=10)            # HF and LF levels, N = 4800
        opt = fda.fda_options_default(host_only=1, rank=rank, nranks=world, leaf_size=30)
        h = fda.fda_plan_create(p.x, p.n, p.w, p.k, p.alpha, p.eps, opt)
        st = fda.fda_plan_stats(h)
        lop, lev, ijk = fda.fda_plan_export_leaves(h, p.N)
        mlev, mt, ms = fda.fda_plan_export_m2l(h)
        lists = {(peer, rv): fda.fda_plan_export_exchange(h, peer, rv) for peer in range(world) for rv in (False, True)}
        counts = fda.fda_dist_counts(h, world)
        fda.fda_plan_destroy(h)
        allr = [None] * world
        dist.all_gather_object(allr, (st["owned_leaf_begin"], st["owned_leaf_end"], st["owned_begin"], st["owned_end"]))
        all_lists = [None] * world
        dist.all_gather_object(all_lists, {k: tuple(a.tolist() for a in v) for k, v in lists.items()})
        res = {"rank": rank, "ranges": allr, "nleaves": int(lev.shape[0]), "N": p.N, "errors": []}
        err = res["errors"]
        ranges = [(a, b) for a, b, _, _ in allr]
        owner = _cube_ranks(lev, ijk, ranges)
        # send / receive symmetry with every peer
        for peer in range(world):
            if peer == rank:
                continue
            mine = all_lists[rank][(peer, True)]          # what I receive from peer
            theirs = all_lists[peer][(rank, False)]       # what peer sends me
            if mine != theirs:
                err.append(f"recv {rank}<-{peer} differs from send {peer}->{rank}")
        # what I need: source cubes of the M2L pairs whose target cube holds my points, held by another rank
        need = set()
        for l, t, s in zip(mlev.tolist(), mt.tolist(), ms.tolist()):
            if rank in owner.get((l,) + tuple(t), ()):
                for qq in owner.get((l,) + tuple(s), ()):
                    if qq != rank:
                        need.add((qq, l) + tuple(s))
        got = set()
        for peer in range(world):
            lv_, _, cj = lists[(peer, True)]
            for l, c in zip(lv_.tolist(), cj.tolist()):
                got.add((peer, l) + tuple(c))
                if peer not in owner.get((l,) + tuple(c), ()):
                    err.append(f"rank {rank} receives cube {(l, c)} from {peer}, which holds none of its points")
        if got != need:
            err.append(f"rank {rank}: received {len(got)} (peer, cube) entries, needs {len(need)}; "
                       f"missing {len(need - got)}, extra {len(got - need)}")
        res["nrecv"] = int(counts[1].sum())
        res["nsend"] = int(counts[0].sum())
        q.put(res)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_exchange_lists_and_partition(world):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.SimpleQueue()
    port = _free_port()
    mp.spawn(_worker, args=(world, port, q), nprocs=world, join=True)
    res = [q.get() for _ in range(world)]
    for r in res:
        assert not r["errors"], r["errors"]
    r0 = res[0]
    ranges = r0["ranges"]
    assert ranges[0][0] == 0 and ranges[-1][1] == r0["nleaves"]
    for a, b in zip(ranges, ranges[1:]):
        assert a[1] == b[0] and a[3] == b[2]               # contiguous Morton leaf and point ranges
    assert ranges[0][2] == 0 and ranges[-1][3] == r0["N"]
    assert all(b[1] > b[0] for b in ranges)                 # every rank owns work
    assert sum(r["nrecv"] for r in res) == sum(r["nsend"] for r in res) > 0
