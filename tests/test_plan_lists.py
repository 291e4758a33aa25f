"""Host-logic audit of the plan's tree and lists (no GPU: plans built with host_only=1).

The list construction (near field N^C, interaction field
I^C = N^P \\ N^C; R14, R20) must cover every ordered pair of
distinct leaves exactly once: by P2P iff the leaves' ancestors at
min(level) are adjacent, otherwise by exactly one M2L between ancestors.
This is checked here by brute force over all leaf pairs.
"""
import numpy as np
import pytest

import synth

fda = pytest.importorskip("paper_1311_5202_b200.fda")


def _plan(p, **kw):
    opt = fda.fda_options_default(host_only=1, **kw)
    return fda.fda_plan_create(p.x, p.n, p.w, p.k, p.alpha, p.eps, opt)


def _audit(p, **kw):
    h = _plan(p, **kw)
    try:
        lop, lev, ijk = fda.fda_plan_export_leaves(h, p.N)
        pt, ps = fda.fda_plan_export_p2p(h)
        ml, mt, ms = fda.fda_plan_export_m2l(h)
        stats_log = fda.fda_plan_log(h)
    finally:
        fda.fda_plan_destroy(h)
    nl = lev.shape[0]
    # every point in exactly one leaf; leaves are Morton-contiguous, sizes <= N_p
    counts = np.bincount(lop, minlength=nl)
    assert counts.sum() == p.N and np.all(counts > 0)
    T, S = np.meshgrid(np.arange(nl), np.arange(nl), indexing="ij")
    T = T.ravel()
    S = S.ravel()
    keep = T != S
    T, S = T[keep], S[keep]
    m = np.minimum(lev[T], lev[S])

    def anc(idx, l):
        return ijk[idx] >> (lev[idx] - l)[:, None]

    at, as_ = anc(T, m), anc(S, m)
    adj = np.abs(at - as_).max(axis=1) <= 1
    # P2P set must equal the adjacency rule exactly
    p2p = set(zip(pt.tolist(), ps.tolist()))
    expect = set(zip(T[adj].tolist(), S[adj].tolist()))
    self_pairs = {(t, t) for t in range(nl)}
    assert p2p - self_pairs == expect
    assert self_pairs <= p2p
    # far pairs: exactly one M2L at some level l <= m between the ancestors
    L = int(lev.max()) + 1

    def enc(l, a, b):
        return ((l.astype(np.int64) * (1 << 20) + a[:, 0]) * (1 << 20) + a[:, 1]) * (1 << 20) + a[:, 2], \
               (b[:, 0] * (1 << 20) + b[:, 1]) * (1 << 20) + b[:, 2]

    mk = np.unique(np.stack(enc(ml, mt, ms), axis=1), axis=0)
    assert mk.shape[0] == ml.shape[0], "duplicate M2L pairs"
    far = ~adj
    Tf, Sf, mf = T[far], S[far], m[far]
    hits = np.zeros(Tf.shape[0], np.int64)
    mset = {tuple(r) for r in mk.tolist()}
    for l in range(L):
        ok = mf >= l
        if not ok.any():
            continue
        idx = np.nonzero(ok)[0]
        a = ijk[Tf[idx]] >> (lev[Tf[idx]] - l)[:, None]
        b = ijk[Sf[idx]] >> (lev[Sf[idx]] - l)[:, None]
        k1, k2 = enc(np.full(idx.shape[0], l), a, b)
        hits[idx] += np.array([(x, y) in mset for x, y in zip(k1.tolist(), k2.tolist())], dtype=np.int64)
    assert np.all(hits == 1), (np.bincount(hits), stats_log)
    # reciprocity of the interaction lists
    k1, k2 = enc(ml, mt, ms)
    r1, r2 = enc(ml, ms, mt)
    fwd = set(zip(k1.tolist(), k2.tolist()))
    assert all((x, y) in fwd for x, y in zip(r1.tolist(), r2.tolist()))
    return lev, ml


def test_lists_config1_lf():
    p = synth.make_problem("1")
    lev, ml = _audit(p)
    assert ml.shape[0] > 0 and lev.max() >= 2


def test_lists_hf_sphere():
    p = synth.make_problem("x", k=50.0, nu=12)        # kD = 100, HF levels above LF leaves
    lev, ml = _audit(p, hf_max_rows=1500, lowrank=0)
    assert ml.shape[0] > 0


def test_lists_spheroid_adaptive():
    nodes = synth.spheroid(10.0, 1.0, 0.35)
    x, n, w, hmax, s = synth.quadrature_cloud(nodes)
    p = synth.Problem("sph", x, n, w, 2.0, 0.5j, 1e-4, nodes, hmax, s)
    lev, ml = _audit(p, lowrank=0)
    assert len(np.unique(lev)) >= 2              # adaptive: leaves on several levels


def test_leaf_threshold_and_single_leaf():
    p = synth.make_problem("1")
    h = _plan(p, single_leaf=1)
    lop, lev, ijk = fda.fda_plan_export_leaves(h, p.N)
    fda.fda_plan_destroy(h)
    assert lev.shape[0] == 1 and np.all(lop == 0)
    h = _plan(p, leaf_size=30)
    lop, lev, ijk = fda.fda_plan_export_leaves(h, p.N)
    fda.fda_plan_destroy(h)
    assert np.bincount(lop).max() <= 30


def test_invalid_arguments():
    p = synth.make_problem("1")
    opt = fda.fda_options_default(host_only=1)
    with pytest.raises(fda.FDAError, match="INVALID_ARG"):
        fda.fda_plan_create(p.x, p.n, -p.w, p.k, p.alpha, 1e-4, opt)
    with pytest.raises(fda.FDAError, match="INVALID_ARG"):
        fda.fda_plan_create(p.x, p.n, p.w, p.k, p.alpha, 0.5, opt)
    with pytest.raises(fda.FDAError, match="INVALID_ARG"):
        fda.fda_plan_create(p.x, p.n * 2, p.w, p.k, p.alpha, 1e-4, opt)
    with pytest.raises(fda.FDAError, match="INVALID_ARG"):
        fda.fda_plan_create(p.x, p.n, p.w, 0.0, 1j, 1e-4, opt)
    x = p.x.copy()
    x[5] = x[4]
    with pytest.raises(fda.FDAError, match="COINCIDENT"):
        fda.fda_plan_create(x, p.n, p.w, p.k, p.alpha, 1e-4, opt)
