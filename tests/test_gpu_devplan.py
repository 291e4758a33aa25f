"""The device plan builder against the host builder (rows a-P0, a-P1, a-P3 of SURVEY.md §8(a)).

* P0 / P1 (tree_dev.cu: validation, Morton keys, stable radix sort, octree level by level) must give the
  host builder's tree exactly: the same leaf of every point, leaf levels and cube indices, and the same
  P2P leaf pairs and M2L cube pairs (integer work: bit-exact).  FDA_HOST_TREE=1 selects the host P0 / P1.
* P3 (plan_dev.cu: K~, its low-rank factors, M2M / L2L, the HF directional sets) against the host linear
  algebra (FDA_HOST_OPS=1): the same low-rank / dense decisions and ranks up to a few groups at the
  truncation boundary, and applies that agree to the accuracy of the method (both are ~1e-5 from the oracle).
* P2 (lists_dev.cu: P2P lists, interaction lists grouped by offset, slots) against the host lists
  (FDA_HOST_LISTS=1): the same pairs and slots.
* Invalid inputs and coincident points are rejected by the device P0 as by the host one.
"""
import os

import numpy as np
import pytest

import oracle
import synth

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def _fda():
    from paper_1311_5202_b200 import fda
    return fda


def _dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def _plan(p, env=None, **kw):
    fda = _fda()
    old = {k: os.environ.get(k) for k in (env or {})}
    os.environ.update(env or {})
    try:
        return fda.fda_plan_create(_dev(p.x), _dev(p.n), _dev(p.w), p.k, p.alpha, p.eps,
                                   fda.fda_options_default(**kw) if kw else None)
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v


def _apply(h, phi):
    fda = _fda()
    d_phi = _dev(phi.view(np.float64))
    d_out = torch.empty_like(d_phi)
    fda.fda_apply(h, d_phi, d_out)
    return d_out.cpu().numpy().view(np.complex128).copy()


@pytest.mark.parametrize("name,nu,k", [("hf", 16, 50.0), ("lf", 12, 2.0), ("cfg3", None, None)])
def test_device_tree_equals_host_tree(name, nu, k):
    fda = _fda()
    p = synth.make_problem("3") if name == "cfg3" else synth.make_problem("x", k=k, nu=nu)
    hd = _plan(p)
    hh = _plan(p, env={"FDA_HOST_TREE": "1"})
    try:
        a, b = fda.fda_plan_export_leaves(hd, p.N), fda.fda_plan_export_leaves(hh, p.N)
        for x, y in zip(a, b):
            assert np.array_equal(x, y)
        assert all(np.array_equal(x, y) for x, y in zip(fda.fda_plan_export_p2p(hd), fda.fda_plan_export_p2p(hh)))
        assert all(np.array_equal(x, y) for x, y in zip(fda.fda_plan_export_m2l(hd), fda.fda_plan_export_m2l(hh)))
        phi = synth.random_phi(p.N, 3)
        assert oracle.rel_l2(_apply(hd, phi), _apply(hh, phi)) <= 1e-13
    finally:
        fda.fda_plan_destroy(hd)
        fda.fda_plan_destroy(hh)


@pytest.mark.parametrize("name,nu,k", [("hf", 16, 50.0), ("lf", 12, 2.0), ("cfg3", None, None), ("cfg1c", None, None)])
def test_device_lists_equal_host_lists(name, nu, k):
    """P2 (lists_dev.cu) against the host lists (FDA_HOST_LISTS=1): the same P2P leaf pairs (arrays equal),
    the same M2L cube pairs with the same offsets (as sets: the order of equal-target pairs inside a group
    may differ), the same slot counts, and applies equal to rounding."""
    fda = _fda()
    p = synth.make_problem(name[3:]) if name.startswith("cfg") else synth.make_problem("x", k=k, nu=nu)
    hd = _plan(p)
    hh = _plan(p, env={"FDA_HOST_LISTS": "1"})
    try:
        for x, y in zip(fda.fda_plan_export_p2p(hd), fda.fda_plan_export_p2p(hh)):
            assert np.array_equal(x, y)
        md, mh = fda.fda_plan_export_m2l(hd), fda.fda_plan_export_m2l(hh)
        key = lambda m: np.lexsort(np.column_stack([m[0], m[1], m[2]]).T)  # noqa: E731
        kd, kh = key(md), key(mh)
        for x, y in zip(md, mh):
            assert np.array_equal(x[kd], y[kh])
        sd, sh = fda.fda_plan_stats(hd), fda.fda_plan_stats(hh)
        for f in ("m2l_pairs", "m2l_groups", "out_slots", "in_slots", "p2p_point_pairs", "lmin"):
            assert sd[f] == sh[f], f
        phi = synth.random_phi(p.N, 7)
        assert oracle.rel_l2(_apply(hd, phi), _apply(hh, phi)) <= 1e-13
    finally:
        fda.fda_plan_destroy(hd)
        fda.fda_plan_destroy(hh)


@pytest.mark.parametrize("name,nu,k", [("hf", 16, 50.0), ("lf", 16, 2.0)])
def test_device_operators_vs_host_operators(name, nu, k):
    fda = _fda()
    p = synth.make_problem("x", k=k, nu=nu)
    phi = synth.random_phi(p.N, 4)
    hd = _plan(p)
    hh = _plan(p, env={"FDA_HOST_OPS": "1"})
    try:
        sd, sh = fda.fda_plan_stats(hd), fda.fda_plan_stats(hh)
        od, oh = _apply(hd, phi), _apply(hh, phi)
    finally:
        fda.fda_plan_destroy(hd)
        fda.fda_plan_destroy(hh)
    ref = oracle.apply_rows(p.x, p.n, p.w, p.k, p.alpha, phi)
    ed, eh = oracle.rel_l2(od, ref), oracle.rel_l2(oh, ref)
    print(f"{name}: device ops {ed:.3e}, host ops {eh:.3e}, between {oracle.rel_l2(od, oh):.3e}; "
          f"m2l flops {sd['flops_m2l']:.4g} vs {sh['flops_m2l']:.4g}, low-rank groups "
          f"{sd['m2l_lowrank_groups']} vs {sh['m2l_lowrank_groups']}")
    assert sd["m2l_groups"] == sh["m2l_groups"] and sd["m2l_pairs"] == sh["m2l_pairs"]
    assert abs(sd["m2l_lowrank_groups"] - sh["m2l_lowrank_groups"]) <= max(2, sd["m2l_groups"] // 100)
    assert abs(sd["flops_m2l"] / sh["flops_m2l"] - 1) <= 0.02
    assert ed <= 1e-4 and eh <= 1e-4
    assert ed <= 1.5 * eh + 1e-6


def test_device_p0_rejects_bad_inputs():
    fda = _fda()
    p = synth.make_problem("x", k=5.0, nu=6)
    bad_w = p.w.copy()
    bad_w[7] = -1.0
    with pytest.raises(fda.FDAError, match="INVALID_ARG"):
        fda.fda_plan_create(_dev(p.x), _dev(p.n), _dev(bad_w), p.k, p.alpha, p.eps)
    bad_n = p.n.copy()
    bad_n[3] *= 1.001
    with pytest.raises(fda.FDAError, match="INVALID_ARG"):
        fda.fda_plan_create(_dev(p.x), _dev(bad_n), _dev(p.w), p.k, p.alpha, p.eps)
    bad_x = p.x.copy()
    bad_x[11, 1] = np.nan
    with pytest.raises(fda.FDAError, match="INVALID_ARG"):
        fda.fda_plan_create(_dev(bad_x), _dev(p.n), _dev(p.w), p.k, p.alpha, p.eps)
    dup = p.x.copy()
    dup[20] = dup[19]
    with pytest.raises(fda.FDAError, match="COINCIDENT"):
        fda.fda_plan_create(_dev(dup), _dev(p.n), _dev(p.w), p.k, p.alpha, p.eps)
