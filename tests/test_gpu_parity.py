"""GPU parity: the CUDA path through the C ABI against the CPU oracle.

Tolerances (BASELINE.json north_star):
  * near-field-only sums (P2P over the plan's exact leaf pairs): <= 1e-12 relative l2
  * correction CSR alone: <= 1e-13 relative l2 (exact up to summation order)
  * single-leaf plan (whole operator by P2P): <= 1e-12
  * full FDA apply at eps = 1e-4: <= 1e-4 relative l2 (full rows, or 2000 seeded rows)
"""
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


def _run(plan, phi, mask=None):
    fda = _fda()
    d_phi = _dev(phi.view(np.float64))
    d_out = torch.empty_like(d_phi)
    if mask is None:
        fda.fda_apply(plan, d_phi, d_out)
    else:
        fda.fda_apply_phases(plan, mask, d_phi, d_out)
    torch.cuda.synchronize()
    return d_out.cpu().numpy().view(np.complex128)


def _plan(p, **kw):
    fda = _fda()
    opt = fda.fda_options_default(**kw) if kw else None
    return fda.fda_plan_create(_dev(p.x), _dev(p.n), _dev(p.w), p.k, p.alpha, p.eps, opt)


@pytest.fixture(scope="module")
def cfg1():
    p = synth.make_problem("1")
    csr = p.correction(seed=5)
    phi = synth.random_phi(p.N, 11)
    ref = oracle.apply_rows(p.x, p.n, p.w, p.k, p.alpha, phi, csr=csr)
    return p, csr, phi, ref


def test_near_only_matches_oracle_pairs(cfg1):
    fda = _fda()
    p, csr, phi, ref = cfg1
    h = _plan(p)
    try:
        got = _run(h, phi, fda.FDA_PHASE_NEAR)
        lop, lev, ijk = fda.fda_plan_export_leaves(h, p.N)
        t, s = fda.fda_plan_export_p2p(h)
    finally:
        fda.fda_plan_destroy(h)
    order = np.argsort(lop, kind="stable")
    leaf_ptr = np.concatenate([[0], np.cumsum(np.bincount(lop, minlength=lev.shape[0]))])
    pair_ptr = np.concatenate([[0], np.cumsum(np.bincount(t, minlength=lev.shape[0]))])
    near = oracle.apply_near(p.x, p.n, p.w, p.k, p.alpha, phi, leaf_ptr, order, pair_ptr, s)
    err = oracle.rel_l2(got, near)
    assert err <= 1e-12, err


def test_csr_only(cfg1):
    import scipy.sparse as sp
    fda = _fda()
    p, csr, phi, ref = cfg1
    h = _plan(p)
    try:
        fda.fda_plan_set_correction(h, _dev(csr[0]), _dev(csr[1]), _dev(csr[2].view(np.float64)))
        got = _run(h, phi, fda.FDA_PHASE_CORR)
    finally:
        fda.fda_plan_destroy(h)
    expect = sp.csr_matrix((csr[2], csr[1], csr[0]), shape=(p.N, p.N)) @ phi
    assert oracle.rel_l2(got, expect) <= 1e-13


def test_single_leaf_equals_direct_sum(cfg1):
    fda = _fda()
    p, csr, phi, ref = cfg1
    h = _plan(p, single_leaf=1)
    try:
        fda.fda_plan_set_correction(h, _dev(csr[0]), _dev(csr[1]), _dev(csr[2].view(np.float64)))
        got = _run(h, phi)
    finally:
        fda.fda_plan_destroy(h)
    assert oracle.rel_l2(got, ref) <= 1e-12


def test_full_apply_config1(cfg1):
    fda = _fda()
    p, csr, phi, ref = cfg1
    h = _plan(p)
    try:
        fda.fda_plan_set_correction(h, _dev(csr[0]), _dev(csr[1]), _dev(csr[2].view(np.float64)))
        got = _run(h, phi)
        near = _run(h, phi, fda.FDA_PHASE_NEAR | fda.FDA_PHASE_CORR)
    finally:
        fda.fda_plan_destroy(h)
    err = oracle.rel_l2(got, ref)
    far_err = oracle.rel_l2(got - near, ref - near)
    print(f"config 1: rel l2 {err:.3e}  far-only {far_err:.3e}")
    assert err <= 1e-4
    assert far_err <= 1e-3


def test_host_pointers_and_linearity(cfg1):
    fda = _fda()
    p, csr, phi, ref = cfg1
    h = _plan(p)
    try:
        fda.fda_plan_set_correction(h, csr[0], csr[1], csr[2].view(np.float64))
        out_h = np.empty_like(phi)
        fda.fda_apply(h, phi.view(np.float64), out_h.view(np.float64))
        out_d = _run(h, phi)
        # M2L items with few pairs per group accumulate with FP64 atomics: summation order (and so
        # the last bits) may differ between applies; identical to rounding.
        assert oracle.rel_l2(out_h, out_d) <= 1e-14
        phi2 = synth.random_phi(p.N, 12)
        a = _run(h, phi)
        b = _run(h, phi2)
        c = _run(h, 2.0 * phi - 3j * phi2)
        assert oracle.rel_l2(c, 2.0 * a - 3j * b) <= 1e-13
        z = _run(h, np.zeros_like(phi))
        assert np.all(z == 0)
        with pytest.raises(fda.FDAError, match="ALIAS"):
            t = _dev(phi.view(np.float64))
            fda.fda_apply(h, t, t)
    finally:
        fda.fda_plan_destroy(h)


@pytest.mark.parametrize("name,nu,k,opts", [("hf-small", 16, 50.0, {}), ("lf-small", 16, 2.0, {}),
                                           # p = 10: 488 surface points (> one check-point block of k_s2m_check)
                                           ("lf-p10", 16, 2.0, {"lf_p_low": 10, "lf_p_high": 10})])
def test_full_apply_full_oracle(name, nu, k, opts):
    fda = _fda()
    p = synth.make_problem("x", k=k, nu=nu)
    csr = p.correction(seed=3)
    phi = synth.random_phi(p.N, 5)
    ref = oracle.apply_rows(p.x, p.n, p.w, p.k, p.alpha, phi, csr=csr)
    h = _plan(p, verbose=1, **opts)
    try:
        fda.fda_plan_set_correction(h, _dev(csr[0]), _dev(csr[1]), _dev(csr[2].view(np.float64)))
        got = _run(h, phi)
        near = _run(h, phi, fda.FDA_PHASE_NEAR | fda.FDA_PHASE_CORR)
        print(fda.fda_plan_log(h))
    finally:
        fda.fda_plan_destroy(h)
    err = oracle.rel_l2(got, ref)
    far_err = oracle.rel_l2(got - near, ref - near)
    print(f"{name}: N={p.N} rel l2 {err:.3e}  far-only {far_err:.3e}")
    assert err <= 1e-4


@pytest.mark.parametrize("nu,k", [(8, 5.0), (24, 50.0)])
def test_symmetric_p2p_equals_one_sided_p2p(nu, k):
    """The symmetric P2P (kernels.cu k_p2p_sym: each leaf pair once, K_ij and K_ji from one evaluation of r and
    e^{ikr}) against the one-sided kernel (FDA_P2P_SYM=0) and against oracle_near on the plan's leaf pairs."""
    import os
    fda = _fda()
    p = synth.make_problem("x", k=k, nu=nu)
    phi = synth.random_phi(p.N, 3)
    h = _plan(p)
    try:
        sym = _run(h, phi, fda.FDA_PHASE_NEAR)
        os.environ["FDA_P2P_SYM"] = "0"
        try:
            one = _run(h, phi, fda.FDA_PHASE_NEAR)
        finally:
            del os.environ["FDA_P2P_SYM"]
        lop, lev, ijk = fda.fda_plan_export_leaves(h, p.N)
        t, s = fda.fda_plan_export_p2p(h)
    finally:
        fda.fda_plan_destroy(h)
    err = oracle.rel_l2(sym, one)
    order = np.argsort(lop, kind="stable")
    leaf_ptr = np.concatenate([[0], np.cumsum(np.bincount(lop, minlength=lev.shape[0]))])
    pair_ptr = np.concatenate([[0], np.cumsum(np.bincount(t, minlength=lev.shape[0]))])
    ref = oracle.apply_near(p.x, p.n, p.w, p.k, p.alpha, phi, leaf_ptr, order, pair_ptr, s)
    print(f"N={p.N}: symmetric vs one-sided P2P {err:.3e}, vs oracle_near {oracle.rel_l2(sym, ref):.3e}")
    assert err <= 1e-13
    assert oracle.rel_l2(sym, ref) <= 1e-12
