"""BM_G apply: K = G + alpha dG/dn_x (eq_gmat; the FDA of
PAPER.md:584-633, eq_gsum / eq_sump0g: single-layer S2M with E_up = G, the same translations, and the
same target operator E_dn = G + alpha dG/dn_x in L2T).  Parity through the C ABI against the oracle's
BM_G kind, same bars as BM_H: near-field-only <= 1e-12, full apply <= 1e-4."""
import numpy as np
import pytest

import oracle
import synth

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def _fda():
    from paper_1311_5202_b200 import fda
    return fda


def _run(h, phi, mask=None):
    fda = _fda()
    d_phi = torch.from_numpy(phi.view(np.float64).copy()).cuda()
    d_out = torch.empty_like(d_phi)
    if mask is None:
        fda.fda_apply(h, d_phi, d_out)
    else:
        fda.fda_apply_phases(h, mask, d_phi, d_out)
    torch.cuda.synchronize()
    return d_out.cpu().numpy().view(np.complex128).copy()


@pytest.mark.parametrize("name,nu,k", [("1", None, None), ("hf-small", 16, 50.0)])
def test_bmg_full_and_near(name, nu, k):
    fda = _fda()
    p = synth.make_problem(name) if nu is None else synth.make_problem("x", k=k, nu=nu)
    csr = p.correction(seed=3)
    phi = synth.random_phi(p.N, 5)
    opt = fda.fda_options_default(kernel=fda.FDA_KERNEL_BMG)
    h = fda.fda_plan_create(p.x, p.n, p.w, p.k, p.alpha, p.eps, opt)
    try:
        fda.fda_plan_set_correction(h, csr[0], csr[1], csr[2].view(np.float64))
        got = _run(h, phi)
        near_only = _run(h, phi, fda.FDA_PHASE_NEAR)
        near = _run(h, phi, fda.FDA_PHASE_NEAR | fda.FDA_PHASE_CORR)
        lop, lev, ijk = fda.fda_plan_export_leaves(h, p.N)
        t, s = fda.fda_plan_export_p2p(h)
    finally:
        fda.fda_plan_destroy(h)
    ref = oracle.apply_rows(p.x, p.n, p.w, p.k, p.alpha, phi, csr=csr, kind=oracle.KIND_BMG)
    order = np.argsort(lop, kind="stable")
    leaf_ptr = np.concatenate([[0], np.cumsum(np.bincount(lop, minlength=lev.shape[0]))])
    pair_ptr = np.concatenate([[0], np.cumsum(np.bincount(t, minlength=lev.shape[0]))])
    near_ref = oracle.apply_near(p.x, p.n, p.w, p.k, p.alpha, phi, leaf_ptr, order, pair_ptr, s, kind=oracle.KIND_BMG)
    assert oracle.rel_l2(near_only, near_ref) <= 1e-12
    err = oracle.rel_l2(got, ref)
    far = oracle.rel_l2(got - near, ref - near)
    print(f"BM_G {name}: N={p.N} rel_l2={err:.3e} far_only={far:.3e}")
    assert err <= 1e-4


def test_bmg_config3_rows():
    fda = _fda()
    p = synth.make_problem("3")
    csr = p.correction(seed=2024)
    phi = synth.random_phi(p.N, 2025)
    dev = torch.device("cuda", 0)
    h = fda.fda_plan_create(torch.from_numpy(p.x).to(dev), torch.from_numpy(p.n).to(dev),
                            torch.from_numpy(p.w).to(dev), p.k, p.alpha, p.eps,
                            fda.fda_options_default(kernel=fda.FDA_KERNEL_BMG))
    try:
        fda.fda_plan_set_correction(h, csr[0], csr[1], csr[2].view(np.float64))
        got = _run(h, phi)
    finally:
        fda.fda_plan_destroy(h)
    rows = synth.sample_rows(p.N, 2000, 7)
    ref = oracle.apply_rows(p.x, p.n, p.w, p.k, p.alpha, phi, rows=rows, csr=csr, kind=oracle.KIND_BMG)
    err = oracle.rel_l2(got[rows], ref)
    print(f"BM_G config 3: rel_l2={err:.3e}")
    assert err <= 1e-4
