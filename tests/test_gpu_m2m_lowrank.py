"""GPU: low-rank LF -> HF transition operators (FDA_M2M_LR, R27) against the dense ones.

The M2M operator from a child cube's LF expansion into a parent wedge, and its transpose (L2L), are compressed as
the M2L's K~ is (truncated SVD, sigma_i < eps sigma_1, low rank iff 2 r < s); the far field must
stay within the apply's accuracy (north_star: full apply <= 1e-4 against the direct sum).
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


def _run(p, phi, lr, csr=None, kernel=0):
    fda = _fda()
    old = os.environ.get("FDA_M2M_LR")
    os.environ["FDA_M2M_LR"] = lr
    try:
        h = fda.fda_plan_create(_dev(p.x), _dev(p.n), _dev(p.w), p.k, p.alpha, p.eps,
                                fda.fda_options_default(verbose=1, kernel=kernel))
    finally:
        if old is None:
            del os.environ["FDA_M2M_LR"]
        else:
            os.environ["FDA_M2M_LR"] = old
    try:
        if csr is not None:
            fda.fda_plan_set_correction(h, csr[0], csr[1], csr[2].view(np.float64))
        d_phi = _dev(phi.view(np.float64))
        d_out = torch.empty_like(d_phi)
        fda.fda_apply_phases(h, fda.FDA_PHASE_FAR, d_phi, d_out)
        far = d_out.cpu().numpy().view(np.complex128).copy()
        fda.fda_apply(h, d_phi, d_out)
        full = d_out.cpu().numpy().view(np.complex128).copy()
        log = fda.fda_plan_log(h)
        st = fda.fda_plan_stats(h)
    finally:
        fda.fda_plan_destroy(h)
    return far, full, log, st


@pytest.mark.parametrize("kernel", [0, 1])
def test_lowrank_transitions_match_dense(kernel):
    p = synth.make_problem("x", k=50.0, nu=24)
    phi = synth.random_phi(p.N, 21)
    csr = p.correction(4)
    far_d, full_d, log_d, st_d = _run(p, phi, "0", csr, kernel)
    far_l, full_l, log_l, st_l = _run(p, phi, "0.1", csr, kernel)
    assert "low rank (s" not in log_d
    assert "low rank (s" in log_l, "no LF -> HF transition was compressed"
    d = oracle.rel_l2(far_l, far_d)
    rows = synth.sample_rows(p.N, 300, 3)
    ref = oracle.apply_rows(p.x, p.n, p.w, p.k, p.alpha, phi, rows=rows, csr=csr,
                            kind=oracle.KIND_BMG if kernel else oracle.KIND_BMH)
    e_d, e_l = oracle.rel_l2(full_d[rows], ref), oracle.rel_l2(full_l[rows], ref)
    print(f"N={p.N} kernel={kernel}: far field low-rank vs dense {d:.2e}; full vs oracle dense {e_d:.2e} low-rank "
          f"{e_l:.2e}; M2M flops {st_d['flops_m2m']:.3e} -> {st_l['flops_m2m']:.3e}")
    assert d <= 1e-4
    assert e_l <= 1e-4
    assert e_l <= 2 * e_d + 1e-6
    assert st_l["flops_m2m"] < st_d["flops_m2m"]
