"""GPU: stored leaf S2M / L2T matrices ("In the FDBEM, the S2M and L2T matrices are precomputed
and saved in memory") against the on-the-fly surface evaluations (FDA_LEAF_MATS=0).

S_leaf = (Sigma^-1 U^H) E_up and T_leaf = E_dn (conj(U) Sigma^-1) are the same products associated the other way
(eq_cmps x eq_evas2mh, eq_eval2t x eq_cmpt), so the far fields agree to rounding for every kernel kind.
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


def _far(p, phi, stored, kernel):
    fda = _fda()
    old = os.environ.get("FDA_LEAF_MATS")
    os.environ["FDA_LEAF_MATS"] = "1" if stored else "0"
    try:
        h = fda.fda_plan_create(_dev(p.x), _dev(p.n), _dev(p.w), p.k, p.alpha, p.eps,
                                fda.fda_options_default(kernel=kernel))
    finally:
        if old is None:
            del os.environ["FDA_LEAF_MATS"]
        else:
            os.environ["FDA_LEAF_MATS"] = old
    try:
        d_phi = _dev(phi.view(np.float64))
        d_out = torch.empty_like(d_phi)
        fda.fda_apply_phases(h, fda.FDA_PHASE_FAR, d_phi, d_out)
        torch.cuda.synchronize()
        st = fda.fda_plan_stats(h)
    finally:
        fda.fda_plan_destroy(h)
    return d_out.cpu().numpy().view(np.complex128), st


@pytest.mark.parametrize("kernel", [0, 1, 2])
@pytest.mark.parametrize("nu,k", [(16, 50.0), (24, 2.0)])
def test_stored_leaf_matrices_equal_surface_evaluations(nu, k, kernel):
    p = synth.make_problem("x", k=k, nu=nu)
    phi = synth.random_phi(p.N, 9)
    a, sa = _far(p, phi, True, kernel)
    b, sb = _far(p, phi, False, kernel)
    err = oracle.rel_l2(a, b)
    print(f"N={p.N} k={k} kernel={kernel}: stored vs evaluated far field {err:.3e}, matrices "
          f"{(sa['bytes_s2m'] + sa['bytes_l2t']) / 1e6:.1f} MB")
    assert sa["bytes_s2m"] > 0 and sa["s2m_evals"] == 0
    assert sb["bytes_s2m"] == 0 and sb["s2m_evals"] > 0
    assert err <= 1e-13
