"""GPU: HF M2L operators shared by the cube symmetry (api.cu m2l_symmetry_classes) against one operator per
(offset, wedge) group (FDA_M2L_NOSHARE=1).

The wedges' point sets are rotations of their orbit representative's, so the groups
(delta, d) and (delta', d') with M_d^T delta = M_d'^T delta' and M_d^T M_t = M_d'^T M_t' have the same
K~ (eq_cmpk) and the same low-rank factors (eq_lrdk).  Sharing only changes which copy of the operator a pair
reads: the far field must agree to rounding, and the plan must store fewer operators than groups.
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


def _far(p, phi, share):
    fda = _fda()
    old = os.environ.get("FDA_M2L_NOSHARE")
    os.environ["FDA_M2L_NOSHARE"] = "0" if share else "1"
    try:
        h = fda.fda_plan_create(_dev(p.x), _dev(p.n), _dev(p.w), p.k, p.alpha, p.eps, fda.fda_options_default())
    finally:
        if old is None:
            del os.environ["FDA_M2L_NOSHARE"]
        else:
            os.environ["FDA_M2L_NOSHARE"] = old
    try:
        d_phi = _dev(phi.view(np.float64))
        d_out = torch.empty_like(d_phi)
        fda.fda_apply_phases(h, fda.FDA_PHASE_FAR, d_phi, d_out)
        torch.cuda.synchronize()
        st = fda.fda_plan_stats(h)
    finally:
        fda.fda_plan_destroy(h)
    return d_out.cpu().numpy().view(np.complex128), st


@pytest.mark.parametrize("name,nu,k", [("hf", 16, 50.0), ("1c", 46, 200.0)])
def test_shared_m2l_operators_equal_per_group_operators(name, nu, k):
    p = synth.make_problem("x", k=k, nu=nu)
    phi = synth.random_phi(p.N, 11)
    a, sa = _far(p, phi, True)
    b, sb = _far(p, phi, False)
    print(f"{name}: N={p.N} groups {sa['m2l_groups']} operators shared {sa['m2l_ops']} / unshared {sb['m2l_ops']}")
    assert sa["m2l_groups"] == sb["m2l_groups"] == sb["m2l_ops"]
    assert sa["m2l_pairs"] == sb["m2l_pairs"]
    assert sa["m2l_ops"] < sa["m2l_groups"]
    err = oracle.rel_l2(a, b)
    print(f"{name}: shared vs per-group far field rel l2 {err:.3e}")
    assert err <= 1e-12
