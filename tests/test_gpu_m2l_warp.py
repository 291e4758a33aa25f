"""GPU: the warp-task low-rank M2L kernel (m2l_warp.cu) against the warp-specialised chunk kernel
(kernels.cu k_gtrans_ws, FDA_M2L_WARP=0).

Both apply eq_lrdk, y_t += U_o (V_o x_s), with the same device-built operators over the
same pairs; only the tiling and the order of the FP64 atomic additions differ, so the far fields must agree
to rounding.  The HF case has directional levels with short wedges (per-group expansion lengths), the LF case
only the non-directional levels.
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


def _far(p, phi, warp):
    fda = _fda()
    old = os.environ.get("FDA_M2L_WARP")
    os.environ["FDA_M2L_WARP"] = "1" if warp else "0"
    try:
        h = fda.fda_plan_create(_dev(p.x), _dev(p.n), _dev(p.w), p.k, p.alpha, p.eps, fda.fda_options_default())
    finally:
        if old is None:
            del os.environ["FDA_M2L_WARP"]
        else:
            os.environ["FDA_M2L_WARP"] = old
    try:
        d_phi = _dev(phi.view(np.float64))
        d_out = torch.empty_like(d_phi)
        fda.fda_apply_phases(h, fda.FDA_PHASE_FAR, d_phi, d_out)
        torch.cuda.synchronize()
    finally:
        fda.fda_plan_destroy(h)
    return d_out.cpu().numpy().view(np.complex128)


@pytest.mark.parametrize("name,nu,k", [("hf", 16, 50.0), ("lf", 16, 2.0), ("1c", 46, 200.0)])
def test_warp_task_m2l_equals_chunk_m2l(name, nu, k):
    p = synth.make_problem("x", k=k, nu=nu)
    phi = synth.random_phi(p.N, 5)
    a = _far(p, phi, True)
    b = _far(p, phi, False)
    err = oracle.rel_l2(a, b)
    print(f"{name}: N={p.N} warp-task vs chunk far field rel l2 {err:.3e}")
    assert np.isfinite(a).all()
    assert err <= 1e-12


def test_warp_task_m2l_high_ranks_eps_1e6():
    """eps = 1e-6: longer expansions and ranks up to 40 (five V row tiles) on every level; the launch must pick
    the instantiation whose RTMAX covers its largest rank."""
    p = synth.make_problem("x", k=50.0, nu=16)
    phi = synth.random_phi(p.N, 5)
    a = _far_eps(p, phi, True, 1e-6)
    b = _far_eps(p, phi, False, 1e-6)
    err = oracle.rel_l2(a, b)
    print(f"eps=1e-6 N={p.N}: warp-task vs chunk far field rel l2 {err:.3e}")
    assert err <= 1e-11


def _far_eps(p, phi, warp, eps):
    fda = _fda()
    old = os.environ.get("FDA_M2L_WARP")
    os.environ["FDA_M2L_WARP"] = "1" if warp else "0"
    try:
        h = fda.fda_plan_create(_dev(p.x), _dev(p.n), _dev(p.w), p.k, p.alpha, eps, fda.fda_options_default())
    finally:
        if old is None:
            del os.environ["FDA_M2L_WARP"]
        else:
            os.environ["FDA_M2L_WARP"] = old
    try:
        d_phi = _dev(phi.view(np.float64))
        d_out = torch.empty_like(d_phi)
        fda.fda_apply_phases(h, fda.FDA_PHASE_FAR, d_phi, d_out)
        torch.cuda.synchronize()
    finally:
        fda.fda_plan_destroy(h)
    return d_out.cpu().numpy().view(np.complex128)
