"""GPU: the target-block M2L (m2l_block.cu) against the group-major atomic M2L.

Both compute eq_lrdk, y_t += U_o (V_o x_s) over the same pairs and the same
device-built operators; only the summation order differs (atomics vs block-owned shared-memory
accumulation).  The far-field-only applies must agree to rounding, and the block path must be
bitwise reproducible from apply to apply when every M2L group of the plan takes it.
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


def _far(p, phi, block):
    fda = _fda()
    old = os.environ.get("FDA_M2L_BLOCK")
    os.environ["FDA_M2L_BLOCK"] = "1" if block else "0"
    try:
        h = fda.fda_plan_create(_dev(p.x), _dev(p.n), _dev(p.w), p.k, p.alpha, p.eps,
                                fda.fda_options_default(verbose=1))
    finally:
        if old is None:
            del os.environ["FDA_M2L_BLOCK"]
        else:
            os.environ["FDA_M2L_BLOCK"] = old
    try:
        d_phi = _dev(phi.view(np.float64))
        outs = []
        for _ in range(2):
            d_out = torch.empty_like(d_phi)
            fda.fda_apply_phases(h, fda.FDA_PHASE_FAR, d_phi, d_out)
            torch.cuda.synchronize()
            outs.append(d_out.cpu().numpy().view(np.complex128))
        log = fda.fda_plan_log(h)
    finally:
        fda.fda_plan_destroy(h)
    return outs, log


@pytest.mark.parametrize("name,nu,k", [("hf", 16, 50.0), ("lf", 16, 2.0), ("1b", 32, 50.0)])
def test_block_m2l_equals_atomic_m2l(name, nu, k):
    p = synth.make_problem("x", k=k, nu=nu)
    phi = synth.random_phi(p.N, 7)
    (b1, b2), log = _far(p, phi, True)
    (a1, _), _ = _far(p, phi, False)
    print(f"{name}: N={p.N}\n" + "\n".join(ln for ln in log.splitlines() if "m2l blocks" in ln))
    assert "m2l blocks" in log
    err = oracle.rel_l2(b1, a1)
    print(f"{name}: block vs atomic far field rel l2 {err:.3e}")
    assert err <= 1e-13
    assert oracle.rel_l2(b1, b2) <= 1e-14
