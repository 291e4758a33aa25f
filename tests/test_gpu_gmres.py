"""Device GMRES around the FDA apply.  Plane-wave right-hand
side b_i = e^{i k x_i . d} (PAPER.md:1043-1048 incidence); the operator is the plan's BM_H apply with
the synthetic correction (whose diagonal carries the free term 1/2).  Checks that the
residual reaches the tolerance and that the solution solves the oracle's operator to the accuracy of
the apply."""
import numpy as np
import pytest

import oracle
import synth

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def test_gmres_config1():
    from paper_1311_5202_b200 import fda
    from paper_1311_5202_b200.gmres import gmres
    p = synth.make_problem("1")
    csr = p.correction(seed=5)
    d = np.array([0.0, 0.6, 0.8])
    b = np.exp(1j * p.k * (p.x @ d))
    plan = fda.Plan(p.x, p.n, p.w, p.k, p.alpha, p.eps)
    try:
        plan.set_correction(csr[0], csr[1], csr[2].view(np.float64))
        x, hist, napply = gmres(plan.h, torch.from_numpy(b).cuda(), tol=1e-7, restart=60, maxiter=600)
    finally:
        plan.close()
    xs = x.cpu().numpy()
    res = oracle.rel_l2(oracle.apply_rows(p.x, p.n, p.w, p.k, p.alpha, xs, csr=csr), b)
    print(f"GMRES config 1: {napply} applies, final residual {hist[-1]:.2e}, oracle residual {res:.2e}")
    assert hist[-1] <= 1e-6
    assert res <= 1e-3
