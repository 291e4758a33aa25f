"""Table-1 mode: the summation p_i = sum_{j != i} [G + alpha dG/dn_y](x_i, y_j) q_j
of PAPER.md:881-884 (eq_sum) on the cube-sphere point sets of Table 1 (N = 72 m^2, ~20 points per
wavelength), unit weights, no correction (the paper's particle summation).  Parity through the C ABI
against the oracle's kind 6 over every row; the paper's own eps_a at eps = 1e-4 is 4.9e-5..3.7e-4
(PAPER.md:907-921); the bar here is the north-star 1e-4."""
import numpy as np
import pytest

import oracle
import synth

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("m,k,original", [(8, 2 * np.pi, 0), (32, 8 * np.pi, 0), (8, 2 * np.pi, 1),
                                           (32, 8 * np.pi, 1)])
def test_table1_summation(m, k, original):
    """improved FDA (original = 0) and the paper's original FDA (original = 1: unreduced equivalent-density
    expansions, dense M2L; R24): both within the north-star bar of the direct sum."""
    from paper_1311_5202_b200 import fda
    nodes = synth.cube_sphere(m)
    x, n, w, hmax, smp = synth.quadrature_cloud(nodes)
    ones = np.ones(x.shape[0])
    alpha = 1j / k
    q = synth.random_phi(x.shape[0], 17)
    h = fda.fda_plan_create(x, n, ones, k, alpha, 1e-4,
                            fda.fda_options_default(kernel=fda.FDA_KERNEL_T1, original=original))
    try:
        d_q = torch.from_numpy(q.view(np.float64).copy()).cuda()
        d_p = torch.empty_like(d_q)
        fda.fda_apply(h, d_q, d_p)
        torch.cuda.synchronize()
        got = d_p.cpu().numpy().view(np.complex128)
    finally:
        fda.fda_plan_destroy(h)
    ref = oracle.apply_rows(x, n, ones, k, alpha, q, kind=oracle.KIND_T1)
    err = oracle.rel_l2(got, ref)
    print(f"Table-1 mode m={m} N={x.shape[0]} k={k:.4g} original={original}: eps_a={err:.3e}")
    assert err <= 1e-4
