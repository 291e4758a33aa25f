"""fda_options.deterministic: bit-reproducible applies.  Every translation runs
as owned items (plain read-modify-write in a fixed order instead of FP64 reductions) and the P2P one-sided; the
result equals the default apply to rounding and the oracle within the usual bar."""
import numpy as np
import pytest

import oracle
import synth

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def _applies(fda, p, csr, phi, opt, count):
    h = fda.fda_plan_create(p.x, p.n, p.w, p.k, p.alpha, p.eps, opt)
    try:
        fda.fda_plan_set_correction(h, csr[0], csr[1], csr[2].view(np.float64))
        d_phi = torch.from_numpy(phi.view(np.float64).copy()).cuda()
        outs = []
        for _ in range(count):
            d_out = torch.empty_like(d_phi)
            fda.fda_apply(h, d_phi, d_out)
            torch.cuda.synchronize()
            outs.append(d_out.cpu().numpy().view(np.complex128).copy())
    finally:
        fda.fda_plan_destroy(h)
    return outs


@pytest.mark.parametrize("name,nu,k", [("1", None, None), ("hf-small", 16, 50.0), ("1b", None, None)])
def test_deterministic_applies_are_bit_identical(name, nu, k):
    from paper_1311_5202_b200 import fda
    p = synth.make_problem(name) if nu is None else synth.make_problem("x", k=k, nu=nu)
    csr = p.correction(seed=3)
    phi = synth.random_phi(p.N, 5)
    det = _applies(fda, p, csr, phi, fda.fda_options_default(deterministic=1), 4)   # the 2nd+ replay the CUDA graph
    for o in det[1:]:
        assert np.array_equal(det[0], o)
    det2 = _applies(fda, p, csr, phi, fda.fda_options_default(deterministic=1, graph=0), 2)   # a second plan
    assert np.array_equal(det[0], det2[0]) and np.array_equal(det2[0], det2[1])
    ref = _applies(fda, p, csr, phi, fda.fda_options_default(), 1)[0]
    d = oracle.rel_l2(det[0], ref)
    print(f"deterministic vs default ({name}, N={p.N}): {d:.2e}")
    assert d <= 1e-13
    if p.N <= 4000:
        full = oracle.apply_rows(p.x, p.n, p.w, p.k, p.alpha, phi, csr=csr)
        assert oracle.rel_l2(det[0], full) <= 1e-4
