"""GPU parity on the benchmark-shaped configs, through the C ABI, default plan.

* 1b (N = 49,152, kD = 100: HF level + LF levels) and 1c (N = 101,568, kD = 400: two HF levels,
  borderline w = 0.995 lambda) against the FULL O(N^2) oracle (every row);
* 2 (kD = 1, LF only), 3 (kD = 100) and 4 (10:1:1 spheroid, kD = 400) against 2000 seeded rows
  (SURVEY.md §8(c) #10), in the launch configuration bench.py times.
Bar: relative l2 <= 1e-4 over the checked rows (BASELINE.json north_star), and the far-field-only
error is reported beside it.
"""
import numpy as np
import pytest

import oracle
import synth

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def _run_cfg(name, rows=None):
    from paper_1311_5202_b200 import fda
    p = synth.make_problem(name)
    csr = p.correction(seed=2024)
    phi = synth.random_phi(p.N, 2025)
    dev = torch.device("cuda", 0)
    h = fda.fda_plan_create(torch.from_numpy(p.x).to(dev), torch.from_numpy(p.n).to(dev),
                            torch.from_numpy(p.w).to(dev), p.k, p.alpha, p.eps)
    try:
        fda.fda_plan_set_correction(h, csr[0], csr[1], csr[2].view(np.float64))
        d_phi = torch.from_numpy(phi.view(np.float64)).to(dev)
        d_out = torch.empty_like(d_phi)
        fda.fda_apply(h, d_phi, d_out)
        got = d_out.cpu().numpy().view(np.complex128).copy()
        fda.fda_apply_phases(h, fda.FDA_PHASE_NEAR | fda.FDA_PHASE_CORR, d_phi, d_out)
        near = d_out.cpu().numpy().view(np.complex128).copy()
        st = fda.fda_plan_stats(h)
    finally:
        fda.fda_plan_destroy(h)
    sel = np.arange(p.N) if rows is None else synth.sample_rows(p.N, rows, 7)
    ref = oracle.apply_rows(p.x, p.n, p.w, p.k, p.alpha, phi, rows=sel, csr=csr)
    err = oracle.rel_l2(got[sel], ref)
    far = oracle.rel_l2(got[sel] - near[sel], ref - near[sel])
    print(f"config {name}: N={p.N} kD={2 * p.k:g} rows={sel.shape[0]} rel_l2={err:.3e} far_only={far:.3e} "
          f"m2l_pairs={st['m2l_pairs']} lowrank_groups={st['m2l_lowrank_groups']}/{st['m2l_groups']}")
    return err, far, st


@pytest.mark.parametrize("name", ["1b", "1c"])
def test_full_oracle_hf_configs(name):
    err, far, st = _run_cfg(name)
    assert st["m2l_pairs"] > 0
    assert err <= 1e-4


@pytest.mark.parametrize("name", ["2", "3", "4"])
def test_sampled_rows_configs(name):
    err, far, st = _run_cfg(name, rows=2000)
    assert err <= 1e-4
