"""GPU parity on the benchmark-shaped configs, through the C ABI, default plan.

* 1b (N = 49,152, kD = 100: HF level + LF levels) and 1c (N = 101,568, kD = 400: two HF levels,
  borderline w = 0.995 lambda) against the FULL O(N^2) oracle (every row);
* 2 (kD = 1, LF only), 3 (kD = 100), 4 (10:1:1 spheroid, kD = 400) and 5 (the bench workload,
  N = 4,009,008, kD = 1000) against 2000 seeded rows, in the launch
  configuration bench.py times.
Two densities: random (Re, Im U(-1,1)) and the smooth plane wave e^{ik d.x}
(PAPER.md:1043-1048), whose far field does not cancel.
Bars (BASELINE.json north_star): relative l2 of the full apply <= 1e-4; the
far field alone ((out - near) against (oracle - near)) <= 1e-3; the largest row
error <= 1e-3 of the largest row.
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
    dens = {"random": synth.random_phi(p.N, 2025), "planewave": synth.plane_wave(p.x, p.k)}
    dev = torch.device("cuda", 0)
    sel = np.arange(p.N) if rows is None else synth.sample_rows(p.N, rows, 7)
    h = fda.fda_plan_create(torch.from_numpy(p.x).to(dev), torch.from_numpy(p.n).to(dev),
                            torch.from_numpy(p.w).to(dev), p.k, p.alpha, p.eps)
    res = {}
    try:
        fda.fda_plan_set_correction(h, csr[0], csr[1], csr[2].view(np.float64))
        st = fda.fda_plan_stats(h)
        for nm, phi in dens.items():
            d_phi = torch.from_numpy(phi.view(np.float64)).to(dev)
            d_out = torch.empty_like(d_phi)
            fda.fda_apply(h, d_phi, d_out)
            got = d_out.cpu().numpy().view(np.complex128)[sel].copy()
            fda.fda_apply_phases(h, fda.FDA_PHASE_NEAR | fda.FDA_PHASE_CORR, d_phi, d_out)
            near = d_out.cpu().numpy().view(np.complex128)[sel].copy()
            ref = oracle.apply_rows(p.x, p.n, p.w, p.k, p.alpha, phi, rows=sel, csr=csr)
            res[nm] = (oracle.rel_l2(got, ref), oracle.rel_l2(got - near, ref - near),
                       float(np.abs(got - ref).max() / np.abs(ref).max()))
            print(f"config {name} {nm}: N={p.N} kD={2 * p.k:g} rows={sel.shape[0]} rel_l2={res[nm][0]:.3e} "
                  f"far_only={res[nm][1]:.3e} max_row={res[nm][2]:.3e} m2l_pairs={st['m2l_pairs']}")
    finally:
        fda.fda_plan_destroy(h)
    return res, st


def _check(res):
    for nm, (full, far, mx) in res.items():
        assert full <= 1e-4, (nm, full)
        assert far <= 1e-3, (nm, far)
        assert mx <= 1e-3, (nm, mx)


@pytest.mark.parametrize("name", ["1b", "1c"])
def test_full_oracle_hf_configs(name):
    res, st = _run_cfg(name)
    assert st["m2l_pairs"] > 0
    _check(res)


@pytest.mark.parametrize("name", ["2", "3", "4"])
def test_sampled_rows_configs(name):
    res, st = _run_cfg(name, rows=2000)
    _check(res)


def test_sampled_rows_config5():
    """The bench workload (N = 4,009,008, kD = 1000) on 2000 seeded rows; the plan takes ~2 minutes."""
    res, st = _run_cfg("5", rows=2000)
    assert st["n"] == 4009008
    _check(res)
