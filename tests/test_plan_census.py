"""HF directional sets (row a-P3, R16) on CPU through host-only plans.

* fig_rankm2l census: at the finest HF level with w = lambda and eps = 1e-4 the paper finds s = 38
  (PAPER.md:742-745).  With the selection tolerance set to the paper's eps (eps_internal = 1e-4) the
  plan's padded expansion length s (the largest wedge) must be 38 +- 20%.
* every wedge's expansion reproduces held-out far fields (random sources in the cube, random points of the
  wedge's far target boxes) to within 20 eps_int (logged per level by the plan);
* a selection from too few sample rows misses it and the plan reports FDA_ERR_SETUP_ACCURACY.
"""
import re

import pytest

import synth

fda = pytest.importorskip("paper_1311_5202_b200.fda")


def _hf_lines(p, **kw):
    h = fda.fda_plan_create(p.x, p.n, p.w, p.k, p.alpha, 1e-4, fda.fda_options_default(host_only=1, verbose=1, **kw))
    try:
        return [l for l in fda.fda_plan_log(h).splitlines() if "HF m=" in l]
    finally:
        fda.fda_plan_destroy(h)


def test_census_s38_at_w_equal_lambda():
    p = synth.make_problem("x", k=25.2, nu=16)       # level 3: w = 0.25 = 1.003 lambda, the finest HF level
    lines = _hf_lines(p, eps_internal=1e-4)
    assert len(lines) == 1 and lines[0].startswith("level 3 HF")
    s = int(re.search(r" s=(\d+)", lines[0]).group(1))
    print(lines[0])
    assert 0.8 * 38 <= s <= 1.2 * 38


def test_held_out_errors_within_tolerance():
    p = synth.make_problem("x", k=25.2, nu=16)
    for line in _hf_lines(p):                          # default eps_int = eps / 100 = 1e-6
        err = float(re.search(r"held-out error max ([0-9.eE+-]+)", line).group(1))
        assert 0 < err <= 20 * 1e-6, line


def test_setup_accuracy_reported():
    p = synth.make_problem("x", k=25.2, nu=16)
    with pytest.raises(fda.FDAError, match="SETUP_ACCURACY"):
        fda.fda_plan_create(p.x, p.n, p.w, p.k, p.alpha, 1e-4, fda.fda_options_default(host_only=1, hf_max_rows=30))
