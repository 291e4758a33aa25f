"""GPU: the CUDA-graph apply (fda_options.graph, the default) against plain launches (graph = 0).

The graph replays the same kernels on the same plan buffers (captured on the second apply of a phase mask), so
the outputs agree to the rounding of the FP64 reductions; new phi / out pointers on every call are taken by the
permute / unpermute outside the graph; fda_plan_set_correction drops the captured graph (the new correction is
applied).  The oracle checks the full apply (north_star bar 1e-4).
"""
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


def _plan(p, graph):
    fda = _fda()
    return fda.fda_plan_create(_dev(p.x), _dev(p.n), _dev(p.w), p.k, p.alpha, p.eps,
                               fda.fda_options_default(graph=graph))


def _apply(h, phi, mask=None):
    fda = _fda()
    d_phi = _dev(phi.view(np.float64))
    d_out = torch.empty_like(d_phi)
    if mask is None:
        fda.fda_apply(h, d_phi, d_out)
    else:
        fda.fda_apply_phases(h, mask, d_phi, d_out)
    torch.cuda.synchronize()
    return d_out.cpu().numpy().view(np.complex128).copy()


@pytest.mark.parametrize("cfg", ["1", "1b"])
def test_graph_apply_equals_plain_launches(cfg):
    fda = _fda()
    p = synth.make_problem(cfg)
    csr = p.correction(3)
    hg, hp = _plan(p, 1), _plan(p, 0)
    try:
        for h in (hg, hp):
            fda.fda_plan_set_correction(h, csr[0], csr[1], csr[2].view(np.float64))
        plain = [_apply(hp, synth.random_phi(p.N, s)) for s in (1, 2, 3, 4)]
        # applies 1 (plain), 2 (captured + replayed), 3-4 (replays), each with fresh phi / out buffers
        graph = [_apply(hg, synth.random_phi(p.N, s)) for s in (1, 2, 3, 4)]
        for a, b in zip(graph, plain):
            assert oracle.rel_l2(a, b) <= 1e-13
        # another phase mask gets its own graph
        far_p = _apply(hp, synth.random_phi(p.N, 5), fda.FDA_PHASE_FAR)
        for _ in range(3):
            far_g = _apply(hg, synth.random_phi(p.N, 5), fda.FDA_PHASE_FAR)
            assert oracle.rel_l2(far_g, far_p) <= 1e-13
        assert "graph capture of the apply failed" not in fda.fda_plan_log(hg)
        # full apply against the oracle
        phi = synth.random_phi(p.N, 4)
        ref = oracle.apply_rows(p.x, p.n, p.w, p.k, p.alpha, phi, csr=csr)
        err = oracle.rel_l2(graph[3], ref)
        print(f"config {cfg} N={p.N}: graph vs oracle {err:.3e}")
        assert err <= 1e-4
    finally:
        fda.fda_plan_destroy(hg)
        fda.fda_plan_destroy(hp)


def test_set_correction_drops_the_graph():
    fda = _fda()
    p = synth.make_problem("1")
    phi = synth.random_phi(p.N, 11)
    n = p.N
    rng = np.random.default_rng(5)
    # a diagonal correction: out changes by val_i phi_i exactly
    row_ptr = np.arange(n + 1, dtype=np.int64)
    col = np.arange(n, dtype=np.int32)
    val = (rng.uniform(-1, 1, n) + 1j * rng.uniform(-1, 1, n)).astype(np.complex128)
    h = _plan(p, 1)
    try:
        base = [_apply(h, phi) for _ in range(3)][-1]    # replayed graph, no correction
        fda.fda_plan_set_correction(h, row_ptr, col, val.view(np.float64))
        got = [_apply(h, phi) for _ in range(3)]          # plain, captured, replayed with the correction
        for g in got:
            d = g - base
            assert oracle.rel_l2(d, val * phi) <= 1e-10
    finally:
        fda.fda_plan_destroy(h)
