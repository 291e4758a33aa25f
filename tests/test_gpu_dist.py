"""Multi-GPU data plane on one GPU.

* Sequential rank emulation: R partitioned plans (rank r of R, no communicator) run fda_apply_up
  (S2M on own leaves, M2M on cubes holding own points, pack of the partial expansions), the test moves
  the packed bytes between the ranks' buffers exactly as the NCCL send/receive would, then
  fda_apply_down (sum of the received partials, P2P, correction, M2L, L2L, L2T).  The ranks' outputs
  are disjoint and add up to the single-rank apply (<= 1e-13: same arithmetic up to the order of the
  FP64 atomic accumulations).  The ranks run one after another: no kernel waits on another rank.
* fda_plan_create_dist with one rank: the NCCL path (communicator, output all-gather) equals the
  plain plan.
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


@pytest.fixture(scope="module")
def prob():
    p = synth.make_problem("x", k=50.0, nu=16)            # HF + LF levels, N = 12288
    csr = p.correction(seed=3)
    phi = synth.random_phi(p.N, 5)
    return p, csr, phi


def _full(p, csr, phi):
    fda = _fda()
    h = fda.fda_plan_create(_dev(p.x), _dev(p.n), _dev(p.w), p.k, p.alpha, p.eps)
    try:
        fda.fda_plan_set_correction(h, csr[0], csr[1], csr[2].view(np.float64))
        d_phi = _dev(phi.view(np.float64))
        d_out = torch.empty_like(d_phi)
        fda.fda_apply(h, d_phi, d_out)
        return d_out.cpu().numpy().view(np.complex128).copy()
    finally:
        fda.fda_plan_destroy(h)


@pytest.mark.parametrize("nranks", [2, 3, 5])
def test_rank_emulation_sums_to_single(prob, nranks):
    fda = _fda()
    p, csr, phi = prob
    full = _full(p, csr, phi)
    d_phi = _dev(phi.view(np.float64))
    plans, send, cnt = [], [], []
    try:
        for r in range(nranks):
            h = fda.fda_plan_create(_dev(p.x), _dev(p.n), _dev(p.w), p.k, p.alpha, p.eps,
                                    fda.fda_options_default(rank=r, nranks=nranks))
            plans.append(h)
            fda.fda_plan_set_correction(h, csr[0], csr[1], csr[2].view(np.float64))
            with pytest.raises(fda.FDAError, match="STATE"):       # no communicator: two halves only
                fda.fda_apply(h, d_phi, torch.empty_like(d_phi))
            sc, rc = fda.fda_dist_counts(h, nranks)
            cnt.append((sc, rc))
        for r, h in enumerate(plans):
            buf = torch.zeros(2 * max(1, int(cnt[r][0].sum())), dtype=torch.float64, device="cuda")
            fda.fda_apply_up(h, d_phi, buf)
            send.append(buf)
        torch.cuda.synchronize()
        total_x = 0
        acc = np.zeros_like(full)
        owned = np.zeros(p.N, dtype=np.int64)
        for r, h in enumerate(plans):
            parts = []
            for q in range(nranks):
                sc_q = cnt[q][0]
                off = int(sc_q[:r].sum())
                assert int(sc_q[r]) == int(cnt[r][1][q])             # q sends r what r expects from q
                parts.append(send[q][2 * off:2 * (off + int(sc_q[r]))])
            total_x += int(cnt[r][1].sum())
            recv = torch.cat(parts) if parts else torch.zeros(2, dtype=torch.float64, device="cuda")
            if recv.numel() == 0:
                recv = torch.zeros(2, dtype=torch.float64, device="cuda")
            out = torch.empty_like(d_phi)
            fda.fda_apply_down(h, recv.contiguous(), out)
            part = out.cpu().numpy().view(np.complex128).copy()
            lop, lev, ijk = fda.fda_plan_export_leaves(h, p.N)
            st = fda.fda_plan_stats(h)
            mine = (lop >= st["owned_leaf_begin"]) & (lop < st["owned_leaf_end"])
            assert np.all(part[~mine] == 0)
            owned += mine
            acc += part
        assert total_x > 0                                         # the exchange is not empty
        assert np.all(owned == 1)
        err = oracle.rel_l2(acc, full)
        print(f"nranks={nranks}: exchanged {16 * total_x / 1e6:.2f} MB, rel to single rank {err:.2e}")
        assert err <= 1e-13
    finally:
        for h in plans:
            fda.fda_plan_destroy(h)


def test_create_dist_one_rank_nccl(prob):
    fda = _fda()
    p, csr, phi = prob
    full = _full(p, csr, phi)
    uid = fda.fda_nccl_unique_id()
    h = fda.fda_plan_create_dist(_dev(p.x), _dev(p.n), _dev(p.w), p.k, p.alpha, p.eps, uid, 0, 1)
    try:
        fda.fda_plan_set_correction(h, csr[0], csr[1], csr[2].view(np.float64))
        d_phi = _dev(phi.view(np.float64))
        d_out = torch.empty_like(d_phi)
        fda.fda_apply(h, d_phi, d_out)
        got = d_out.cpu().numpy().view(np.complex128)
        ms = fda.fda_apply_timed(h, fda.FDA_PHASE_ALL, d_phi, d_out)
    finally:
        fda.fda_plan_destroy(h)
    assert oracle.rel_l2(got, full) <= 1e-13
    assert set(ms) == set(fda.PHASES)
