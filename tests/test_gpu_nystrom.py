"""Locally corrected Nystrom weights on the device through the C ABI
(`fda_nystrom_weights`) against the oracle (`oracle.corrected_weights`, pinned by tests/test_oracle_nystrom.py).

Bar (R27): per pair, max_j |wbar_j - oracle_j| <= 1e-10 max_j |oracle_j| with the oracle at its own,
finer parameters (nq = 12, theta = 0.25); <= 1e-11 when both sides run the same (nq, theta) with the device's
flatness split switched off, where the two subdivisions take the same decisions and only the order of the sums
differs.
"""
import numpy as np
import pytest

import oracle
import synth

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

KINDS = {"bmh": oracle.KIND_BMH, "bmg": oracle.KIND_BMG, "t1": oracle.KIND_T1}


def _fda():
    from paper_1311_5202_b200 import fda
    return fda


def _rule():
    rp = synth.rule_points()
    return np.ascontiguousarray(rp[:, :2]), np.ascontiguousarray(0.5 * rp[:, 2])


def _pairs(p, stride, offset=0):
    """(t, e) for every element e of D_t except the one holding t, for t = offset, offset + stride, ..."""
    ptr, idx = synth.local_regions(p.samples, p.hmax, p.x)
    ts, es = [], []
    for t in range(offset, p.N, stride):
        for e in idx[ptr[t]:ptr[t + 1]]:
            if e != t // 6:
                ts.append(t), es.append(int(e))
    return np.array(ts, dtype=np.int64), np.array(es, dtype=np.int64)


def _pair_err(a, b):
    return float(np.max(np.max(np.abs(a - b), axis=1) / np.max(np.abs(b), axis=1)))


@pytest.mark.parametrize("kind", ["bmh", "bmg", "t1"])
def test_weights_match_oracle(kind):
    fda = _fda()
    p = synth.make_problem("1")
    xi, wref = _rule()
    ts, es = _pairs(p, 5 if kind == "bmh" else 23)
    kcode = {"bmh": fda.FDA_KERNEL_BMH, "bmg": fda.FDA_KERNEL_BMG, "t1": fda.FDA_KERNEL_T1}[kind]
    wbar = np.zeros((ts.shape[0], 6), np.complex128)
    delta = np.zeros_like(wbar)
    fda.fda_nystrom_weights(kcode, p.k, p.alpha, p.nodes, xi, wref, p.x, p.n, ts, es, wbar, delta)
    ref = oracle.corrected_weights(KINDS[kind], p.nodes, xi, p.x, p.n, ts, es, p.k, p.alpha)
    err = _pair_err(wbar, ref)
    # delta = wbar_j - w_j K(x_t, y_j) with the plain weights of the cloud (reading R4)
    plain = np.array([[p.w[6 * e + j] * oracle.kernel(KINDS[kind], p.x[t], p.n[t], p.x[6 * e + j], p.n[6 * e + j],
                                                      p.k, p.alpha) for j in range(6)]
                      for t, e in zip(ts[:400], es[:400])])
    derr = float(np.max(np.abs(delta[:400] - (ref[:400] - plain))) / np.max(np.abs(ref[:400])))
    print(f"nystrom weights {kind}: {ts.shape[0]} pairs, max pair error {err:.2e}, delta error {derr:.2e}")
    assert err <= 1e-10
    assert derr <= 1e-10


def test_same_parameters_same_subdivision():
    fda = _fda()
    p = synth.make_problem("1")
    xi, wref = _rule()
    ts, es = _pairs(p, 41, offset=3)
    ts, es = ts[:-1], es[:-1]          # a ragged last CTA
    for nq, theta in ((6, 0.35), (5, 0.8), (16, 0.5)):
        wbar = np.zeros((ts.shape[0], 6), np.complex128)
        fda.fda_nystrom_weights(fda.FDA_KERNEL_BMH, p.k, p.alpha, p.nodes, xi, wref, p.x, p.n, ts, es, wbar, None,
                                nq=nq, theta=theta, gamma=1e30, max_depth=20)
        ref = oracle.corrected_weights(oracle.KIND_BMH, p.nodes, xi, p.x, p.n, ts, es, p.k, p.alpha, nq=nq,
                                       theta=theta, maxdepth=20)
        err = _pair_err(wbar, ref)
        print(f"nq={nq} theta={theta}: {err:.2e}")
        assert err <= 1e-11


def test_device_pointers_and_determinism():
    fda = _fda()
    p = synth.make_problem("1")
    xi, wref = _rule()
    ts, es = _pairs(p, 97)
    host = np.zeros((ts.shape[0], 6), np.complex128)
    fda.fda_nystrom_weights(fda.FDA_KERNEL_BMH, p.k, p.alpha, p.nodes, xi, wref, p.x, p.n, ts, es, host)
    dev = torch.device("cuda", 0)
    d = {k: torch.from_numpy(np.ascontiguousarray(v)).to(dev) for k, v in
         dict(nodes=p.nodes, xi=xi, wref=wref, x=p.x, n=p.n, ts=ts, es=es).items()}
    out = torch.zeros(ts.shape[0], 12, dtype=torch.float64, device=dev)
    dl = torch.zeros_like(out)
    for _ in range(2):
        fda.fda_nystrom_weights(fda.FDA_KERNEL_BMH, p.k, p.alpha, d["nodes"], d["xi"], d["wref"], d["x"], d["n"],
                                d["ts"], d["es"], out, dl)
        got = out.cpu().numpy().view(np.complex128)
        assert np.array_equal(got, host)       # same launch, same order of operations: bit-identical


def test_edge_cases():
    fda = _fda()
    p = synth.make_problem("1")
    xi, wref = _rule()
    empty = np.zeros(0, np.int64)
    fda.fda_nystrom_weights(fda.FDA_KERNEL_BMH, p.k, p.alpha, p.nodes, xi, wref, p.x, p.n, empty, empty,
                            np.zeros((0, 6), np.complex128))
    one = np.zeros((1, 6), np.complex128)
    # the self element is the singular case of [rjj_int]: refused, not approximated
    with pytest.raises(fda.FDAError, match="INVALID_ARG"):
        fda.fda_nystrom_weights(fda.FDA_KERNEL_BMH, p.k, p.alpha, p.nodes, xi, wref, p.x, p.n,
                                np.array([13], np.int64), np.array([2], np.int64), one)
    with pytest.raises(fda.FDAError, match="INVALID_ARG"):      # element index out of range
        fda.fda_nystrom_weights(fda.FDA_KERNEL_BMH, p.k, p.alpha, p.nodes, xi, wref, p.x, p.n,
                                np.array([0], np.int64), np.array([p.nodes.shape[0]], np.int64), one)
    with pytest.raises(fda.FDAError, match="INVALID_ARG"):      # nq above the limit
        fda.fda_nystrom_weights(fda.FDA_KERNEL_BMH, p.k, p.alpha, p.nodes, xi, wref, p.x, p.n,
                                np.array([0], np.int64), np.array([5], np.int64), one, nq=17)
    with pytest.raises(fda.FDAError, match="INVALID_ARG"):      # six collinear points: singular moment matrix
        bad = np.stack([np.linspace(0.1, 0.4, 6), np.linspace(0.1, 0.4, 6)], axis=1)
        fda.fda_nystrom_weights(fda.FDA_KERNEL_BMH, p.k, p.alpha, p.nodes, bad, wref, p.x, p.n,
                                np.array([0], np.int64), np.array([5], np.int64), one)
    # a field point very close to (not on) the element: 1e-3 side lengths above the centroid of a flat triangle,
    # against the closed-form solid angle (k = 0, alpha = 0 gives the double layer)
    tri = np.array([[0, 0, 0], [1, 0, 0], [0, 1, 0]], float)
    el = np.stack([tri[0], tri[1], tri[2], 0.5 * (tri[0] + tri[1]), 0.5 * (tri[1] + tri[2]), 0.5 * (tri[2] + tri[0])])
    x = np.array([[1 / 3, 1 / 3, 1e-3]])
    w6 = np.zeros((1, 6), np.complex128)
    fda.fda_nystrom_weights(fda.FDA_KERNEL_BMH, 0.0, 0.0, el[None], xi, wref, x, np.array([[0.0, 0.0, 1.0]]),
                            np.array([0], np.int64), np.array([0], np.int64), w6)
    a, b, c = tri - x[0]
    num = np.dot(a, np.cross(b, c))
    den = (np.linalg.norm(a) * np.linalg.norm(b) * np.linalg.norm(c) + np.dot(a, b) * np.linalg.norm(c)
           + np.dot(a, c) * np.linalg.norm(b) + np.dot(b, c) * np.linalg.norm(a))
    omega = 2.0 * np.arctan2(num, den)
    assert abs(w6.sum() - (-omega / (4 * np.pi))) <= 1e-10    # sum_j wbar_j = I_0 (phi^(0) = 1)


def test_anisotropic_mesh_pairs():
    """Prolate spheroid 10:1:1 (the geometry of config 4, coarse): stretched elements, larger local regions."""
    fda = _fda()
    nodes = synth.spheroid(10.0, 1.0, 0.5)
    x, n, w, hmax, samples = synth.quadrature_cloud(nodes)
    ptr, idx = synth.local_regions(samples, hmax, x)
    xi, wref = _rule()
    ts, es = [], []
    for t in range(1, x.shape[0], 9):
        for e in idx[ptr[t]:ptr[t + 1]]:
            if e != t // 6:
                ts.append(t), es.append(int(e))
    ts, es = np.array(ts, np.int64), np.array(es, np.int64)
    k = 4.0
    wbar = np.zeros((ts.shape[0], 6), np.complex128)
    fda.fda_nystrom_weights(fda.FDA_KERNEL_BMH, k, 1j / k, nodes, xi, wref, x, n, ts, es, wbar)
    ref = oracle.corrected_weights(oracle.KIND_BMH, nodes, xi, x, n, ts, es, k, 1j / k)
    err = _pair_err(wbar, ref)
    print(f"spheroid: {ts.shape[0]} pairs, max pair error {err:.2e}")
    assert err <= 1e-10


def test_corrected_rows_feed_the_apply():
    """The delta values fill the D_i pattern of the correction CSR (self elements left zero: [rjj_int] is out of
    scope) and the apply with them matches the oracle's rows built from the oracle's own weights."""
    fda = _fda()
    p = synth.make_problem("1")
    xi, wref = _rule()
    ptr, idx = synth.local_regions(p.samples, p.hmax, p.x)
    row_ptr, col, _ = synth.correction_csr(ptr, idx, p.w, p.hmax, p.k, 1)
    ts = np.repeat(np.arange(p.N, dtype=np.int64), np.diff(ptr))
    es = idx.astype(np.int64)
    assert np.array_equal(col.reshape(-1, 6)[:, 0], 6 * es)       # row t holds the 6 nodes of each e in D_t
    notself = es != ts // 6
    delta = np.zeros((int(notself.sum()), 6), np.complex128)
    fda.fda_nystrom_weights(fda.FDA_KERNEL_BMH, p.k, p.alpha, p.nodes, xi, wref, p.x, p.n,
                            np.ascontiguousarray(ts[notself]), np.ascontiguousarray(es[notself]), None, delta)
    val = np.zeros((es.shape[0], 6), np.complex128)
    val[notself] = delta
    val = np.ascontiguousarray(val.reshape(-1))
    phi = synth.plane_wave(p.x, p.k)
    h = fda.fda_plan_create(p.x, p.n, p.w, p.k, p.alpha, p.eps)
    try:
        fda.fda_plan_set_correction(h, row_ptr, col, val.view(np.float64))
        d_phi = torch.from_numpy(phi.view(np.float64).copy()).cuda()
        d_out = torch.empty_like(d_phi)
        fda.fda_apply(h, d_phi, d_out)
        torch.cuda.synchronize()
        got = d_out.cpu().numpy().view(np.complex128)
    finally:
        fda.fda_plan_destroy(h)
    rows = synth.sample_rows(p.N, 300, 11)
    # the oracle's rows: plain far quadrature outside D_i, its own corrected weights inside (kcorrection)
    sel = notself & np.isin(ts, rows)
    wb = oracle.corrected_weights(oracle.KIND_BMH, p.nodes, xi, p.x, p.n, ts[sel], es[sel], p.k, p.alpha)
    ref = oracle.apply_rows(p.x, p.n, p.w, p.k, p.alpha, phi, rows=rows)
    pos = {int(r): i for i, r in enumerate(rows)}
    for (t, e), w6 in zip(zip(ts[sel], es[sel]), wb):
        for j in range(6):
            c = 6 * e + j
            plain = p.w[c] * oracle.kernel(oracle.KIND_BMH, p.x[t], p.n[t], p.x[c], p.n[c], p.k, p.alpha)
            ref[pos[int(t)]] += (w6[j] - plain) * phi[c]
    err = oracle.rel_l2(got[rows], ref)
    print(f"apply with device-computed corrections: rel_l2={err:.3e}")
    assert err <= 1e-4
