"""Pins of the oracle's locally corrected Nystrom weights.

`oracle.element_moments` / `oracle.corrected_weights` are pinned to facts outside the oracle:
  N1  k = 0 double layer over a flat triangle = -(solid angle)/(4 pi), van Oosterom-Strackee closed form
  N2  k = 0 hypersingular moment = n_x . grad_x of N1's closed form (finite differences of the closed form)
  N3  Helmholtz BM_H moments on a curved element = brute-force uniform subdivision with the 6-point rule
      (no adaptivity, no Gauss-Legendre, evaluated by the pinned plain sum `oracle.apply_targets`)
  N4  far limit: wbar_j -> w_j K(x, y_j) at the rate of the 6-point rule (pins the order of j and the
      orientation of the moment system)
  N5  the subdivision has converged (default parameters vs finer ones)
"""
import numpy as np
import pytest

import oracle
import synth


def _flat_element(rng, scale=1.0):
    c = rng.normal(size=(3, 3)) * scale
    return np.stack([c[0], c[1], c[2], 0.5 * (c[0] + c[1]), 0.5 * (c[1] + c[2]), 0.5 * (c[2] + c[0])])


def _solid_angle(x, tri):
    a, b, c = tri[0] - x, tri[1] - x, tri[2] - x
    la, lb, lc = np.linalg.norm(a), np.linalg.norm(b), np.linalg.norm(c)
    num = np.dot(a, np.cross(b, c))
    den = la * lb * lc + np.dot(a, b) * lc + np.dot(a, c) * lb + np.dot(b, c) * la
    return 2.0 * np.arctan2(num, den)


def _unit(v):
    return v / np.linalg.norm(v)


@pytest.mark.parametrize("seed", [1, 2, 3])
def test_n1_double_layer_is_solid_angle(seed):
    rng = np.random.default_rng(seed)
    el = _flat_element(rng)
    cen = el[:3].mean(axis=0)
    nrm = _unit(np.cross(el[1] - el[0], el[2] - el[0]))
    h = max(np.linalg.norm(el[i] - el[j]) for i, j in ((0, 1), (1, 2), (2, 0)))
    for dist in (0.02, 0.3, 3.0):   # very near, near, far (in units of the side length)
        x = cen + dist * h * nrm + 0.2 * h * _unit(el[1] - el[0])
        tn = _unit(rng.normal(size=3))
        mom = oracle.element_moments(oracle.KIND_DNY, el[None], x[None], tn[None], [0], [0], 0.0, 0j)
        want = -_solid_angle(x, el[:3]) / (4 * np.pi)
        assert abs(mom[0, 0] - want) <= 1e-11 * max(1.0, abs(want)), (dist, mom[0, 0], want)


@pytest.mark.parametrize("seed", [4, 5])
def test_n2_hypersingular_is_gradient_of_solid_angle(seed):
    rng = np.random.default_rng(seed)
    el = _flat_element(rng)
    cen = el[:3].mean(axis=0)
    nrm = _unit(np.cross(el[1] - el[0], el[2] - el[0]))
    h = np.linalg.norm(el[1] - el[0])
    for dist in (0.05, 0.5):
        x = cen - dist * h * nrm + 0.1 * h * _unit(el[2] - el[0])
        tn = _unit(rng.normal(size=3))
        mom = oracle.element_moments(oracle.KIND_HYP, el[None], x[None], tn[None], [0], [0], 0.0, 0j)
        e = 1e-5 * dist * h
        fd = (_solid_angle(x + e * tn, el[:3]) - _solid_angle(x - e * tn, el[:3])) / (2 * e)
        want = -fd / (4 * np.pi)
        assert abs(mom[0, 0] - want) <= 2e-7 * abs(want), (dist, mom[0, 0], want)


def _brute_moments(kind, el, x, tn, k, alpha, level):
    """Uniform 4^level subdivision of the reference triangle, 6-point degree-4 rule on every piece."""
    rp = synth.rule_points()
    m = 2 ** level
    pts, wts = [], []
    for i in range(m):
        for j in range(m - i):
            o = np.array([i, j], float) / m
            pts.append(o + rp[:, :2] / m)                       # upright piece
            wts.append(rp[:, 2] * 0.5 / m ** 2)
            if i + j + 2 <= m:                                   # inverted piece
                pts.append(o + (1.0 - rp[:, :2]) / m)
                wts.append(rp[:, 2] * 0.5 / m ** 2)
    xi = np.concatenate(pts)
    wr = np.concatenate(wts)
    assert abs(wr.sum() - 0.5) < 1e-13
    N, d1, d2 = synth.shape_functions(xi[:, 0], xi[:, 1])
    y = N @ el
    cr = np.cross(d1 @ el, d2 @ el)
    jac = np.linalg.norm(cr, axis=1)
    ny = cr / jac[:, None]
    out = []
    for p, q in ((0, 0), (1, 0), (0, 1), (2, 0), (1, 1), (0, 2)):
        dens = (xi[:, 0] ** p * xi[:, 1] ** q).astype(np.complex128)
        out.append(oracle.apply_targets(kind, x[None], tn[None], y, ny, wr * jac, k, alpha, dens)[0])
    return np.array(out)


@pytest.mark.parametrize("kind", [oracle.KIND_BMH, oracle.KIND_BMG])
def test_n3_helmholtz_moments_vs_uniform_brute_force(kind):
    nodes = synth.octa_sphere(4)
    el = nodes[7]
    k = 6.0
    alpha = 1j / k
    xq, nq, wq, hmax, _ = synth.quadrature_cloud(nodes)
    # field point: a quadrature point of another element of D_i (not adjacent to the element's edge)
    d = np.linalg.norm(xq - el[:3].mean(axis=0), axis=1)
    cand = [i for i in np.argsort(d) if i // 6 != 7 and d[i] > 0.6 * hmax[7]]
    i = cand[0]
    mom = oracle.element_moments(kind, el[None], xq[i][None], nq[i][None], [0], [0], k, alpha)[0]
    want = _brute_moments(kind, el, xq[i], nq[i], k, alpha, level=6)
    assert np.max(np.abs(mom - want)) <= 1e-7 * np.max(np.abs(want)), (mom, want)


def test_n4_far_limit_recovers_the_plain_weights():
    xi = synth.rule_points()[:, :2]
    # (a) flat element, k = 0: K J phi^(n) is smooth on the scale d, and the 6-point rule is exact to degree 4,
    # so wbar_j - w_j K(x, y_j) decays like (h / d)^3 relative to w_j K
    rng = np.random.default_rng(7)
    el = _flat_element(rng)
    xq, nq, wq, hmax, _ = synth.quadrature_cloud(el[None])
    cen = el[:3].mean(axis=0)
    tn = _unit(np.array([0.2, 0.9, -0.4]))
    errs = []
    for dist in (5.0, 10.0, 20.0):
        x = cen + dist * hmax[0] * _unit(np.array([0.3, -0.5, 0.8]))
        wb = oracle.corrected_weights(oracle.KIND_BMH, el[None], xi, x[None], tn[None], [0], [0], 0.0, 1.0)[0]
        plain = np.array([wq[j] * oracle.kernel(oracle.KIND_BMH, x, tn, xq[j], nq[j], 0.0, 1.0) for j in range(6)])
        errs.append(np.max(np.abs(wb - plain)) / np.max(np.abs(plain)))
    assert errs[0] < 1e-2 and errs[1] < errs[0] / 5.0 and errs[2] < errs[1] / 5.0, errs
    # (b) curved element, Helmholtz: the difference stays at the (k h)^3 / curvature level of the rule; a
    # permutation of j or a transposed moment system would be an O(1) error
    nodes = synth.octa_sphere(4)
    e = 11
    el = nodes[e]
    xq, nq, wq, hmax, _ = synth.quadrature_cloud(nodes)
    k = 2.0
    alpha = 1j / k
    x = el[:3].mean(axis=0) + 10.0 * hmax[e] * _unit(_unit(el[:3].mean(axis=0)) + np.array([0.3, -0.2, 0.1]))
    wb = oracle.corrected_weights(oracle.KIND_BMH, el[None], xi, x[None], tn[None], [0], [0], k, alpha)[0]
    plain = np.array([wq[6 * e + j] * oracle.kernel(oracle.KIND_BMH, x, tn, xq[6 * e + j], nq[6 * e + j], k, alpha)
                      for j in range(6)])
    assert np.max(np.abs(wb - plain)) / np.max(np.abs(plain)) < 2e-3


def test_n5_subdivision_converged():
    nodes = synth.octa_sphere(8)
    xq, nq, wq, hmax, samples = synth.quadrature_cloud(nodes)
    ptr, idx = synth.local_regions(samples, hmax, xq)
    k = 5.0
    alpha = 1j / k
    xi = synth.rule_points()[:, :2]
    ts, es = [], []
    for t in (0, 100, 1234):
        for e in idx[ptr[t]:ptr[t + 1]]:
            if e != t // 6:
                ts.append(t), es.append(int(e))
    a = oracle.corrected_weights(oracle.KIND_BMH, nodes, xi, xq, nq, ts, es, k, alpha)
    b = oracle.corrected_weights(oracle.KIND_BMH, nodes, xi, xq, nq, ts, es, k, alpha, nq=16, theta=0.125)
    assert np.max(np.abs(a - b)) <= 1e-11 * np.max(np.abs(b))
    # moment identity of eq:local correction with the independent numpy Vandermonde
    mom = oracle.element_moments(oracle.KIND_BMH, nodes, xq, nq, ts, es, k, alpha)
    V = np.stack([xi[:, 0] ** p * xi[:, 1] ** q for p, q in ((0, 0), (1, 0), (0, 1), (2, 0), (1, 1), (0, 2))])
    assert np.max(np.abs(a @ V.T - mom)) <= 1e-12 * np.max(np.abs(mom))
