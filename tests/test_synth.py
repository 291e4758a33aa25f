"""Generator pins: these fix the oracle's *inputs*."""
import numpy as np
import pytest

import synth


def test_rule_integrates_monomial_exactly():
    # the degree-4 rule integrates xi1^2 xi2^2 over the reference triangle to 1/180
    rp = synth.rule_points()
    val = 0.5 * np.sum(rp[:, 2] * rp[:, 0] ** 2 * rp[:, 1] ** 2)
    assert abs(val - 1.0 / 180.0) < 1e-14
    assert abs(0.5 * rp[:, 2].sum() - 0.5) < 1e-14


def test_shape_partition_of_unity():
    rng = np.random.default_rng(0)
    a = rng.uniform(0, 1, 1000)
    b = rng.uniform(0, 1, 1000) * (1 - a)
    N, d1, d2 = synth.shape_functions(a, b)
    assert np.abs(N.sum(-1) - 1).max() < 1e-13
    assert np.abs(d1.sum(-1)).max() < 1e-13
    assert np.abs(d2.sum(-1)).max() < 1e-13


def test_sphere_counts_and_normals():
    p = synth.make_problem("1")
    assert p.N == 3072 and p.nodes.shape[0] == 512
    assert np.abs(np.linalg.norm(p.n, axis=1) - 1).max() < 1e-12
    assert np.all(p.w > 0)
    # outward: sum w n.(x - c) > 0, and n ~ x on the unit sphere
    assert np.sum(p.w * np.einsum("ij,ij->i", p.n, p.x - p.x.mean(0))) > 0
    assert np.min(np.einsum("ij,ij->i", p.n, p.x)) > 0.99
    # closed surface: sum w n = 0 (divergence theorem)
    assert np.abs((p.w[:, None] * p.n).sum(0)).max() < 1e-10 * 4 * np.pi


def test_area_converges_order3():
    errs = []
    for nu in (4, 8, 16):
        p = synth.make_problem("x", k=1.0, nu=nu)
        errs.append(abs(p.w.sum() - 4 * np.pi))
    rates = [np.log2(errs[i] / errs[i + 1]) for i in range(2)]
    assert min(rates) >= 3.0, (errs, rates)


def test_spheroid_mesh():
    nodes = synth.spheroid(10.0, 1.0, 0.5)
    x, n, w, hmax, s = synth.quadrature_cloud(nodes)
    # area of the 10:1:1 prolate spheroid: 2 pi b^2 (1 + a/(b e) asin e)
    a, b = 10.0, 1.0
    e = np.sqrt(1 - b * b / (a * a))
    area = 2 * np.pi * b * b * (1 + a / (b * e) * np.arcsin(e))
    assert abs(w.sum() - area) / area < 2e-3
    assert np.abs((w[:, None] * n).sum(0)).max() < 1e-8 * area
    assert np.sum(w * np.einsum("ij,ij->i", n, x)) > 0
    # near-isotropic elements: aspect bounded
    assert hmax.max() / hmax.min() < 4.0


def test_local_regions_bruteforce():
    p = synth.make_problem("x", k=1.0, nu=4)
    ptr, idx = synth.local_regions(p.samples, p.hmax, p.x)
    for i in range(0, p.N, 7):
        d = np.linalg.norm(p.samples - p.x[i][None, None, :], axis=-1).min(axis=1)
        expect = np.nonzero(d <= 2 * p.hmax)[0]
        got = idx[ptr[i]:ptr[i + 1]]
        assert np.array_equal(expect, got)
        assert (i // 6) in got


def test_correction_csr_recipe():
    p = synth.make_problem("1")
    rp, col, val = p.correction(seed=3)
    nnz_row = np.diff(rp)
    assert 250 < nnz_row.mean() < 360                  # ~307 per row
    for i in (0, 100, 3071):
        cols = col[rp[i]:rp[i + 1]]
        assert np.all(np.diff(cols) > 0) and i in cols
    # counter-based values are reproducible per (seed, i, j)
    i = 17
    p0 = rp[i]
    j = int(col[p0])
    h = p.hmax[i // 6]
    scale = 0.1 / (4 * np.pi * max(p.k, 1.0) * h ** 3)
    re = synth.counter_u11(3, i, j, 0)
    im = synth.counter_u11(3, i, j, 1)
    expect = scale * p.w[j] * (re + 1j * im) + (0.5 if i == j else 0.0)
    assert abs(val[p0] - expect) < 1e-15


def test_phi_seeded():
    a = synth.random_phi(100, 5)
    b = synth.random_phi(100, 5)
    assert np.array_equal(a, b)
    assert np.all(np.abs(a.real) <= 1) and np.all(np.abs(a.imag) <= 1)


def test_cube_sphere_table1_counts_and_geometry():
    """Table-1 point sets: N = 72 m^2 = 73,728 at m = 32; outward unit normals,
    area -> 4 pi at >= third order under m -> 2m."""
    import numpy as np
    import synth
    nd = synth.cube_sphere(32)
    assert nd.shape[0] * 6 == 73728
    errs = []
    for m in (4, 8, 16):
        x, n, w, hmax, s = synth.quadrature_cloud(synth.cube_sphere(m))
        assert x.shape[0] == 72 * m * m
        assert np.abs(np.linalg.norm(n, axis=1) - 1).max() < 1e-12
        assert np.all(np.einsum("ij,ij->i", n, x) > 0)
        errs.append(abs(w.sum() - 4 * np.pi))
    assert errs[1] / errs[2] > 7.0 and errs[0] / errs[1] > 7.0
