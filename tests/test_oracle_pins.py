"""Pins of the CPU oracle against things other than itself.

Each test names what fixes the expected value: an independent 30-digit mpmath
differentiation of G (P1), closed forms (P2, P7), symmetry (P3), the
Gegenbauer addition theorem (P5), Green's representation formula with a plane
wave (P6), the Gauss double-layer identity (P8), an independent sparse library
(P9).  A dropped term, a wrong sign or a transposed operand in oracle.c fails
at least one of them.
"""
import numpy as np
import pytest

import oracle
import synth

mp = pytest.importorskip("mpmath")


def _rand_unit(rng):
    v = rng.normal(size=3)
    return v / np.linalg.norm(v)


# --------------------------------------------------------------- P1: mpmath
def _mp_G(k, x, y):
    r = mp.sqrt(sum((x[i] - y[i]) ** 2 for i in range(3)))
    return mp.exp(1j * k * r) / (4 * mp.pi * r)


def _mp_kernels(k, x, nx, y, ny):
    """G and its normal derivatives by 30-digit numerical differentiation of G (independent of oracle.c)."""
    mp.mp.dps = 30
    x = [mp.mpf(float(v)) for v in x]
    y = [mp.mpf(float(v)) for v in y]
    nx = [mp.mpf(float(v)) for v in nx]
    ny = [mp.mpf(float(v)) for v in ny]
    k = mp.mpf(float(k))

    def f(s, t):
        return _mp_G(k, [x[i] + s * nx[i] for i in range(3)], [y[i] + t * ny[i] for i in range(3)])

    g = f(0, 0)
    dny = mp.diff(f, (0, 0), (0, 1))
    dnx = mp.diff(f, (0, 0), (1, 0))
    hyp = mp.diff(f, (0, 0), (1, 1))
    return [complex(v) for v in (g, dny, dnx, hyp)]


@pytest.mark.parametrize("seed", range(6))
def test_p1_kernels_vs_mpmath(seed):
    rng = np.random.default_rng(seed)
    k = [0.3, 2.0, 5.0, 17.0, 50.0, 1e-3][seed]
    x = rng.normal(size=3)
    y = x + rng.normal(size=3) * [0.05, 0.5, 1.0, 0.2, 0.03, 2.0][seed]
    nx, ny = _rand_unit(rng), _rand_unit(rng)
    ref = _mp_kernels(k, x, nx, y, ny)
    alpha = 1j / k
    got = [oracle.kernel(kind, x, nx, y, ny, k, alpha) for kind in range(4)]
    for a, b in zip(got, ref):
        assert abs(a - b) <= 1e-12 * abs(b) + 1e-300, (got, ref)
    bmh = oracle.kernel(oracle.KIND_BMH, x, nx, y, ny, k, alpha)
    assert abs(bmh - (ref[1] + alpha * ref[3])) <= 1e-12 * abs(ref[1] + alpha * ref[3])
    bmg = oracle.kernel(oracle.KIND_BMG, x, nx, y, ny, k, alpha)
    assert abs(bmg - (ref[0] + alpha * ref[2])) <= 1e-12 * abs(ref[0] + alpha * ref[2])


def test_p1_tiny_full_sum_vs_mpmath():
    """N = 10 points: the whole discrete operator incl. the j != i exclusion, at 30 digits."""
    rng = np.random.default_rng(11)
    n = 10
    x = rng.normal(size=(n, 3))
    nr = rng.normal(size=(n, 3))
    nr /= np.linalg.norm(nr, axis=1, keepdims=True)
    w = rng.uniform(0.1, 1.0, n)
    phi = rng.uniform(-1, 1, n) + 1j * rng.uniform(-1, 1, n)
    k = 3.0
    alpha = 1j / k
    got = oracle.apply_rows(x, nr, w, k, alpha, phi)
    for i in range(n):
        acc = 0
        for j in range(n):
            if j == i:
                continue
            g, dny, dnx, hyp = _mp_kernels(k, x[i], nr[i], x[j], nr[j])
            acc += w[j] * (dny + alpha * hyp) * phi[j]
        assert abs(got[i] - acc) <= 1e-12 * abs(acc)


# --------------------------------------------------------------- P2: closed forms
def test_p2_point_values():
    # G at kr = 2 pi equals 1/(4 pi)
    g = oracle.kernel(oracle.KIND_G, [0, 0, 0], None, [1, 0, 0], None, 2 * np.pi)
    assert abs(g - 1 / (4 * np.pi)) < 1e-16
    # dG/dn_y = 0 when n_y is perpendicular to y - x
    v = oracle.kernel(oracle.KIND_DNY, [0, 0, 0], [0, 0, 1], [1, 0, 0], [0, 1, 0], 3.0)
    assert v == 0
    # with n_x = n_y = (y - x)/r: d2G/dn_x dn_y = -g''(r)   (SPEC.md:124 has the wrong sign)
    mp.mp.dps = 30
    k, r = 1.7, 0.9
    g2 = complex(mp.diff(lambda t: mp.exp(1j * k * t) / (4 * mp.pi * t), r, 2))
    e = [1.0, 0.0, 0.0]
    h = oracle.kernel(oracle.KIND_HYP, [0, 0, 0], e, [r, 0, 0], e, k)
    assert abs(h + g2) < 1e-13 * abs(g2)
    assert abs(h - g2) > 0.1 * abs(g2)


# --------------------------------------------------------------- P3: symmetry
def test_p3_reciprocity():
    rng = np.random.default_rng(3)
    for _ in range(20):
        x, y = rng.normal(size=3), rng.normal(size=3)
        a, b = _rand_unit(rng), _rand_unit(rng)
        k = rng.uniform(0.1, 30)
        assert oracle.kernel(0, x, None, y, None, k) == oracle.kernel(0, y, None, x, None, k)
        d1 = oracle.kernel(oracle.KIND_DNY, x, None, y, a, k)
        d2 = oracle.kernel(oracle.KIND_DNX, y, a, x, None, k)
        assert abs(d1 - d2) <= 1e-15 * abs(d1)
        h1 = oracle.kernel(oracle.KIND_HYP, x, a, y, b, k)
        h2 = oracle.kernel(oracle.KIND_HYP, y, b, x, a, k)
        assert abs(h1 - h2) <= 1e-14 * abs(h1)


# --------------------------------------------------------------- P4: finite differences
def test_p4_finite_differences():
    rng = np.random.default_rng(4)
    for _ in range(10):
        x, y = rng.normal(size=3), rng.normal(size=3)
        a, b = _rand_unit(rng), _rand_unit(rng)
        k = rng.uniform(0.5, 5)
        r = np.linalg.norm(x - y)
        h = 1e-5 * r
        G = lambda p, q: oracle.kernel(0, p, None, q, None, k)
        fd = (G(x, y + h * b) - G(x, y - h * b)) / (2 * h)
        assert abs(fd - oracle.kernel(oracle.KIND_DNY, x, None, y, b, k)) < 1e-8 * abs(fd) + 1e-12
        fd = (G(x + h * a, y) - G(x - h * a, y)) / (2 * h)
        assert abs(fd - oracle.kernel(oracle.KIND_DNX, x, a, y, None, k)) < 1e-8 * abs(fd) + 1e-12
        h = 1e-4 * r
        D = lambda p: (G(p, y + h * b) - G(p, y - h * b)) / (2 * h)
        fd2 = (D(x + h * a) - D(x - h * a)) / (2 * h)
        ex = oracle.kernel(oracle.KIND_HYP, x, a, y, b, k)
        assert abs(fd2 - ex) < 1e-6 * abs(ex)


# --------------------------------------------------------------- P5: Gegenbauer addition theorem
@pytest.mark.parametrize("k", [0.5, 5.0, 50.0])
def test_p5_addition_theorem(k):
    from scipy.special import eval_legendre, spherical_jn, spherical_yn
    rng = np.random.default_rng(int(k * 10))
    for _ in range(5):
        xx = _rand_unit(rng) * 1.0
        yy = _rand_unit(rng) * 0.6
        rx, ry = np.linalg.norm(xx), np.linalg.norm(yy)
        c = xx @ yy / (rx * ry)
        nmax = int(max(k * rx + 10 * (k * rx) ** (1 / 3) + 10, np.log(1e-16) / np.log(ry / rx))) + 5
        n = np.arange(nmax + 1)
        h = spherical_jn(n, k * rx) + 1j * spherical_yn(n, k * rx)
        s = (1j * k / (4 * np.pi)) * np.sum((2 * n + 1) * spherical_jn(n, k * ry) * h * eval_legendre(n, c))
        g = oracle.kernel(0, xx, None, yy, None, k)
        assert abs(g - s) < 1e-10 * abs(g)


# --------------------------------------------------------------- P6: Green representation
def _product_sphere(nt, nph, R=1.0):
    ct, wt = np.polynomial.legendre.leggauss(nt)
    ph = 2 * np.pi * np.arange(nph) / nph
    C, P = np.meshgrid(ct, ph, indexing="ij")
    S = np.sqrt(1 - C ** 2)
    nrm = np.stack([S * np.cos(P), S * np.sin(P), C], -1).reshape(-1, 3)
    w = (wt[:, None] * np.full(nph, 2 * np.pi / nph)[None, :]).reshape(-1) * R * R
    return R * nrm, nrm, w


def test_p6_green_identity_plane_wave():
    k = 7.0
    alpha = 1j / k
    y, ny, w = _product_sphere(200, 400)
    d = np.array([1.0, 2.0, -0.5])
    d /= np.linalg.norm(d)
    u = np.exp(1j * k * y @ d)
    q = 1j * k * (ny @ d) * u
    rng = np.random.default_rng(6)
    xin = np.array([_rand_unit(rng) * 0.5 for _ in range(4)])
    xout = np.array([_rand_unit(rng) * 2.0 for _ in range(4)])
    tn = np.array([_rand_unit(rng) for _ in range(4)])
    for tx, inside in ((xin, True), (xout, False)):
        lhs = (oracle.apply_targets(oracle.KIND_BMG, tx, tn, y, ny, w, k, alpha, q)
               - oracle.apply_targets(oracle.KIND_BMH, tx, tn, y, ny, w, k, alpha, u))
        ux = np.exp(1j * k * tx @ d)
        rhs = ux + alpha * 1j * k * (tn @ d) * ux if inside else 0 * ux
        assert np.abs(lhs - rhs).max() < 1e-12, (inside, np.abs(lhs - rhs).max())


def test_p6_wrong_sign_would_fail():
    """The hypersingular sign matters in P6: flipping it changes lhs at O(1)."""
    k = 7.0
    alpha = 1j / k
    y, ny, w = _product_sphere(60, 120)
    d = np.array([0.0, 0.0, 1.0])
    u = np.exp(1j * k * y @ d)
    tx = np.array([[0.1, 0.2, 0.3]])
    tn = np.array([[0.0, 0.6, 0.8]])
    hyp = oracle.apply_targets(oracle.KIND_HYP, tx, tn, y, ny, w, k, alpha, u)
    assert abs(alpha * hyp[0]) > 0.1


# --------------------------------------------------------------- P7: sphere n=0 closed form
def test_p7_sphere_monopole_mode():
    from scipy.special import spherical_jn
    k, a = 3.3, 1.0
    y, ny, w = _product_sphere(80, 160, a)
    dens = np.ones(y.shape[0], dtype=complex)
    rng = np.random.default_rng(7)
    h0p = lambda z: np.exp(1j * z) * (z + 1j) / z ** 2
    for _ in range(4):
        xh = _rand_unit(rng)
        rho = 0.4
        tx = (rho * xh)[None]
        tn = _rand_unit(rng)[None]
        dl = oracle.apply_targets(oracle.KIND_DNY, tx, None, y, ny, w, k, 0, dens)[0]
        ex = 1j * k * k * a * a * spherical_jn(0, k * rho) * h0p(k * a)
        assert abs(dl - ex) < 1e-12 * abs(ex)
        hy = oracle.apply_targets(oracle.KIND_HYP, tx, tn, y, ny, w, k, 0, dens)[0]
        ex = 1j * k ** 3 * a * a * spherical_jn(0, k * rho, derivative=True) * h0p(k * a) * (xh @ tn[0])
        assert abs(hy - ex) < 1e-11 * abs(ex)


# --------------------------------------------------------------- P8: Gauss identity
def test_p8_gauss_offsurface():
    p = synth.make_problem("x", k=1.0, nu=8)
    dens = np.ones(p.N, dtype=complex)
    tin = np.array([[0.1, -0.2, 0.3], [0.0, 0.0, 0.0]])
    tout = np.array([[1.5, 0.2, 0.0], [0.0, -3.0, 1.0]])
    vin = oracle.apply_targets(oracle.KIND_DNY, tin, None, p.x, p.n, p.w, 0.0, 0, dens)
    vout = oracle.apply_targets(oracle.KIND_DNY, tout, None, p.x, p.n, p.w, 0.0, 0, dens)
    assert np.abs(vin + 1).max() < 1e-4
    assert np.abs(vout).max() < 1e-4


def test_p8_gauss_onsurface_converges_to_half():
    errs = []
    for nu in (4, 8, 16):
        p = synth.make_problem("x", k=1.0, nu=nu)
        rows = np.arange(0, p.N, max(1, p.N // 50))
        v = oracle.apply_rows(p.x, p.n, p.w, 0.0, 0, np.ones(p.N), rows=rows, kind=oracle.KIND_DNY)
        errs.append(np.abs(v + 0.5).max())
    assert errs[2] < errs[1] < errs[0]
    assert errs[1] / errs[2] > 1.6          # first order (missing self patch)


# --------------------------------------------------------------- P9: CSR term, structure
def test_p9_csr_term_vs_scipy():
    import scipy.sparse as sp
    p = synth.make_problem("1")
    rp, col, val = p.correction(seed=9)
    phi = synth.random_phi(p.N, 1)
    rows = synth.sample_rows(p.N, 200, 2)
    a = oracle.apply_rows(p.x, p.n, p.w, p.k, p.alpha, phi, rows=rows, csr=(rp, col, val))
    b = oracle.apply_rows(p.x, p.n, p.w, p.k, p.alpha, phi, rows=rows)
    ref = (sp.csr_matrix((val, col, rp), shape=(p.N, p.N)) @ phi)[rows]
    assert np.abs((a - b) - ref).max() <= 1e-15 * np.abs(ref).max() * 10


def test_oracle_rows_subset_linearity_and_near():
    p = synth.make_problem("x", k=5.0, nu=3)
    phi1 = synth.random_phi(p.N, 1)
    phi2 = synth.random_phi(p.N, 2)
    full1 = oracle.apply_rows(p.x, p.n, p.w, p.k, p.alpha, phi1)
    full2 = oracle.apply_rows(p.x, p.n, p.w, p.k, p.alpha, phi2)
    comb = oracle.apply_rows(p.x, p.n, p.w, p.k, p.alpha, 2 * phi1 - 3j * phi2)
    assert np.abs(comb - (2 * full1 - 3j * full2)).max() < 1e-12 * np.abs(comb).max()
    rows = np.array([5, 0, 77])
    sub = oracle.apply_rows(p.x, p.n, p.w, p.k, p.alpha, phi1, rows=rows)
    assert np.array_equal(sub, full1[rows])
    # near sum with one leaf holding everything and the pair (0,0) equals the full sum
    n = p.N
    near = oracle.apply_near(p.x, p.n, p.w, p.k, p.alpha, phi1, [0, n], np.arange(n), [0, 1], [0])
    assert np.abs(near - full1).max() <= 1e-13 * np.abs(full1).max()
    # dense matrix from single kernel calls
    K = np.array([[0 if i == j else p.w[j] * oracle.kernel(4, p.x[i], p.n[i], p.x[j], p.n[j], p.k, p.alpha)
                   for j in range(n)] for i in range(0, n, 9)])
    assert np.abs(K @ phi1 - full1[::9]).max() < 1e-12 * np.abs(full1).max()


def test_p3_table1_kernel_reciprocity():
    """Kind 6, the Table-1 summation kernel G + alpha dG/dn_y, is the BM_G kernel with
    the roles of the two points exchanged: K_T1(x, n_x; y, n_y) = K_G(y, n_y; x, n_x) (G symmetric,
    d/dn_y acting on the second argument); and it is the sum of the separately pinned G and dG/dn_y."""
    rng = np.random.default_rng(11)
    for _ in range(20):
        x, y = rng.normal(size=3), rng.normal(size=3)
        a, b = _rand_unit(rng), _rand_unit(rng)
        k = rng.uniform(0.1, 30)
        al = complex(rng.normal(), rng.normal())
        t1 = oracle.kernel(oracle.KIND_T1, x, a, y, b, k, al)
        assert abs(t1 - oracle.kernel(oracle.KIND_BMG, y, b, x, a, k, al)) <= 1e-14 * abs(t1)
        parts = oracle.kernel(oracle.KIND_G, x, None, y, None, k) + al * oracle.kernel(oracle.KIND_DNY, x, None, y, b, k)
        assert abs(t1 - parts) <= 1e-14 * abs(t1)


# --------------------------------------------------------------- oracle_near: the leaf-pair restriction
def _near_brute(K, phi, members, pairs):
    """Brute force of the restricted sum from a dense kernel matrix built by single oracle.kernel calls:
    out_i = sum over listed leaf pairs (t, s) with i in t, j in s, j != i of K_ij phi_j."""
    out = np.zeros(K.shape[0], dtype=np.complex128)
    for t, s in pairs:
        for i in members[t]:
            for j in members[s]:
                if j != i:
                    out[i] += K[i, j] * phi[j]
    return out


@pytest.mark.parametrize("kind", [oracle.KIND_BMH, oracle.KIND_BMG])
def test_oracle_near_multi_leaf_pairs(kind):
    """oracle_near (the <= 1e-12 reference of the P2P parity) on >= 8 'leaves' of a random
    cloud, given as shuffled, non-contiguous point-index lists of unequal sizes:
      * all leaf pairs including self pairs  ==  oracle_rows (the whole j != i sum);
      * a random subset of pairs             ==  brute force from a dense single-call kernel matrix;
      * two disjoint halves of the pair list add up to the whole list.
    A wrong index in the pair loop (source range taken from the target leaf, a skipped self pair, the
    j != i test on leaf-local instead of global indices) fails one of these."""
    p = synth.make_problem("x", k=4.0, nu=3)      # N = 432 surface points
    N = p.N
    rng = np.random.default_rng(21)
    phi = synth.random_phi(N, 8)
    nleaf = 11
    perm = rng.permutation(N)
    cuts = np.sort(rng.choice(np.arange(1, N), nleaf - 1, replace=False))
    members = np.split(perm, cuts)
    leaf_ptr = np.concatenate([[0], np.cumsum([len(m) for m in members])])
    leaf_pts = np.concatenate(members)
    all_pairs = [(t, s) for t in range(nleaf) for s in range(nleaf)]

    def near(pairs):
        pairs = sorted(pairs)
        tgt = np.array([t for t, _ in pairs], dtype=np.int64)
        src = np.array([s for _, s in pairs], dtype=np.int64)
        pair_ptr = np.concatenate([[0], np.cumsum(np.bincount(tgt, minlength=nleaf))])
        return oracle.apply_near(p.x, p.n, p.w, p.k, p.alpha, phi, leaf_ptr, leaf_pts, pair_ptr, src, kind=kind)

    full = oracle.apply_rows(p.x, p.n, p.w, p.k, p.alpha, phi, kind=kind)
    got = near(all_pairs)
    assert np.abs(got - full).max() <= 1e-13 * np.abs(full).max()
    K = np.array([[0 if i == j else p.w[j] * oracle.kernel(kind, p.x[i], p.n[i], p.x[j], p.n[j], p.k, p.alpha)
                   for j in range(N)] for i in range(N)])
    sel = [all_pairs[i] for i in rng.choice(len(all_pairs), 40, replace=False)]
    a = near(sel)
    b = _near_brute(K, phi, members, sel)
    assert np.abs(a - b).max() <= 1e-13 * np.abs(b).max()
    # rows of targets in no listed pair are exactly zero
    listed = np.zeros(N, bool)
    for t, _ in sel:
        listed[members[t]] = True
    assert np.all(a[~listed] == 0)
    half = set(sel[:20])
    rest = [q for q in all_pairs if q not in half]
    assert np.abs(near(list(half)) + near(rest) - full).max() <= 1e-13 * np.abs(full).max()
