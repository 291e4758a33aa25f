"""Design exploration (not product, not oracle): accuracy / rank of LF surfaces and
HF directional equivalent sets, used to choose the plan parameters recorded in
DESIGN.md.  Pure numpy, dense, small.

  python tools/proto_ops.py lf
  python tools/proto_ops.py hf
"""
import sys
import time

import numpy as np


def G(x, y, k):
    d = x[:, None, :] - y[None, :, :]
    r = np.sqrt((d * d).sum(-1))
    return np.exp(1j * k * r) / (4 * np.pi * r)


def dGdny(x, y, ny, k):
    d = x[:, None, :] - y[None, :, :]
    r = np.sqrt((d * d).sum(-1))
    b = (d * ny[None, :, :]).sum(-1) / r
    return -np.exp(1j * k * r) * (1j * k * r - 1) / (4 * np.pi * r * r) * b


def BMeval(x, nx, y, k, alpha):
    d = x[:, None, :] - y[None, :, :]
    r = np.sqrt((d * d).sum(-1))
    a = (d * nx[:, None, :]).sum(-1) / r
    e = np.exp(1j * k * r)
    return e / (4 * np.pi * r) + alpha * e * (1j * k * r - 1) / (4 * np.pi * r * r) * a


def surface(p):
    g = np.linspace(-0.5, 0.5, p)
    X, Y, Z = np.meshgrid(g, g, g, indexing="ij")
    m = (np.abs(X) == 0.5) | (np.abs(Y) == 0.5) | (np.abs(Z) == 0.5)
    return np.stack([X[m], Y[m], Z[m]], -1)


def tsvd(R, eps):
    U, s, Vh = np.linalg.svd(R)
    r = int(np.sum(s >= eps * s[0]))
    return U[:, :r], s[:r], Vh[:r].conj().T


def rand_box(n, w, rng):
    return rng.uniform(-0.5, 0.5, (n, 3)) * w


def unit(n, rng):
    v = rng.normal(size=(n, 3))
    return v / np.linalg.norm(v, axis=1, keepdims=True)


def lf_test(w_over_lambda, p, eps, ri=1.05, ro=2.95, offsets=((2, 0, 0), (2, 2, 2), (3, 1, 0), (7, 3, 1))):
    k = 2 * np.pi
    w = w_over_lambda
    alpha = 1j / k
    rng = np.random.default_rng(0)
    S = surface(p)
    b = S * ri * w          # equivalent (inner)
    a = S * ro * w          # check (outer)
    U, s, V = tsvd(G(a, b, k), eps)
    out = []
    for off in offsets:
        off = np.array(off, float) * w
        ys = rand_box(40, w, rng)
        ny = unit(40, rng)
        q = rng.normal(size=40) + 1j * rng.normal(size=40)
        xt = rand_box(40, w, rng) + off
        nx = unit(40, rng)
        direct = BMeval  # noqa
        # direct H-type: dipole sources, BM target derivative -> build via finite kernel
        d = xt[:, None, :] - ys[None, :, :]
        r = np.sqrt((d * d).sum(-1))
        A_ = (d * nx[:, None, :]).sum(-1) / r
        B_ = (d * ny[None, :, :]).sum(-1) / r
        C_ = nx @ ny.T
        e = np.exp(1j * k * r)
        K = -e / (4 * np.pi) * ((1j * k * r - 1) * B_ / r ** 2
                                + alpha * ((3 - 3j * k * r - k * k * r * r) * A_ * B_ / r ** 3 + (1j * k * r - 1) * C_ / r ** 3))
        ref = K @ q
        xt_ = (U.conj().T @ (dGdny(a, ys, ny, k) @ q)) / s                 # S~ q
        Kt = V.T @ G(b + off, b, k) @ V                                       # K~ = V^T K V
        yt = Kt @ xt_
        rho = U.conj() @ (yt / s)                                            # incoming equivalent at a + off
        got = BMeval(xt, nx, a + off, k, alpha) @ rho
        out.append(np.linalg.norm(got - ref) / np.linalg.norm(ref))
    return len(s), out


def cmd_lf():
    for eps in (1e-5,):
        for wl in (0.05, 0.25, 0.5, 0.75, 0.99):
            for p in (6, 8, 10):
                for ri, ro in ((1.05, 2.95), (1.3, 3.0)):
                    r, errs = lf_test(wl, p, eps, ri, ro)
                    print(f"w/l={wl:5.2f} p={p:2d} ri={ri} ro={ro} s={r:4d} n={p**3-(p-2)**3:4d} err=" +
                          " ".join(f"{e:.1e}" for e in errs))


# ------------------------------------------------------------------ HF
def face_dir(v, m):
    ax = int(np.argmax(np.abs(v)))
    sgn = 1 if v[ax] > 0 else -1
    o = [i for i in range(3) if i != ax]
    u = v[o[0]] / abs(v[ax])
    t = v[o[1]] / abs(v[ax])
    a = min(m - 1, int(np.floor((u + 1) / 2 * m)))
    b = min(m - 1, int(np.floor((t + 1) / 2 * m)))
    f = 2 * ax + (0 if sgn > 0 else 1)
    return (f * m + a) * m + b


def dir_center(d, m):
    f, rem = divmod(d, m * m)
    a, b = divmod(rem, m)
    ax, neg = divmod(f, 2)
    v = np.zeros(3)
    v[ax] = -1.0 if neg else 1.0
    o = [i for i in range(3) if i != ax]
    v[o[0]] = -1 + (2 * a + 1) / m
    v[o[1]] = -1 + (2 * b + 1) / m
    return v / np.linalg.norm(v)


def rot_to(z):
    e = np.array([1.0, 0, 0])
    c = e @ z
    if c > 1 - 1e-15:
        return np.eye(3)
    if c < -1 + 1e-15:
        return np.diag([-1.0, -1.0, 1.0])
    v = np.cross(e, z)
    s = np.linalg.norm(v)
    vx = np.array([[0, -v[2], v[1]], [v[2], 0, -v[0]], [-v[1], v[0], 0]])
    return np.eye(3) + vx + vx @ vx * ((1 - c) / s ** 2)


def fib_sphere(n):
    i = np.arange(n) + 0.5
    phi = np.arccos(1 - 2 * i / n)
    th = np.pi * (1 + 5 ** 0.5) * i
    return np.stack([np.cos(th) * np.sin(phi), np.sin(th) * np.sin(phi), np.cos(phi)], -1)


def pivqr_cols(A, eps, maxr=400):
    """column-pivoted MGS, stop at residual < eps * first pivot norm. Returns selected columns."""
    A = A.copy()
    nrm = np.sum(np.abs(A) ** 2, axis=0)
    sel = []
    n0 = None
    for it in range(min(maxr, min(A.shape))):
        j = int(np.argmax(nrm))
        if n0 is None:
            n0 = np.sqrt(nrm[j])
        if np.sqrt(nrm[j]) < eps * n0:
            break
        sel.append(j)
        q = A[:, j] / np.linalg.norm(A[:, j])
        A -= np.outer(q, q.conj() @ A)
        A -= np.outer(q, q.conj() @ A)
        nrm = np.sum(np.abs(A) ** 2, axis=0)
        nrm[sel] = -1
    return np.array(sel)


def hf_sets(W, k, m, eps, rho=1.0, cone_extra=1.0, nrad=10, verbose=True):
    """canonical (e1) equivalent points (ball radius rho W) and check points (cone)."""
    lam = 2 * np.pi / k
    # cell angular radius: max angle between a cell centre and its corners, over cells
    cell = 0.0
    for d in range(6 * m * m):
        if d // (m * m) != 0:
            continue
        z = dir_center(d, m)
        f, rem = divmod(d, m * m)
        a, b = divmod(rem, m)
        for ca in (a, a + 1):
            for cb in (b, b + 1):
                v = np.array([1.0, -1 + 2 * ca / m, -1 + 2 * cb / m])
                v /= np.linalg.norm(v)
                cell = max(cell, np.arccos(np.clip(v @ z, -1, 1)))
    R = 1 + int(np.floor(k * W / np.pi))    # near radius in box units
    rmin = (R + 1) * W                       # closest non-near centre (inf-norm)
    ball = np.arcsin(min(1.0, rho * W / rmin))
    theta = cone_extra * (1.5 * cell + ball)
    # candidates for equivalent points: two spherical shells inside the ball
    nsurf = int(max(200, 6 * (2 * np.pi * rho * W / (lam / 3)) ** 2 / np.pi))
    cand = np.concatenate([fib_sphere(nsurf) * rho * W, fib_sphere(nsurf // 2) * 0.8 * rho * W])
    # check samples in the cone, 1/r uniform from rmin to "infinity"
    kR = k * rho * W
    nang = int(np.ceil(2 * theta * kR * 2.0)) + 4
    tt = np.linspace(-np.sin(theta), np.sin(theta), nang)
    TY, TZ = np.meshgrid(tt, tt, indexing="ij")
    msk = TY ** 2 + TZ ** 2 <= np.sin(theta) ** 2
    dirs = np.stack([np.sqrt(1 - TY[msk] ** 2 - TZ[msk] ** 2), TY[msk], TZ[msk]], -1)
    inv = np.linspace(1 / (rmin - rho * W), 1e-4 / rmin, nrad)
    chk = np.concatenate([dirs / iv for iv in inv])
    A = G(chk, cand, k) * np.linalg.norm(chk, axis=1)[:, None] * 4 * np.pi
    t0 = time.time()
    J = pivqr_cols(A, eps)
    b = cand[J]
    I = pivqr_cols(A[:, J].T.copy(), eps)
    a = chk[I]
    if verbose:
        print(f"  W/l={W / lam:.2f} m={m} cell={np.degrees(cell):.1f}deg ball={np.degrees(ball):.1f} theta={np.degrees(theta):.1f}"
              f" cand={cand.shape[0]} chk={chk.shape[0]} |J|={len(J)} |I|={len(I)} t={time.time() - t0:.1f}s")
    return b, a, R


def hf_test(Wl, eps=1e-5, rho=1.0, cone_extra=1.0):
    k = 2 * np.pi
    W = Wl
    m = int(np.ceil(k * W / np.pi))
    b, a, R = hf_sets(W, k, m, eps, rho, cone_extra)
    U, s, V = tsvd(G(a, b, k), eps)
    print(f"  s={len(s)} (of {len(b)})")
    rng = np.random.default_rng(1)
    errs = []
    # M2L test over all far offsets in the parent-near shell, sources in box C at 0, targets in box B
    Rp = 1 + int(np.floor(k * 2 * W / np.pi))
    offs = []
    for i in range(-2 * Rp - 1, 2 * Rp + 2):
        for j in range(-2 * Rp - 1, 2 * Rp + 2):
            for l in range(-2 * Rp - 1, 2 * Rp + 2):
                if max(abs(i), abs(j), abs(l)) > R and max(abs(i), abs(j), abs(l)) <= 2 * Rp + 1:
                    offs.append((i, j, l))
    offs = np.array(offs, float)
    pick = rng.choice(len(offs), 25, replace=False)
    worst = 0
    for off in offs[pick]:
        delta = off * W
        d = face_dir(delta, m)
        z = dir_center(d, m)
        Rz = rot_to(z)
        Rmz = rot_to(-z)
        ys = rand_box(30, W, rng)
        q = rng.normal(size=30) + 1j * rng.normal(size=30)
        xt = rand_box(30, W, rng) + delta
        ref = G(xt, ys, k) @ q
        # source outgoing in direction z: check points Rz a, equivalent Rz b
        xs = (U.conj().T @ (G(a @ Rz.T, ys, k) @ q)) / s
        # target incoming in direction -z: check points delta + Rmz b, equivalent delta + Rmz a
        Kt = V.T @ G(delta + b @ Rmz.T, b @ Rz.T, k) @ V
        yt = Kt @ xs
        rho_ = U.conj() @ (yt / s)
        got = G(xt, delta + a @ Rmz.T, k) @ rho_
        e = np.linalg.norm(got - ref) / np.linalg.norm(ref)
        worst = max(worst, e)
        errs.append(e)
    print(f"  M2L chain err: median {np.median(errs):.1e} max {worst:.1e}")


def cmd_hf():
    for Wl in (1.0, 2.0, 4.0):
        for rho in (1.0,):
            hf_test(Wl, 1e-5, rho)


if __name__ == "__main__":
    if sys.argv[1] in ("lf", "hf"):
        {"lf": cmd_lf, "hf": cmd_hf}[sys.argv[1]]()


# ---------------------------------------------------------------- HF, per-direction box sets
def box_grid(side, n):
    g = np.linspace(-0.5, 0.5, n) * side
    X, Y, Z = np.meshgrid(g, g, g, indexing="ij")
    m = (np.abs(X) == 0.5 * side) | (np.abs(Y) == 0.5 * side) | (np.abs(Z) == 0.5 * side)
    return np.stack([X[m], Y[m], Z[m]], -1)


def hf_box_sets(W, k, m, eps, d, spacing=0.25, maxrows=6000, seed=0):
    lam = 2 * np.pi / k
    R = 1 + int(np.floor(k * W / np.pi))
    Rp = 1 + int(np.floor(k * 2 * W / np.pi))
    ng = max(4, int(np.ceil(1.05 * W / (spacing * lam))) + 1)
    cand = np.concatenate([box_grid(1.05 * W, ng), box_grid(0.7 * W, max(3, int(ng * 0.7)))])
    offs = []
    L = 2 * Rp + 1
    rng = np.random.default_rng(seed)
    tb = np.concatenate([box_grid(1.05 * W, 3), np.zeros((1, 3))])   # 27-1+1 samples per target box
    rows = []
    for i in range(-L, L + 1):
        for j in range(-L, L + 1):
            for l in range(-L, L + 1):
                mx = max(abs(i), abs(j), abs(l))
                if mx <= R:
                    continue
                v = np.array([i, j, l], float)
                if face_dir(v, m) != d:
                    continue
                rows.append(v * W + tb)
    rows = np.concatenate(rows)
    if rows.shape[0] > maxrows:
        rows = rows[rng.choice(rows.shape[0], maxrows, replace=False)]
    A = G(rows, cand, k) * np.linalg.norm(rows, axis=1)[:, None]
    J = pivqr_cols(A, eps)
    I = pivqr_cols(A[:, J].T.copy(), eps)
    return cand[J], rows[I], rows.shape[0], cand.shape[0]


def hf_test2(Wl, mfac=1, eps=1e-5):
    k = 2 * np.pi
    W = Wl
    m = mfac * int(np.ceil(k * W / np.pi))
    R = 1 + int(np.floor(k * W / np.pi))
    Rp = 1 + int(np.floor(k * 2 * W / np.pi))
    rng = np.random.default_rng(2)
    # pick a few directions on face 0
    for d in [0 * m * m + (m // 2) * m + (m // 2), 0 * m * m + 0 * m + 0, (m // 2) * m + 0]:
        t0 = time.time()
        b, a, nrow, ncand = hf_box_sets(W, k, m, eps, d)
        U, s, V = tsvd(G(a, b, k), eps)
        errs = []
        L = 2 * Rp + 1
        offs = [np.array([i, j, l], float) for i in range(-L, L + 1) for j in range(-L, L + 1) for l in range(-L, L + 1)
                if max(abs(i), abs(j), abs(l)) > R and face_dir(np.array([i, j, l], float), m) == d]
        pick = rng.choice(len(offs), min(20, len(offs)), replace=False)
        for pi in pick:
            delta = offs[pi] * W
            ys = rand_box(30, W, rng)
            q = rng.normal(size=30) + 1j * rng.normal(size=30)
            xt = rand_box(30, W, rng) + delta
            ref = G(xt, ys, k) @ q
            xs = (U.conj().T @ (G(a, ys, k) @ q)) / s
            # target incoming (direction -d): points = -b, -a (central inversion of the set)
            Kt = V.T @ G(delta - b, b, k) @ V
            rho_ = U.conj() @ ((Kt @ xs) / s)
            got = G(xt, delta - a, k) @ rho_
            errs.append(np.linalg.norm(got - ref) / np.linalg.norm(ref))
        print(f"  W/l={Wl} m={m} d={d} rows={nrow} cand={ncand} |J|={len(b)} s={len(s)} "
              f"err med {np.median(errs):.1e} max {np.max(errs):.1e} t={time.time()-t0:.1f}s")


def cmd_hf2():
    for Wl in (1.0, 2.0, 4.0):
        for mfac in (1, 2):
            hf_test2(Wl, mfac)


if __name__ == "__main__" and sys.argv[1] == "hf2":
    cmd_hf2()
