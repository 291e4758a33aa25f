"""Seeded synthetic inputs shaped like the paper's workloads.

This package is the INPUT GENERATOR shared by the oracle tests, the GPU parity
tests and ``bench.py``.  It holds none of the method's arithmetic (no Green's
function, no kernel, no FDA step): only geometry (meshes, the 6-point rule,
normals, weights), the local-region sparsity pattern D_i and seeded random
numbers.  See DESIGN.md "input recipe".

Sources in the paper:
  * curved quadratic triangles, 6-point Gauss rule, N = 6 N_e
  * far-field quadrature weights w_j (rule weight x Jacobian)
  * local region D_i (elements within 2x their largest side)
  * random densities with mean 0
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = None

# Degree-4 symmetric 6-point triangle rule: two orbits of three
# points, barycentric (a, a, 1-2a) and (b, b, 1-2b); weights are fractions of
# the triangle area (they sum to 1).
RULE_A = 0.091576213509771
RULE_B = 0.445948490915965
RULE_WA = 0.109951743655322
RULE_WB = 0.223381589678011


def rule_points():
    """(xi1, xi2, area-fraction) of the 6 points, reference triangle (0,0),(1,0),(0,1)."""
    a, b = RULE_A, RULE_B
    pts = [(a, a, RULE_WA), (1 - 2 * a, a, RULE_WA), (a, 1 - 2 * a, RULE_WA),
           (b, b, RULE_WB), (1 - 2 * b, b, RULE_WB), (b, 1 - 2 * b, RULE_WB)]
    return np.array(pts, dtype=np.float64)


def shape_functions(xi1, xi2):
    """6-node isoparametric triangle: corners 1,2,3 then mid-edges 12,23,31.

    Returns (N[6], dN/dxi1[6], dN/dxi2[6]) for arrays xi1, xi2 (broadcast on a new last axis)."""
    xi1 = np.asarray(xi1, dtype=np.float64)[..., None]
    xi2 = np.asarray(xi2, dtype=np.float64)[..., None]
    l1 = 1.0 - xi1 - xi2
    l2 = xi1
    l3 = xi2
    N = np.concatenate([l1 * (2 * l1 - 1), l2 * (2 * l2 - 1), l3 * (2 * l3 - 1),
                        4 * l1 * l2, 4 * l2 * l3, 4 * l3 * l1], axis=-1)
    # d/dxi1: dl1 = -1, dl2 = 1, dl3 = 0
    d1 = np.concatenate([-(4 * l1 - 1), (4 * l2 - 1), 0 * l3,
                         4 * (l1 - l2), 4 * l3, -4 * l3], axis=-1)
    # d/dxi2: dl1 = -1, dl2 = 0, dl3 = 1
    d2 = np.concatenate([-(4 * l1 - 1), 0 * l2, (4 * l3 - 1),
                         -4 * l2, 4 * l2, 4 * (l1 - l3)], axis=-1)
    return N, d1, d2


def octa_sphere(nu: int, radius: float = 1.0) -> np.ndarray:
    """Frequency-nu octahedral geodesic sphere of curved quadratic triangles.

    8 nu^2 elements (nu = 8 gives the 512 elements / N = 3072 of
    config 1).  Corner and mid-edge nodes are the flat subdivision points
    projected radially onto the sphere.  Returns nodes (Ne, 6, 3), counter-
    clockwise seen from outside (outward normals).
    """
    elems = []
    for s1 in (1, -1):
        for s2 in (1, -1):
            for s3 in (1, -1):
                A = np.array([s1, 0, 0], float)
                B = np.array([0, s2, 0], float)
                C = np.array([0, 0, s3], float)
                if s1 * s2 * s3 < 0:
                    B, C = C, B
                # integer lattice i,j on the face: P = A + i/nu (B-A) + j/nu (C-A)
                ii, jj = [], []
                for i in range(nu):
                    for j in range(nu - i):
                        ii.append((i, j, i + 1, j, i, j + 1))          # up triangle
                        if i + j + 2 <= nu:
                            jj.append((i + 1, j, i + 1, j + 1, i, j + 1))  # down triangle
                tri = np.array(ii + jj, dtype=np.float64)  # (T, 6): three (i,j) corners

                def P(i, j):
                    return A[None, :] + (i[:, None] / nu) * (B - A)[None, :] + (j[:, None] / nu) * (C - A)[None, :]

                c1 = P(tri[:, 0], tri[:, 1])
                c2 = P(tri[:, 2], tri[:, 3])
                c3 = P(tri[:, 4], tri[:, 5])
                nodes = np.stack([c1, c2, c3, 0.5 * (c1 + c2), 0.5 * (c2 + c3), 0.5 * (c3 + c1)], axis=1)
                elems.append(nodes)
    nodes = np.concatenate(elems, axis=0)
    nodes = radius * nodes / np.linalg.norm(nodes, axis=-1, keepdims=True)
    return nodes


def cube_sphere(m: int, radius: float = 1.0) -> np.ndarray:
    """Equiangular cube-sphere of curved quadratic triangles: m x m cells per cube face, 2 triangles per
    cell, 12 m^2 elements, N = 72 m^2 quadrature points -- the point counts of PAPER.md Table 1
    (73,728 * 4^j at m = 32 * 2^j).  Nodes: corners and mid-edges in the face's angular
    coordinates mapped radially onto the sphere; counter-clockwise seen from outside."""
    t = np.linspace(-np.pi / 4, np.pi / 4, 2 * m + 1)          # half-cell steps (mid-edge nodes)
    elems = []
    for ax in range(3):
        for sgn in (1.0, -1.0):
            o0, o1 = [a for a in range(3) if a != ax]

            def P(i, j):
                v = np.zeros(np.broadcast(i, j).shape + (3,))
                v[..., ax] = sgn
                v[..., o0] = np.tan(t[i])
                v[..., o1] = np.tan(t[j])
                return v

            I, J = np.meshgrid(np.arange(m), np.arange(m), indexing="ij")
            a, b = 2 * I.ravel(), 2 * J.ravel()
            # two triangles per cell: (00, 20, 22) and (00, 22, 02) in half-step indices
            for (i1, j1), (i2, j2), (i3, j3) in (((0, 0), (2, 0), (2, 2)), ((0, 0), (2, 2), (0, 2))):
                c1, c2, c3 = P(a + i1, b + j1), P(a + i2, b + j2), P(a + i3, b + j3)
                m12 = P(a + (i1 + i2) // 2, b + (j1 + j2) // 2)
                m23 = P(a + (i2 + i3) // 2, b + (j2 + j3) // 2)
                m31 = P(a + (i3 + i1) // 2, b + (j3 + j1) // 2)
                elems.append(np.stack([c1, c2, c3, m12, m23, m31], axis=1))
    nodes = np.concatenate(elems, axis=0)
    nodes = radius * nodes / np.linalg.norm(nodes, axis=-1, keepdims=True)
    e1 = nodes[:, 1] - nodes[:, 0]
    e2 = nodes[:, 2] - nodes[:, 0]
    flip = np.einsum('ij,ij->i', np.cross(e1, e2), nodes[:, :3].mean(axis=1)) < 0
    nodes[flip] = nodes[flip][:, [0, 2, 1, 5, 4, 3]]
    return nodes


def spheroid(a: float, b: float, h: float) -> np.ndarray:
    """Prolate spheroid x^2/a^2 + (y^2+z^2)/b^2 = 1 meshed by rings.

    Rings equally spaced (step ~h) in meridian arc length; each ring carries
    n = max(3, round(2 pi rho / h)) nodes; consecutive rings are zipped into
    triangles; mid-edge nodes are flat midpoints mapped radially onto the surface.
    Returns nodes (Ne, 6, 3) oriented outward.
    """
    # meridian: (x, rho) = (a cos t, b sin t), t in [0, pi]
    t = np.linspace(0.0, np.pi, 200001)
    dx = -a * np.sin(t)
    dr = b * np.cos(t)
    ds = np.sqrt(dx * dx + dr * dr)
    s = np.concatenate([[0.0], np.cumsum(0.5 * (ds[1:] + ds[:-1]) * np.diff(t))])
    L = s[-1]
    nr = max(2, int(round(L / h)))
    sk = np.linspace(0.0, L, nr + 1)
    tk = np.interp(sk, s, t)
    xs = a * np.cos(tk)
    rs = b * np.sin(tk)
    rings = []
    for q in range(nr + 1):
        if q == 0 or q == nr:
            rings.append(np.array([[xs[q], 0.0, 0.0]]))
            continue
        m = max(3, int(round(2 * np.pi * rs[q] / h)))
        phase = 0.5 * (q % 2) * 2 * np.pi / m
        ang = phase + 2 * np.pi * np.arange(m) / m
        rings.append(np.stack([np.full(m, xs[q]), rs[q] * np.cos(ang), rs[q] * np.sin(ang)], axis=1))

    def angle(p):
        return np.mod(np.arctan2(p[:, 2], p[:, 1]), 2 * np.pi)

    tris = []
    for q in range(nr):
        R0, R1 = rings[q], rings[q + 1]
        n0, n1 = len(R0), len(R1)
        if n0 == 1:
            for j in range(n1):
                tris.append((R0[0], R1[j], R1[(j + 1) % n1]))
            continue
        if n1 == 1:
            for i in range(n0):
                tris.append((R0[i], R1[0], R0[(i + 1) % n0]))
            continue
        a0 = angle(R0)
        a1 = angle(R1)
        # unwrap both rings to start at the same angle and zip by angle
        i0 = int(np.argmin(a0))
        i1 = int(np.argmin(a1))
        o0 = [(i0 + k) % n0 for k in range(n0 + 1)]
        o1 = [(i1 + k) % n1 for k in range(n1 + 1)]
        u0 = np.unwrap(a0[o0])
        u1 = np.unwrap(a1[o1])
        u0 = u0 - 2 * np.pi * np.floor((u0[0] - 0.0) / (2 * np.pi))
        u1 = u1 - 2 * np.pi * np.floor((u1[0] - 0.0) / (2 * np.pi))
        i, j = 0, 0
        while i < n0 or j < n1:
            if j >= n1 or (i < n0 and u0[i + 1] <= u1[j + 1]):
                tris.append((R0[o0[i]], R1[o1[j]], R0[o0[i + 1]]))
                i += 1
            else:
                tris.append((R0[o0[i]], R1[o1[j]], R1[o1[j + 1]]))
                j += 1
    tri = np.array(tris)  # (T, 3, 3)
    c1, c2, c3 = tri[:, 0], tri[:, 1], tri[:, 2]
    nodes = np.stack([c1, c2, c3, 0.5 * (c1 + c2), 0.5 * (c2 + c3), 0.5 * (c3 + c1)], axis=1)
    scale = np.sqrt(nodes[..., 0] ** 2 / a ** 2 + (nodes[..., 1] ** 2 + nodes[..., 2] ** 2) / b ** 2)
    nodes = nodes / scale[..., None]
    # orient outward: flip element if its centroid normal points inward
    e1 = nodes[:, 1] - nodes[:, 0]
    e2 = nodes[:, 2] - nodes[:, 0]
    nrm = np.cross(e1, e2)
    cen = nodes[:, :3].mean(axis=1)
    flip = np.einsum('ij,ij->i', nrm, cen) < 0
    nodes[flip] = nodes[flip][:, [0, 2, 1, 5, 4, 3]]
    return nodes


def quadrature_cloud(nodes: np.ndarray):
    """Nyström points of a quadratic mesh.

    Returns x (N,3), n (N,3) unit outward normals, w (N,) = rule weight x Jacobian,
    hmax (Ne,) largest side length (sum of the two half-chords through the mid-edge node),
    samples (Ne,12,3) = 6 nodes then 6 quadrature points (for D_i).
    Point 6e+q belongs to element e.
    """
    rp = rule_points()
    N, d1, d2 = shape_functions(rp[:, 0], rp[:, 1])        # (6 q, 6 n)
    x = np.einsum('qn,enk->eqk', N, nodes)
    t1 = np.einsum('qn,enk->eqk', d1, nodes)
    t2 = np.einsum('qn,enk->eqk', d2, nodes)
    cr = np.cross(t1, t2)
    jac = np.linalg.norm(cr, axis=-1)
    nrm = cr / jac[..., None]
    w = 0.5 * rp[None, :, 2] * jac                           # reference-triangle area 1/2
    ne = nodes.shape[0]

    def L(a, b):
        return np.linalg.norm(nodes[:, a] - nodes[:, b], axis=-1)

    hmax = np.maximum.reduce([L(0, 3) + L(3, 1), L(1, 4) + L(4, 2), L(2, 5) + L(5, 0)])
    samples = np.concatenate([nodes, x], axis=1)
    return (np.ascontiguousarray(x.reshape(ne * 6, 3)), np.ascontiguousarray(nrm.reshape(ne * 6, 3)),
            np.ascontiguousarray(w.reshape(ne * 6)), hmax, np.ascontiguousarray(samples))


# ---------------------------------------------------------------- C helper
def _lib():
    global _LIB
    if _LIB is None:
        so = os.path.join(_HERE, "libcsynth.so")
        src = os.path.join(_HERE, "csynth.c")
        if not os.path.exists(so) or os.path.getmtime(so) < os.path.getmtime(src):
            build()
        lib = ctypes.CDLL(so)
        lib.csynth_local_regions.restype = ctypes.c_int64
        lib.csynth_local_regions.argtypes = [ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p,
                                             ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]
        lib.csynth_fill_csr.restype = None
        lib.csynth_fill_csr.argtypes = [ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                        ctypes.c_void_p, ctypes.c_double, ctypes.c_uint64,
                                        ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]
        lib.csynth_u11.restype = ctypes.c_double
        lib.csynth_u11.argtypes = [ctypes.c_uint64] * 4
        _LIB = lib
    return _LIB


def build():
    so = os.path.join(_HERE, "libcsynth.so")
    src = os.path.join(_HERE, "csynth.c")
    subprocess.check_call(["gcc", "-O3", "-fopenmp", "-shared", "-fPIC", src, "-o", so + ".tmp", "-lm"])
    os.replace(so + ".tmp", so)


def _p(a):
    return a.ctypes.data_as(ctypes.c_void_p)


def local_regions(samples, hmax, x):
    """D_i element lists.  Returns (elem_ptr int64[n+1], elem_idx int32[...])."""
    lib = _lib()
    samples = np.ascontiguousarray(samples, dtype=np.float64)
    hmax = np.ascontiguousarray(hmax, dtype=np.float64)
    x = np.ascontiguousarray(x, dtype=np.float64)
    ne, n = samples.shape[0], x.shape[0]
    ptr = np.zeros(n + 1, dtype=np.int64)
    tot = lib.csynth_local_regions(ne, _p(samples), _p(hmax), n, _p(x), _p(ptr), None)
    if tot < 0:
        raise MemoryError("csynth_local_regions failed")
    idx = np.empty(int(tot), dtype=np.int32)
    tot2 = lib.csynth_local_regions(ne, _p(samples), _p(hmax), n, _p(x), _p(ptr), _p(idx))
    if tot2 != tot:
        raise RuntimeError("csynth_local_regions: inconsistent passes")
    return ptr, idx


def correction_csr(elem_ptr, elem_idx, w, hmax, kref, seed):
    """Synthetic correction CSR on the D_i pattern (DESIGN.md input recipe)."""
    lib = _lib()
    n = elem_ptr.shape[0] - 1
    nnz = 6 * int(elem_ptr[-1])
    row_ptr = np.empty(n + 1, dtype=np.int64)
    col = np.empty(nnz, dtype=np.int32)
    val = np.empty(2 * nnz, dtype=np.float64)
    w = np.ascontiguousarray(w, dtype=np.float64)
    hmax = np.ascontiguousarray(hmax, dtype=np.float64)
    lib.csynth_fill_csr(n, _p(elem_ptr), _p(elem_idx), _p(w), _p(hmax), float(max(kref, 1.0)),
                        ctypes.c_uint64(seed), _p(row_ptr), _p(col), _p(val))
    return row_ptr, col, val.view(np.complex128)


def counter_u11(seed, i, j, lane):
    return _lib().csynth_u11(seed, i, j, lane)


def random_phi(n: int, seed: int) -> np.ndarray:
    """Densities with Re, Im i.i.d. U(-1,1) ("randomly defined with mean 0")."""
    rng = np.random.default_rng(seed)
    v = rng.uniform(-1.0, 1.0, size=(n, 2))
    return np.ascontiguousarray(v[:, 0] + 1j * v[:, 1])


def plane_wave(x: np.ndarray, k: float, d=(0.0, 0.6, 0.8)) -> np.ndarray:
    """Smooth density phi_j = e^{ik d.x_j}, |d| = 1: the incident plane wave of PAPER.md:1043-1048, used as a
    density whose far field does not cancel (the random density's far field largely does)."""
    d = np.asarray(d, dtype=np.float64)
    d = d / np.linalg.norm(d)
    return np.ascontiguousarray(np.exp(1j * float(k) * (np.asarray(x) @ d)))


def sample_rows(n: int, count: int, seed: int) -> np.ndarray:
    """Seeded target-row sample."""
    if count >= n:
        return np.arange(n, dtype=np.int64)
    return np.sort(np.random.default_rng(seed).choice(n, count, replace=False)).astype(np.int64)


# ---------------------------------------------------------------- configs
@dataclass
class Problem:
    name: str
    x: np.ndarray        # (N,3)
    n: np.ndarray        # (N,3)
    w: np.ndarray        # (N,)
    k: float
    alpha: complex
    eps: float
    nodes: np.ndarray    # (Ne,6,3)
    hmax: np.ndarray
    samples: np.ndarray

    @property
    def N(self):
        return self.x.shape[0]

    def correction(self, seed: int = 7):
        ptr, idx = local_regions(self.samples, self.hmax, self.x)
        return correction_csr(ptr, idx, self.w, self.hmax, self.k, seed)


# name -> (geometry, geometry params, k)
#   1  : N=3072, kD=10      (BASELINE.json configs[0]; octahedral nu=8)
#   1b : N=49152, kD=100    (parity-only)
#   1c : N=101568, kD=400   (parity-only)
#   2  : N=196608, kD=1     (configs[1])
#   3  : N=397488, kD=100   (configs[2])
#   4  : prolate 10:1:1, N~1M, kD=400 along the long axis (configs[3])
#   5  : N=4009008, kD=1000 (configs[4]; the bench workload)
CONFIGS = {
    "1": ("sphere", 8, 5.0),
    "1b": ("sphere", 32, 50.0),
    "1c": ("sphere", 46, 200.0),
    "2": ("sphere", 64, 0.5),
    "3": ("sphere", 91, 50.0),
    "4": ("spheroid", 0.0345, 20.0),
    "5": ("sphere", 289, 500.0),
    # Table-1 workloads: cube-sphere, ~20 points per wavelength, N = 73,728 * 4^j
    "t1": ("cubesphere", 32, 8 * np.pi),
    "t1b": ("cubesphere", 64, 16 * np.pi),
    "t1c": ("cubesphere", 128, 32 * np.pi),
    "t1d": ("cubesphere", 256, 64 * np.pi),
}


def make_problem(name: str, eps: float = 1e-4, k: float | None = None, nu: int | None = None) -> Problem:
    geo, par, kk = CONFIGS[name] if name in CONFIGS else ("sphere", nu, k)
    if k is not None:
        kk = k
    if nu is not None and geo == "sphere":
        par = nu
    if geo == "sphere":
        nodes = octa_sphere(int(par), 1.0)
    elif geo == "cubesphere":
        nodes = cube_sphere(int(par), 1.0)
    else:
        nodes = spheroid(10.0, 1.0, float(par))
    x, n, w, hmax, samples = quadrature_cloud(nodes)
    return Problem(name, x, n, w, float(kk), 1j / float(kk), eps, nodes, hmax, samples)
