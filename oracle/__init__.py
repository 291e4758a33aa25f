"""TEST INFRASTRUCTURE ONLY -- the CPU oracle for the FDA Burton-Miller apply.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline``
/ ``--impl reference`` leg may import this package.  The product package
(``paper_1311_5202_b200``) never imports it and shares no code with it.

The arithmetic lives in ``oracle.c`` (plain C, FP64, OpenMP over rows); see its
header for the definition it computes and the PAPER.md passages it follows.
This module only marshals numpy arrays through ctypes.

Kernel kinds (``KIND_*``): G, dG/dn_y, dG/dn_x, d2G/dn_x dn_y, BM_H, BM_G, and the Table-1 summation
kernel G + alpha dG/dn_y.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = None

KIND_G, KIND_DNY, KIND_DNX, KIND_HYP, KIND_BMH, KIND_BMG, KIND_T1 = range(7)


def build():
    so = os.path.join(_HERE, "liboracle.so")
    src = os.path.join(_HERE, "oracle.c")
    subprocess.check_call(["gcc", "-O3", "-march=x86-64-v3", "-fopenmp", "-fno-fast-math", "-shared",
                           "-fPIC", src, "-o", so + ".tmp", "-lm"])
    os.replace(so + ".tmp", so)


def _lib():
    global _LIB
    if _LIB is None:
        so = os.path.join(_HERE, "liboracle.so")
        src = os.path.join(_HERE, "oracle.c")
        if not os.path.exists(so) or os.path.getmtime(so) < os.path.getmtime(src):
            build()
        lib = ctypes.CDLL(so)
        V = ctypes.c_void_p
        D = ctypes.c_double
        L = ctypes.c_int64
        lib.oracle_kernel.argtypes = [ctypes.c_int, V, V, V, V, D, D, D, V]
        lib.oracle_rows.argtypes = [ctypes.c_int, L, V, V, V, D, D, D, V, L, V, V, V, V, V]
        lib.oracle_near.argtypes = [ctypes.c_int, L, V, V, V, D, D, D, V, L, V, V, V, V, V]
        lib.oracle_targets.argtypes = [ctypes.c_int, L, V, V, L, V, V, V, D, D, D, V, V]
        lib.oracle_moments.argtypes = [ctypes.c_int, V, V, V, L, V, V, D, D, D, ctypes.c_int, V, V, D, ctypes.c_int, V]
        lib.oracle_weights_from_moments.argtypes = [V, L, V, V]
        lib.oracle_num_threads.restype = ctypes.c_int
        _LIB = lib
    return _LIB


def _p(a):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def _c128(a):
    return np.ascontiguousarray(a, dtype=np.complex128)


def num_threads() -> int:
    return int(_lib().oracle_num_threads())


def kernel(kind, x, nx, y, ny, k, alpha=0j) -> complex:
    """One kernel value K(x, n_x; y, n_y)."""
    out = np.zeros(2)
    x, y = _f64(x), _f64(y)
    nx = None if nx is None else _f64(nx)
    ny = None if ny is None else _f64(ny)
    _lib().oracle_kernel(kind, _p(x), _p(nx), _p(y), _p(ny), float(k), float(np.real(alpha)),
                         float(np.imag(alpha)), _p(out))
    return complex(out[0], out[1])


def apply_rows(x, n, w, k, alpha, phi, rows=None, csr=None, kind=KIND_BMH) -> np.ndarray:
    """out[rows] of the discrete operator: sum_{j != i} w_j K_ij phi_j + (C phi)_i."""
    x, n, w = _f64(x), _f64(n), _f64(w)
    phi = _c128(phi)
    N = x.shape[0]
    rows = np.arange(N, dtype=np.int64) if rows is None else np.ascontiguousarray(rows, dtype=np.int64)
    out = np.zeros(rows.shape[0], dtype=np.complex128)
    if csr is not None:
        rp, col, val = csr
        rp = np.ascontiguousarray(rp, dtype=np.int64)
        col = np.ascontiguousarray(col, dtype=np.int32)
        val = _c128(val)
    else:
        rp = col = val = None
    _lib().oracle_rows(kind, N, _p(x), _p(n), _p(w), float(k), float(np.real(alpha)), float(np.imag(alpha)),
                       _p(phi), rows.shape[0], _p(rows), _p(rp), _p(col), _p(val), _p(out))
    return out


def apply_near(x, n, w, k, alpha, phi, leaf_ptr, leaf_pts, pair_ptr, pair_src, kind=KIND_BMH) -> np.ndarray:
    """Sum restricted to the listed leaf pairs (j != i).  Leaves are point-index lists."""
    x, n, w = _f64(x), _f64(n), _f64(w)
    phi = _c128(phi)
    N = x.shape[0]
    out = np.zeros(N, dtype=np.complex128)
    a = [np.ascontiguousarray(v, dtype=np.int64) for v in (leaf_ptr, leaf_pts, pair_ptr, pair_src)]
    _lib().oracle_near(kind, N, _p(x), _p(n), _p(w), float(k), float(np.real(alpha)), float(np.imag(alpha)),
                       _p(phi), a[0].shape[0] - 1, _p(a[0]), _p(a[1]), _p(a[2]), _p(a[3]), _p(out))
    return out


def apply_targets(kind, tx, tn, y, ny, w, k, alpha, dens) -> np.ndarray:
    """Off-surface targets: sum_j w_j K(kind; t, tn; y_j, n_j) dens_j (no exclusion)."""
    tx = _f64(tx)
    tn = None if tn is None else _f64(tn)
    y, ny, w = _f64(y), _f64(ny), _f64(w)
    dens = _c128(dens)
    out = np.zeros(tx.shape[0], dtype=np.complex128)
    _lib().oracle_targets(kind, tx.shape[0], _p(tx), _p(tn), y.shape[0], _p(y), _p(ny), _p(w), float(k),
                          float(np.real(alpha)), float(np.imag(alpha)), _p(dens), _p(out))
    return out


def element_moments(kind, elem, tx, tn, pair_t, pair_e, k, alpha, nq=12, theta=0.25, maxdepth=24) -> np.ndarray:
    """I_n = int_Delta K(x_t, y) xi1^p xi2^q dy, (p,q) = (0,0),(1,0),(0,1),(2,0),(1,1),(0,2), per pair
    (recursive subdivision quadrature).  Returns (npairs, 6) complex."""
    elem, tx, tn = _f64(elem), _f64(tx), _f64(tn)
    pt = np.ascontiguousarray(pair_t, dtype=np.int64)
    pe = np.ascontiguousarray(pair_e, dtype=np.int64)
    g, w = np.polynomial.legendre.leggauss(int(nq))  # on [-1, 1]
    gu, gw = _f64(0.5 * (g + 1.0)), _f64(0.5 * w)
    out = np.zeros((pt.shape[0], 6), dtype=np.complex128)
    _lib().oracle_moments(kind, _p(elem), _p(tx), _p(tn), pt.shape[0], _p(pt), _p(pe), float(k),
                          float(np.real(alpha)), float(np.imag(alpha)), int(nq), _p(gu), _p(gw), float(theta),
                          int(maxdepth), _p(out))
    return out


def corrected_weights(kind, elem, xi, tx, tn, pair_t, pair_e, k, alpha, **kw) -> np.ndarray:
    """Locally corrected weights wbar_j^Delta(K; x_t): (npairs, 6) complex, j in the order
    of the quadrature points xi (6 x 2 intrinsic coordinates)."""
    mom = element_moments(kind, elem, tx, tn, pair_t, pair_e, k, alpha, **kw)
    xi = _f64(xi)
    out = np.zeros_like(mom)
    _lib().oracle_weights_from_moments(_p(xi), mom.shape[0], _p(mom), _p(out))
    return out


def rel_l2(a, b) -> float:
    """epsilon_a of PAPER.md:893-901: ||a - b||_2 / ||b||_2."""
    a = np.asarray(a)
    b = np.asarray(b)
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))
