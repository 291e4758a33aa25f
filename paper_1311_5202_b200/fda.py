"""Thin ctypes binding of libfda.so (include/fda.h).  Argument marshalling only.

Every function here has the name of the C entry point it calls.  Arrays may be
torch tensors (CUDA or CPU) or numpy arrays; they are passed by pointer.  There
is no Python or CPU implementation of any step: if libfda.so is missing the
import fails, and without a CUDA device fda_plan_create raises (FDA_ERR_CUDA).
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIBPATH = os.path.join(_HERE, "libfda.so")
if not os.path.exists(_LIBPATH):
    raise ImportError(f"{_LIBPATH} not built: run `python -m paper_1311_5202_b200.build` "
                      "(the CUDA path has no fallback)")
_lib = ctypes.CDLL(_LIBPATH)

FDA_OK = 0
STATUS = {0: "FDA_OK", 1: "FDA_ERR_INVALID_ARG", 2: "FDA_ERR_COINCIDENT_POINTS", 3: "FDA_ERR_ALIAS",
          4: "FDA_ERR_CUDA", 5: "FDA_ERR_OOM", 6: "FDA_ERR_SETUP_ACCURACY", 7: "FDA_ERR_NCCL", 8: "FDA_ERR_STATE"}
FDA_PHASE_NEAR, FDA_PHASE_CORR, FDA_PHASE_FAR, FDA_PHASE_ALL = 1, 2, 4, 7
FDA_KERNEL_BMH, FDA_KERNEL_BMG, FDA_KERNEL_T1 = 0, 1, 2
PHASES = ("permute", "p2p", "csr", "s2m", "m2m", "m2l", "l2l", "l2t", "unpermute", "exchange")
FDA_NPHASES = len(PHASES)

# every symbol include/fda.h declares (checked by tests/test_abi.py)
EXPORTS = ("fda_options_default", "fda_plan_create", "fda_plan_create_ex", "fda_plan_set_correction", "fda_apply",
           "fda_apply_phases", "fda_apply_timed", "fda_plan_set_stream", "fda_plan_stats", "fda_plan_log",
           "fda_plan_export_leaves", "fda_plan_export_p2p", "fda_plan_export_m2l", "fda_plan_destroy",
           "fda_status_str", "fda_plan_launches", "fda_nccl_unique_id", "fda_plan_create_dist", "fda_dist_counts",
           "fda_apply_up", "fda_apply_down", "fda_plan_export_exchange", "fda_nystrom_weights")


class fda_options(ctypes.Structure):
    _fields_ = [("leaf_size", ctypes.c_int32), ("eps_internal", ctypes.c_double), ("lf_p_low", ctypes.c_int32),
                ("lf_p_high", ctypes.c_int32), ("lf_p_switch", ctypes.c_double), ("lowrank", ctypes.c_int32),
                ("single_leaf", ctypes.c_int32), ("hf_max_rows", ctypes.c_int32), ("hf_spacing", ctypes.c_double),
                ("rank", ctypes.c_int32), ("nranks", ctypes.c_int32), ("verbose", ctypes.c_int32),
                ("eps_lowrank", ctypes.c_double), ("kernel", ctypes.c_int32), ("host_only", ctypes.c_int32),
                ("original", ctypes.c_int32), ("graph", ctypes.c_int32), ("deterministic", ctypes.c_int32)]


class fda_stats(ctypes.Structure):
    _fields_ = [(f, ctypes.c_int64) for f in
                ("n", "nleaves", "nlevels", "lmin", "p2p_leaf_pairs", "p2p_point_pairs", "m2l_pairs", "m2l_groups",
                 "m2l_lowrank_groups", "out_slots", "in_slots", "csr_nnz", "device_bytes", "owned_begin",
                 "owned_end", "owned_leaf_begin", "owned_leaf_end")] + \
               [(f, ctypes.c_double) for f in
                ("setup_tree_s", "setup_lists_s", "setup_ops_s", "setup_upload_s", "flops_p2p", "flops_m2l",
                 "flops_m2m", "flops_l2l", "flops_s2m", "flops_l2t", "bytes_csr")] + \
               [(f, ctypes.c_int64) for f in ("s2m_evals", "l2t_evals", "xchg_send_bytes", "xchg_recv_bytes",
                                                 "m2l_ops")] + \
               [(f, ctypes.c_double) for f in ("bytes_s2m", "bytes_l2t")]

    def as_dict(self):
        return {f: getattr(self, f) for f, _ in self._fields_}


_P = ctypes.c_void_p
_I64 = ctypes.c_int64
_D = ctypes.c_double
_lib.fda_options_default.argtypes = [ctypes.POINTER(fda_options)]
_lib.fda_options_default.restype = None
_lib.fda_plan_create.argtypes = [_I64, _P, _P, _P, _D, _D, _D, _D, ctypes.POINTER(_P)]
_lib.fda_plan_create_ex.argtypes = [_I64, _P, _P, _P, _D, _D, _D, _D, ctypes.POINTER(fda_options), ctypes.POINTER(_P)]
_lib.fda_plan_set_correction.argtypes = [_P, _I64, _P, _P, _P]
_lib.fda_apply.argtypes = [_P, _P, _P]
_lib.fda_apply_phases.argtypes = [_P, ctypes.c_uint32, _P, _P]
_lib.fda_apply_timed.argtypes = [_P, ctypes.c_uint32, _P, _P, ctypes.POINTER(ctypes.c_float)]
_lib.fda_plan_set_stream.argtypes = [_P, _P]
_lib.fda_plan_stats.argtypes = [_P, ctypes.POINTER(fda_stats)]
_lib.fda_plan_log.argtypes = [_P]
_lib.fda_plan_log.restype = ctypes.c_char_p
_lib.fda_plan_export_leaves.argtypes = [_P, ctypes.POINTER(_I64), _P, _P, _P]
_lib.fda_plan_export_p2p.argtypes = [_P, ctypes.POINTER(_I64), _P, _P]
_lib.fda_plan_export_m2l.argtypes = [_P, ctypes.POINTER(_I64), _P, _P, _P]
_lib.fda_plan_destroy.argtypes = [_P]
_lib.fda_status_str.argtypes = [ctypes.c_int]
_lib.fda_status_str.restype = ctypes.c_char_p
_lib.fda_plan_launches.argtypes = [_P]
_lib.fda_plan_launches.restype = ctypes.c_int64
_lib.fda_nccl_unique_id.argtypes = [ctypes.c_char_p]
_lib.fda_plan_create_dist.argtypes = [_I64, _P, _P, _P, _D, _D, _D, _D, ctypes.POINTER(fda_options), ctypes.c_char_p,
                                      ctypes.c_int, ctypes.c_int, ctypes.POINTER(_P)]
_lib.fda_dist_counts.argtypes = [_P, _P, _P]
_lib.fda_apply_up.argtypes = [_P, _P, _P]
_lib.fda_apply_down.argtypes = [_P, _P, _P]
_lib.fda_plan_export_exchange.argtypes = [_P, ctypes.c_int, ctypes.c_int, ctypes.POINTER(_I64), _P, _P, _P]
_lib.fda_nystrom_weights.argtypes = [ctypes.c_int, ctypes.c_double, ctypes.c_double, ctypes.c_double, _P, _I64, _P, _P,
                                     _P, _P, _I64, _P, _P, _I64, ctypes.c_int, ctypes.c_double, ctypes.c_double, ctypes.c_int, _P,
                                     _P]


class FDAError(RuntimeError):
    def __init__(self, status, where):
        super().__init__(f"{where}: {STATUS.get(status, status)}")
        self.status = status


def _check(status, where):
    if status != FDA_OK:
        raise FDAError(status, where)


def _ptr(a):
    """Data pointer of a torch tensor or numpy array (must be contiguous)."""
    if a is None:
        return None
    if hasattr(a, "data_ptr"):
        if not a.is_contiguous():
            raise ValueError("tensor must be contiguous")
        return ctypes.c_void_p(a.data_ptr())
    if isinstance(a, np.ndarray):
        if not a.flags["C_CONTIGUOUS"]:
            raise ValueError("array must be C-contiguous")
        return a.ctypes.data_as(ctypes.c_void_p)
    raise TypeError(type(a))


def fda_options_default(**kw) -> fda_options:
    o = fda_options()
    _lib.fda_options_default(ctypes.byref(o))
    for key, v in kw.items():
        setattr(o, key, v)
    return o


def fda_plan_create(points, normals, quad_weights, k, alpha, eps, options: fda_options | None = None):
    """Returns an opaque plan handle (ctypes.c_void_p).  points/normals (n,3) float64, weights (n,)."""
    n = int(points.shape[0])
    h = _P()
    a = complex(alpha)
    if options is None:
        st = _lib.fda_plan_create(n, _ptr(points), _ptr(normals), _ptr(quad_weights), float(k), a.real, a.imag,
                                  float(eps), ctypes.byref(h))
    else:
        st = _lib.fda_plan_create_ex(n, _ptr(points), _ptr(normals), _ptr(quad_weights), float(k), a.real, a.imag,
                                     float(eps), ctypes.byref(options), ctypes.byref(h))
    _check(st, "fda_plan_create")
    return h


def fda_plan_set_correction(plan, row_ptr, col, val):
    nnz = int(col.shape[0])
    _check(_lib.fda_plan_set_correction(plan, nnz, _ptr(row_ptr), _ptr(col), _ptr(val)), "fda_plan_set_correction")


def fda_apply(plan, phi, out):
    _check(_lib.fda_apply(plan, _ptr(phi), _ptr(out)), "fda_apply")


def fda_apply_phases(plan, mask, phi, out):
    _check(_lib.fda_apply_phases(plan, int(mask), _ptr(phi), _ptr(out)), "fda_apply_phases")


def fda_apply_timed(plan, mask, phi, out):
    ms = (ctypes.c_float * FDA_NPHASES)()
    _check(_lib.fda_apply_timed(plan, int(mask), _ptr(phi), _ptr(out), ms), "fda_apply_timed")
    return dict(zip(PHASES, list(ms)))


def fda_plan_set_stream(plan, stream_handle: int):
    _check(_lib.fda_plan_set_stream(plan, ctypes.c_void_p(stream_handle)), "fda_plan_set_stream")


def fda_plan_stats(plan) -> dict:
    s = fda_stats()
    _check(_lib.fda_plan_stats(plan, ctypes.byref(s)), "fda_plan_stats")
    return s.as_dict()


def fda_plan_log(plan) -> str:
    return (_lib.fda_plan_log(plan) or b"").decode()


def fda_plan_export_leaves(plan, n):
    nl = _I64()
    _check(_lib.fda_plan_export_leaves(plan, ctypes.byref(nl), None, None, None), "fda_plan_export_leaves")
    lop = np.empty(n, np.int32)
    lev = np.empty(nl.value, np.int32)
    ijk = np.empty((nl.value, 3), np.int64)
    _check(_lib.fda_plan_export_leaves(plan, ctypes.byref(nl), _ptr(lop), _ptr(lev), _ptr(ijk)),
           "fda_plan_export_leaves")
    return lop, lev, ijk


def fda_plan_export_p2p(plan):
    npairs = _I64()
    _check(_lib.fda_plan_export_p2p(plan, ctypes.byref(npairs), None, None), "fda_plan_export_p2p")
    t = np.empty(npairs.value, np.int32)
    s = np.empty(npairs.value, np.int32)
    _check(_lib.fda_plan_export_p2p(plan, ctypes.byref(npairs), _ptr(t), _ptr(s)), "fda_plan_export_p2p")
    return t, s


def fda_plan_export_m2l(plan):
    npairs = _I64()
    _check(_lib.fda_plan_export_m2l(plan, ctypes.byref(npairs), None, None, None), "fda_plan_export_m2l")
    lev = np.empty(npairs.value, np.int32)
    t = np.empty((npairs.value, 3), np.int64)
    s = np.empty((npairs.value, 3), np.int64)
    _check(_lib.fda_plan_export_m2l(plan, ctypes.byref(npairs), _ptr(lev), _ptr(t), _ptr(s)), "fda_plan_export_m2l")
    return lev, t, s


def fda_nccl_unique_id() -> bytes:
    """128-byte NCCL unique id (rank 0 makes it; the caller distributes it)."""
    buf = ctypes.create_string_buffer(128)
    _check(_lib.fda_nccl_unique_id(buf), "fda_nccl_unique_id")
    return buf.raw


def fda_plan_create_dist(points, normals, quad_weights, k, alpha, eps, nccl_id: bytes, rank: int, nranks: int,
                         options: fda_options | None = None):
    """Collective plan over nranks processes (one GPU each); fda_apply then returns the full out on every rank."""
    if len(nccl_id) != 128:
        raise ValueError("nccl_id must be the 128 bytes of fda_nccl_unique_id()")
    n = int(points.shape[0])
    h = _P()
    a = complex(alpha)
    opt = options if options is not None else fda_options_default()
    _check(_lib.fda_plan_create_dist(n, _ptr(points), _ptr(normals), _ptr(quad_weights), float(k), a.real, a.imag,
                                     float(eps), ctypes.byref(opt), ctypes.create_string_buffer(nccl_id, 128),
                                     int(rank), int(nranks), ctypes.byref(h)), "fda_plan_create_dist")
    return h


def fda_dist_counts(plan, nranks: int):
    """(send_counts, recv_counts) per peer, complex128 elements."""
    s = np.zeros(nranks, np.int64)
    r = np.zeros(nranks, np.int64)
    _check(_lib.fda_dist_counts(plan, _ptr(s), _ptr(r)), "fda_dist_counts")
    return s, r


def fda_apply_up(plan, phi, sendbuf):
    _check(_lib.fda_apply_up(plan, _ptr(phi), _ptr(sendbuf)), "fda_apply_up")


def fda_apply_down(plan, recvbuf, out):
    _check(_lib.fda_apply_down(plan, _ptr(recvbuf), _ptr(out)), "fda_apply_down")


def fda_plan_export_exchange(plan, peer: int, recv: bool):
    """(level, slot, cube_ijk) of the entries this rank sends to (recv=False) / receives from (True) peer."""
    cnt = _I64()
    _check(_lib.fda_plan_export_exchange(plan, int(peer), int(recv), ctypes.byref(cnt), None, None, None),
           "fda_plan_export_exchange")
    lev = np.empty(cnt.value, np.int32)
    slot = np.empty(cnt.value, np.int64)
    ijk = np.empty((cnt.value, 3), np.int64)
    _check(_lib.fda_plan_export_exchange(plan, int(peer), int(recv), ctypes.byref(cnt), _ptr(lev), _ptr(slot),
                                         _ptr(ijk)), "fda_plan_export_exchange")
    return lev, slot, ijk


def fda_nystrom_weights(kernel, k, alpha, elem_nodes, xi, wref, tx, tn, pair_t, pair_e, wbar=None, delta=None,
                        nq=0, theta=0.0, gamma=0.0, max_depth=0):
    """Locally corrected weights of (field point, element) pairs (include/fda.h).  elem_nodes (ne, 6, 3),
    xi (6, 2), wref (6), tx / tn (nt, 3), pair_t / pair_e int64 (npairs); wbar / delta (npairs, 6) complex128,
    filled in place (numpy arrays or torch tensors, host or device)."""
    alpha = complex(alpha)
    ne = int(elem_nodes.shape[0])
    nt = int(tx.shape[0])
    npairs = int(pair_t.shape[0])
    _check(_lib.fda_nystrom_weights(int(kernel), float(k), alpha.real, alpha.imag, _ptr(elem_nodes), ne, _ptr(xi),
                                    _ptr(wref), _ptr(tx), _ptr(tn), nt, _ptr(pair_t), _ptr(pair_e), npairs, int(nq),
                                    float(theta), float(gamma), int(max_depth), _ptr(wbar), _ptr(delta)),
           "fda_nystrom_weights")


def fda_plan_destroy(plan):
    _check(_lib.fda_plan_destroy(plan), "fda_plan_destroy")


def fda_plan_launches(plan) -> int:
    return int(_lib.fda_plan_launches(plan))


def fda_status_str(status: int) -> str:
    return _lib.fda_status_str(int(status)).decode()


class Plan:
    """Convenience owner of a plan handle (destroyed on close / garbage collection)."""

    def __init__(self, points, normals, quad_weights, k, alpha, eps=1e-4, **options):
        self.n = int(points.shape[0])
        opt = fda_options_default(**options) if options else None
        self.h = fda_plan_create(points, normals, quad_weights, k, alpha, eps, opt)

    def set_correction(self, row_ptr, col, val):
        fda_plan_set_correction(self.h, row_ptr, col, val)

    def apply(self, phi, out, mask=FDA_PHASE_ALL):
        if mask == FDA_PHASE_ALL:
            fda_apply(self.h, phi, out)
        else:
            fda_apply_phases(self.h, mask, phi, out)
        return out

    def apply_timed(self, phi, out, mask=FDA_PHASE_ALL):
        return fda_apply_timed(self.h, mask, phi, out)

    def stats(self):
        return fda_plan_stats(self.h)

    def log(self):
        return fda_plan_log(self.h)

    def close(self):
        if getattr(self, "h", None) is not None:
            fda_plan_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
