"""ctypes binding of the CPU oracle (oracle/liboracle.so).

TEST INFRASTRUCTURE ONLY.  Imported by tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / --impl reference legs -- never by the product package.
The oracle restates the reference ACR H-matrix path (see acr_oracle.cpp header
for the file:line map); its parity with the reference is pinned by the
reference's own tolerance tests (tests/test_oracle_*.py).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liboracle.so")

F_CLASSES = ("gemm", "geqrf", "orgqr", "svd", "lu", "apply")


class OracleError(RuntimeError):
    def __init__(self, code, msg, level=-1, plane=-1):
        super().__init__(msg)
        self.code, self.level, self.plane = code, level, plane


class _Err(C.Structure):
    _fields_ = [("code", C.c_int), ("level", C.c_int), ("plane", C.c_int), ("msg", C.c_char * 256)]


class _Cfg(C.Structure):
    _fields_ = [("mode", C.c_int), ("eps", C.c_double), ("eta", C.c_double), ("leaf_size", C.c_int),
                ("weak", C.c_int), ("stop_planes", C.c_int), ("leaf_memory_cap", C.c_long),
                ("threads", C.c_int)]


def build():
    subprocess.run(["make", "-s", "-C", _HERE], check=True)


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        L = C.CDLL(_LIB_PATH)
        P, I, D, L_ = C.c_void_p, C.c_int, C.c_double, C.c_long
        dp, ip, lp = C.POINTER(C.c_double), C.POINTER(C.c_int), C.POINTER(C.c_long)
        ep = C.POINTER(_Err)
        sig = {
            "orc_flops_reset": (None, []),
            "orc_flops_read": (None, [dp]),
            "orc_trace_enable": (None, [I]),
            "orc_trace_read": (L_, [ip, L_]),
            "orc_bct_create": (P, [I, dp, I, D, I, ep]),
            "orc_bct_free": (None, [P]),
            "orc_bct_perm": (None, [P, ip]),
            "orc_bct_cluster_info": (None, [P, ip, ip]),
            "orc_bct_leaves": (L_, [P, ip, L_]),
            "orc_h_compress_sparse": (P, [P, L_, ip, ip, dp, D, L_, ep]),
            "orc_h_compress_dense": (P, [P, dp, D, ep]),
            "orc_h_free": (None, [P]),
            "orc_h_clone": (P, [P]),
            "orc_h_to_dense": (None, [P, dp]),
            "orc_h_apply_checked": (I, [P, I, I, dp, dp, ep]),
            "orc_h_multiply": (P, [P, P, D, ep]),
            "orc_h_multiply_add": (I, [P, P, P, D, D, ep]),
            "orc_h_add": (P, [P, P, D, D, ep]),
            "orc_h_invert": (P, [P, D, ep]),
            "orc_h_recompress": (None, [P, D]),
            "orc_h_rank_stats": (None, [P, dp, ip, ip, ip, lp]),
            "orc_h_leaf_ranks": (L_, [P, ip, L_]),
            "orc_truncate": (I, [I, I, I, dp, dp, D, D, dp, dp]),
            "orc_svd_values": (None, [I, I, dp, dp]),
            "orc_lu_inverse": (D, [I, dp, dp]),
            "orc_factor": (P, [I, I, dp, lp, ip, ip, dp, C.POINTER(_Cfg), ep]),
            "orc_factor_free": (None, [P]),
            "orc_solve": (I, [P, I, dp, dp, I, ep]),
            "orc_factor_stats": (None, [P, dp, ip, ip, ip, lp, lp]),
            "orc_level_info": (I, [P, I, ip, ip, ip, lp, ip, dp]),
            "orc_factor_dinv_ranks": (L_, [P, I, I, ip, L_]),
        }
        for name, (res, args) in sig.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def _d(a):
    return a.ctypes.data_as(C.POINTER(C.c_double))


def _i(a):
    return a.ctypes.data_as(C.POINTER(C.c_int))


def _l(a):
    return a.ctypes.data_as(C.POINTER(C.c_long))


def _check(err):
    if err.code:
        raise OracleError(err.code, err.msg.decode(), err.level, err.plane)


def flops_reset():
    lib().orc_flops_reset()


def flops_read():
    out = np.zeros(len(F_CLASSES) + 1)
    lib().orc_flops_read(_d(out))
    d = dict(zip(F_CLASSES, out[:-1]))
    d["truncations"] = out[-1]
    return d


def trace(enable=None):
    if enable is not None:
        lib().orc_trace_enable(1 if enable else 0)
        return None
    n = lib().orc_trace_read(None, 0)
    out = np.zeros((n, 6), np.int32)
    lib().orc_trace_read(_i(out), n)
    return out


class Structure:
    """ClusterTree + BlockClusterTree over plane coordinates (cluster.cpp:39-126)."""

    def __init__(self, coords, leaf=32, eta=2.0, weak=False):
        coords = np.ascontiguousarray(coords, np.float64)
        self.dim = coords.shape[0]
        err = _Err()
        self.h = lib().orc_bct_create(self.dim, _d(coords), leaf, eta, 1 if weak else 0, C.byref(err))
        _check(err)

    def __del__(self):
        if getattr(self, "h", None):
            lib().orc_bct_free(self.h)
            self.h = None

    def perm(self):
        p = np.zeros(self.dim, np.int32)
        lib().orc_bct_perm(self.h, _i(p))
        return p

    def cluster_info(self):
        a, b = C.c_int(), C.c_int()
        lib().orc_bct_cluster_info(self.h, C.byref(a), C.byref(b))
        return a.value, b.value

    def leaves(self):
        n = lib().orc_bct_leaves(self.h, None, 0)
        out = np.zeros((n, 5), np.int32)
        lib().orc_bct_leaves(self.h, _i(out), n)
        return out


class HMatrix:
    def __init__(self, handle, structure):
        self.h = handle
        self.s = structure

    def __del__(self):
        if getattr(self, "h", None):
            lib().orc_h_free(self.h)
            self.h = None

    @staticmethod
    def compress_sparse(structure, rows, cols, vals, eps, cap=2 << 30):
        rows = np.ascontiguousarray(rows, np.int32)
        cols = np.ascontiguousarray(cols, np.int32)
        vals = np.ascontiguousarray(vals, np.float64)
        err = _Err()
        h = lib().orc_h_compress_sparse(structure.h, len(vals), _i(rows), _i(cols), _d(vals), eps, cap, C.byref(err))
        _check(err)
        return HMatrix(h, structure)

    @staticmethod
    def compress_dense(structure, A, eps):
        A = np.asfortranarray(A, np.float64)
        err = _Err()
        h = lib().orc_h_compress_dense(structure.h, A.ctypes.data_as(C.POINTER(C.c_double)), eps, C.byref(err))
        _check(err)
        return HMatrix(h, structure)

    def copy(self):
        return HMatrix(lib().orc_h_clone(self.h), self.s)

    def to_dense(self):
        out = np.zeros((self.s.dim, self.s.dim), order="F")
        lib().orc_h_to_dense(self.h, out.ctypes.data_as(C.POINTER(C.c_double)))
        return out

    def apply(self, X):
        X = np.asfortranarray(X, np.float64)
        vec = X.ndim == 1
        if vec:
            X = X.reshape(-1, 1, order="F")
        Y = np.zeros_like(X, order="F")
        err = _Err()
        lib().orc_h_apply_checked(self.h, X.shape[0], X.shape[1], X.ctypes.data_as(C.POINTER(C.c_double)),
                                  Y.ctypes.data_as(C.POINTER(C.c_double)), C.byref(err))
        _check(err)
        return Y[:, 0] if vec else Y

    def multiply(self, B, eps):
        err = _Err()
        h = lib().orc_h_multiply(self.h, B.h, eps, C.byref(err))
        _check(err)
        return HMatrix(h, self.s)

    def multiply_add(self, A, B, alpha, eps):
        err = _Err()
        lib().orc_h_multiply_add(self.h, A.h, B.h, alpha, eps, C.byref(err))
        _check(err)

    def add(self, B, alpha, eps):
        err = _Err()
        h = lib().orc_h_add(self.h, B.h, alpha, eps, C.byref(err))
        _check(err)
        return HMatrix(h, self.s)

    def invert(self, eps):
        err = _Err()
        h = lib().orc_h_invert(self.h, eps, C.byref(err))
        _check(err)
        return HMatrix(h, self.s)

    def recompress(self, eps):
        lib().orc_h_recompress(self.h, eps)

    def rank_stats(self):
        a, l, nd, nr, b = C.c_double(), C.c_int(), C.c_int(), C.c_int(), C.c_long()
        lib().orc_h_rank_stats(self.h, C.byref(a), C.byref(l), C.byref(nd), C.byref(nr), C.byref(b))
        return dict(average_rank=a.value, largest_rank=l.value, dense_leaf_count=nd.value,
                    lowrank_leaf_count=nr.value, bytes=b.value)

    def leaf_ranks(self):
        n = lib().orc_h_leaf_ranks(self.h, None, 0)
        out = np.zeros(n, np.int32)
        lib().orc_h_leaf_ranks(self.h, _i(out), n)
        return out


def truncate(U, V, eps, abs_cut=0.0):
    U = np.asfortranarray(U, np.float64)
    V = np.asfortranarray(V, np.float64)
    m, K = U.shape
    n = V.shape[0]
    Uo = np.zeros((m, K), order="F")
    Vo = np.zeros((n, K), order="F")
    r = lib().orc_truncate(m, n, K, U.ctypes.data_as(C.POINTER(C.c_double)), V.ctypes.data_as(C.POINTER(C.c_double)),
                           eps, abs_cut, Uo.ctypes.data_as(C.POINTER(C.c_double)),
                           Vo.ctypes.data_as(C.POINTER(C.c_double)))
    return Uo[:, :r].copy(), Vo[:, :r].copy()


def svd_values(A):
    A = np.asfortranarray(A, np.float64)
    s = np.zeros(min(A.shape))
    lib().orc_svd_values(A.shape[0], A.shape[1], A.ctypes.data_as(C.POINTER(C.c_double)), _d(s))
    return s


def lu_inverse(A):
    A = np.asfortranarray(A, np.float64)
    inv = np.zeros_like(A, order="F")
    rc = lib().orc_lu_inverse(A.shape[0], A.ctypes.data_as(C.POINTER(C.c_double)),
                              inv.ctypes.data_as(C.POINTER(C.c_double)))
    return inv, rc


class Factorization:
    """Oracle ACR factorization (acr_factor + AcrFactorization, acr.hpp:195-224)."""

    def __init__(self, system, eps=1e-3, eta=2.0, leaf_size=32, weak=False, stop_planes=1, mode="hmatrix",
                 leaf_memory_cap=2 << 30, threads=1):
        cfg = _Cfg(0 if mode == "hmatrix" else 1, eps, eta, leaf_size, 1 if weak else 0, stop_planes,
                   leaf_memory_cap, threads)
        self.system = system
        self.threads = threads
        err = _Err()
        self.h = lib().orc_factor(system.n, system.dim, _d(system.coords), _l(system.blk_off), _i(system.rows),
                                  _i(system.cols), _d(system.vals), C.byref(cfg), C.byref(err))
        _check(err)
        self.n, self.dim = system.n, system.dim

    def __del__(self):
        if getattr(self, "h", None):
            lib().orc_factor_free(self.h)
            self.h = None

    def solve(self, f=None):
        """f: (nrhs, n, dim) or (n, dim); defaults to the system's RHS."""
        f = self.system.rhs if f is None else f
        squeeze = f.ndim == 2
        f = np.ascontiguousarray(f.reshape(-1, f.shape[-2], f.shape[-1]), np.float64)
        if f.shape[1] != self.n:
            raise OracleError(1, f"solve: right-hand side has {f.shape[1]} planes, factorization has {self.n}")
        if f.shape[2] != self.dim:
            raise OracleError(1, "solve: plane right-hand side dimension mismatch")
        u = np.zeros_like(f)
        err = _Err()
        lib().orc_solve(self.h, f.shape[0], _d(f), _d(u), self.threads, C.byref(err))
        _check(err)
        return u[0] if squeeze else u

    def stats(self):
        a, l, nd, nr, ib, fb = C.c_double(), C.c_int(), C.c_int(), C.c_int(), C.c_long(), C.c_long()
        lib().orc_factor_stats(self.h, C.byref(a), C.byref(l), C.byref(nd), C.byref(nr), C.byref(ib), C.byref(fb))
        return dict(average_rank=a.value, largest_rank=l.value, dense_leaf_count=nd.value,
                    lowrank_leaf_count=nr.value, inverse_bytes=ib.value, factor_bytes=fb.value)

    def level_info(self):
        cap = 64
        lv, pc, el, lr = (np.zeros(cap, np.int32) for _ in range(4))
        by = np.zeros(cap, np.int64)
        av = np.zeros(cap)
        k = lib().orc_level_info(self.h, cap, _i(lv), _i(pc), _i(el), _l(by), _i(lr), _d(av))
        return [dict(level=int(lv[i]), plane_count=int(pc[i]), eliminated=int(el[i]), bytes=int(by[i]),
                     largest_rank=int(lr[i]), average_rank=float(av[i])) for i in range(k)]

    def dinv_ranks(self, level, plane):
        n = lib().orc_factor_dinv_ranks(self.h, level, plane, None, 0)
        if n < 0:
            return None
        out = np.zeros(n, np.int32)
        lib().orc_factor_dinv_ranks(self.h, level, plane, _i(out), n)
        return out
