"""ctypes front end of the CPU oracle (``oracle/h2oracle.c``).

TEST INFRASTRUCTURE ONLY: imported by ``tests/``, ``__graft_entry__.smoke()``
(as the checker) and ``bench.py`` (cpu_baseline / ``--impl reference``).
The product package ``paper_2203_14832_b200`` never imports this module.

The oracle restates the reference h2cross algorithm for the hot path
(geometry.py:230 build_tree, compress.py:216 select_pivots, _core.pyx:70
aca_kernel, matvec.py:169 h2_matvec_reference); it is pinned against golden
vectors produced by the reference itself (tests/golden/make_golden.py).
"""

from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "_build", "libh2oracle.so")

KIND = {
    "reg-log-2d": 0,
    "reg-inverse": 1,
    "coulomb-3d": 2,
    "matern": 3,
    "gaussian": 4,
    "laplace-3d": 5,
    "log": 6,
    "gaussian-scaled": 7,
}

_i64p = ctypes.POINTER(ctypes.c_int64)
_dp = ctypes.POINTER(ctypes.c_double)
_lib = None


def build():
    subprocess.run(["make", "-s", "-C", _HERE], check=True)


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        L = ctypes.CDLL(_LIB_PATH)
        L.oh2_last_error.restype = ctypes.c_char_p
        L.oh2_build_tree.argtypes = [_dp, ctypes.c_int64, _dp, ctypes.c_int64, ctypes.c_int, ctypes.c_int,
                                     ctypes.c_int64, ctypes.c_double, ctypes.POINTER(ctypes.c_void_p)]
        L.oh2_tree_free.argtypes = [ctypes.c_void_p]
        L.oh2_tree_depth.argtypes = [ctypes.c_void_p]
        L.oh2_tree_over_capacity.argtypes = [ctypes.c_void_p]
        L.oh2_tree_root.argtypes = [ctypes.c_void_p, _dp, _dp]
        L.oh2_tree_ncells.argtypes = [ctypes.c_void_p, ctypes.c_int]
        L.oh2_tree_ncells.restype = ctypes.c_int64
        L.oh2_tree_get.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_int, _i64p]
        L.oh2_tree_get.restype = ctypes.c_int64
        L.oh2_boxes_admissible.argtypes = [_dp, ctypes.c_double, _dp, ctypes.c_double, ctypes.c_int, ctypes.c_double]
        L.oh2_kval.argtypes = [ctypes.c_int, ctypes.c_double, ctypes.c_double]
        L.oh2_kval.restype = ctypes.c_double
        L.oh2_kernel_block.argtypes = [ctypes.c_int, ctypes.c_double, _dp, ctypes.c_int64, _dp, ctypes.c_int64,
                                       ctypes.c_int, _dp]
        L.oh2_aca.argtypes = [ctypes.c_int, ctypes.c_double, _dp, ctypes.c_int64, _dp, ctypes.c_int64, ctypes.c_int,
                              ctypes.c_double, ctypes.c_int64, _dp, _dp, _i64p, _i64p,
                              ctypes.POINTER(ctypes.c_int), _i64p]
        L.oh2_aca.restype = ctypes.c_int64
        L.oh2_row_interpolator.argtypes = [_dp, ctypes.c_int64, ctypes.c_int64, _i64p, _dp]
        L.oh2_col_interpolator.argtypes = [_dp, ctypes.c_int64, ctypes.c_int64, _i64p, _dp]
        L.oh2_assemble.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_double, ctypes.c_double, ctypes.c_int,
                                   ctypes.c_int64, ctypes.POINTER(ctypes.c_void_p)]
        L.oh2_h2_free.argtypes = [ctypes.c_void_p]
        L.oh2_h2_get_i64.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_int, _i64p]
        L.oh2_h2_get_i64.restype = ctypes.c_int64
        L.oh2_h2_get_interp.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_int64, ctypes.c_int, _i64p, _dp]
        L.oh2_h2_get_interp.restype = ctypes.c_int64
        L.oh2_h2_stats.argtypes = [ctypes.c_void_p] + [_i64p] * 5
        L.oh2_matvec.argtypes = [ctypes.c_void_p, _dp, _dp, ctypes.c_int64]
        L.oh2_dense_matvec.argtypes = [ctypes.c_int, ctypes.c_double, _dp, ctypes.c_int64, _dp, ctypes.c_int64,
                                       ctypes.c_int, _dp, _dp, ctypes.c_int64]
        L.oh2_dense_rows.argtypes = [ctypes.c_int, ctypes.c_double, _dp, _i64p, ctypes.c_int64, _dp, ctypes.c_int64,
                                     ctypes.c_int, _dp, _dp]
        L.oh2_set_threads.argtypes = [ctypes.c_int]
        _lib = L
    return _lib


def _d(a):
    return a.ctypes.data_as(_dp)


def _i(a):
    return a.ctypes.data_as(_i64p)


def set_threads(n: int) -> None:
    lib().oh2_set_threads(int(n))


def threads() -> int:
    return int(lib().oh2_get_threads())


def _err():
    return lib().oh2_last_error().decode()


class OTree:
    """Oracle tree: nonempty cells per level in row-major key order."""

    FIELDS = {"key": 0, "mi": 1, "t_ptr": 2, "t_idx": 3, "s_ptr": 4, "s_idx": 5, "nb_ptr": 6, "nb_idx": 7,
              "il_ptr": 8, "il_idx": 9, "parent": 10, "ch_ptr": 11, "ch_idx": 12}

    def __init__(self, P, Q=None, nu=64, eta=float(np.sqrt(2.0))):
        self.P = np.ascontiguousarray(P, dtype=np.float64)
        self.shared = Q is None
        self.Q = self.P if Q is None else np.ascontiguousarray(Q, dtype=np.float64)
        self.d = self.P.shape[1]
        h = ctypes.c_void_p()
        rc = lib().oh2_build_tree(_d(self.P), self.P.shape[0], _d(self.Q), self.Q.shape[0], self.d,
                                  int(self.shared), int(nu), float(eta), ctypes.byref(h))
        if rc != 0:
            raise ValueError(_err())
        self.h = h
        self.depth = lib().oh2_tree_depth(h)
        self.over_capacity = bool(lib().oh2_tree_over_capacity(h))
        mid = np.zeros(self.d)
        half = ctypes.c_double()
        lib().oh2_tree_root(h, _d(mid), ctypes.byref(half))
        self.mid, self.half = mid, half.value

    def ncells(self, level):
        return int(lib().oh2_tree_ncells(self.h, level))

    def get(self, level, name):
        w = self.FIELDS[name]
        n = lib().oh2_tree_get(self.h, level, w, None)
        out = np.empty(max(n, 0), dtype=np.int64)
        if n:
            lib().oh2_tree_get(self.h, level, w, _i(out))
        return out

    def __del__(self):
        if getattr(self, "h", None):
            lib().oh2_tree_free(self.h)
            self.h = None


class OH2:
    """Oracle H2 representation (pivots + interpolation operators)."""

    def __init__(self, tree: OTree, kind: int, a: float, eps: float, force_general=False, max_rank=None):
        self.tree = tree
        h = ctypes.c_void_p()
        rc = lib().oh2_assemble(tree.h, int(kind), float(a), float(eps), int(bool(force_general)),
                                -1 if max_rank is None else int(max_rank), ctypes.byref(h))
        if rc != 0:
            raise ValueError(_err())
        self.h = h

    def get(self, level, what):
        names = {"k_in": 0, "k_out": 1, "t_in": 2, "s_in": 3, "t_out": 4, "s_out": 5, "nevals": 6, "conv_in": 7}
        w = names[what]
        n = lib().oh2_h2_get_i64(self.h, level, w, None)
        out = np.empty(max(n, 0), dtype=np.int64)
        if n > 0:
            lib().oh2_h2_get_i64(self.h, level, w, _i(out))
        return out

    def interp(self, level, cell, which=0):
        cols = ctypes.c_int64()
        rows = lib().oh2_h2_get_interp(self.h, level, int(cell), which, ctypes.byref(cols), None)
        out = np.empty((rows, cols.value))
        if rows * cols.value:
            lib().oh2_h2_get_interp(self.h, level, int(cell), which, ctypes.byref(cols), _d(out))
        return out

    def stats(self):
        vals = [ctypes.c_int64() for _ in range(5)]
        lib().oh2_h2_stats(self.h, *[ctypes.byref(v) for v in vals])
        keys = ["evals_pivots", "evals_couplings", "evals_nearfield", "max_rank", "cells_visited"]
        return {k: v.value for k, v in zip(keys, vals)}

    def matvec(self, w):
        w = np.ascontiguousarray(w, dtype=np.float64)
        nrhs = 1 if w.ndim == 1 else w.shape[1]
        u = np.empty((self.tree.P.shape[0], nrhs))
        lib().oh2_matvec(self.h, _d(w), _d(u), nrhs)
        return u[:, 0] if w.ndim == 1 else u

    def __del__(self):
        if getattr(self, "h", None):
            lib().oh2_h2_free(self.h)
            self.h = None


def aca(kind, a, X, Y, eps, cap=None):
    """Restated _core.pyx:70 aca_kernel: returns (U, V, rp, cp, converged, nevals)."""
    X = np.ascontiguousarray(X, dtype=np.float64)
    Y = np.ascontiguousarray(Y, dtype=np.float64)
    m, n, d = X.shape[0], Y.shape[0], X.shape[1]
    cap = min(m, n) if cap is None else int(cap)
    U = np.zeros((m, max(cap, 1)))
    V = np.zeros((n, max(cap, 1)))
    rp = np.zeros(max(cap, 1), dtype=np.int64)
    cp = np.zeros(max(cap, 1), dtype=np.int64)
    conv = ctypes.c_int()
    nev = ctypes.c_int64()
    k = lib().oh2_aca(int(kind), float(a), _d(X), m, _d(Y), n, d, float(eps), cap, _d(U), _d(V), _i(rp), _i(cp),
                      ctypes.byref(conv), ctypes.byref(nev))
    return U[:, :k].copy(), V[:, :k].copy(), rp[:k].copy(), cp[:k].copy(), bool(conv.value), int(nev.value)


def row_interpolator(U, rp):
    U = np.ascontiguousarray(U, dtype=np.float64)
    rp = np.ascontiguousarray(rp, dtype=np.int64)
    out = np.empty_like(U)
    if U.size:
        lib().oh2_row_interpolator(_d(U), U.shape[0], U.shape[1], _i(rp), _d(out))
    return out


def col_interpolator(V, cp):
    V = np.ascontiguousarray(V, dtype=np.float64)
    cp = np.ascontiguousarray(cp, dtype=np.int64)
    out = np.empty_like(V)
    if V.size:
        lib().oh2_col_interpolator(_d(V), V.shape[0], V.shape[1], _i(cp), _d(out))
    return out


def kernel_block(kind, a, X, Y):
    X = np.ascontiguousarray(X, dtype=np.float64)
    Y = np.ascontiguousarray(Y, dtype=np.float64)
    out = np.empty((X.shape[0], Y.shape[0]))
    lib().oh2_kernel_block(int(kind), float(a), _d(X), X.shape[0], _d(Y), Y.shape[0], X.shape[1], _d(out))
    return out


def kval(kind, a, r2):
    return float(lib().oh2_kval(int(kind), float(a), float(r2)))


def admissible(cx, hwx, cy, hwy, eta):
    cx = np.ascontiguousarray(cx, dtype=np.float64)
    cy = np.ascontiguousarray(cy, dtype=np.float64)
    return bool(lib().oh2_boxes_admissible(_d(cx), float(hwx), _d(cy), float(hwy), cx.size, float(eta)))


def dense_matvec(kind, a, P, Q, w):
    P = np.ascontiguousarray(P, dtype=np.float64)
    Q = np.ascontiguousarray(Q, dtype=np.float64)
    w = np.ascontiguousarray(w, dtype=np.float64)
    nrhs = 1 if w.ndim == 1 else w.shape[1]
    u = np.empty((P.shape[0], nrhs))
    lib().oh2_dense_matvec(int(kind), float(a), _d(P), P.shape[0], _d(Q), Q.shape[0], P.shape[1], _d(w), _d(u), nrhs)
    return u[:, 0] if w.ndim == 1 else u


def dense_rows(kind, a, P, rows, Q, w):
    P = np.ascontiguousarray(P, dtype=np.float64)
    Q = np.ascontiguousarray(Q, dtype=np.float64)
    rows = np.ascontiguousarray(rows, dtype=np.int64)
    w = np.ascontiguousarray(w, dtype=np.float64)
    u = np.empty(rows.size)
    lib().oh2_dense_rows(int(kind), float(a), _d(P), _i(rows), rows.size, _d(Q), Q.shape[0], P.shape[1], _d(w), _d(u))
    return u
