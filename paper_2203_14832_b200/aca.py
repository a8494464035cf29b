"""Partially pivoted adaptive cross approximation (aca.py of h2cross).

``partial_aca`` over a ``KernelOracle`` runs the GPU kernel
(h2b_aca_kernel, replacing _accel/_core.pyx:70 aca_kernel): one CTA, the
reference's pivot rules and exact residual arithmetic, so pivots, U and V
match the reference bit-for-bit for the IEEE-exact kernels.

The small triangular post-processing helpers (``apply_pivot_inverse``,
``row_interpolator``, ``col_interpolator``) act on the returned host
factors exactly as in the reference; inside ``assemble`` the same
operators are formed on the GPU.
"""

from __future__ import annotations

import ctypes
import warnings
from dataclasses import dataclass

import numpy as np
from scipy.linalg import solve_triangular

from . import _lib
from .kernels import EVALS, KIND_CUSTOM, KernelSpec

PIVOT_RTOL = 1e-14


@dataclass
class ACAResult:
    """Low-rank factors, pivots, and the pivot-block triangular factors (aca.py:41)."""

    row_pivots: np.ndarray
    col_pivots: np.ndarray
    row_pivots_local: np.ndarray
    col_pivots_local: np.ndarray
    u_factor: np.ndarray
    v_factor: np.ndarray
    rank: int
    pivot_lu: tuple
    converged: bool
    n_evals: int = 0

    def pivot_block(self) -> np.ndarray:
        low, up = self.pivot_lu
        return low @ up


class EntryOracle:
    """Adapts a scalar ``f(i, j)`` entry function (aca.py:60)."""

    def __init__(self, fn):
        self.fn = fn

    def row(self, i, cols):
        return np.array([self.fn(i, j) for j in cols], dtype=np.float64)

    def col(self, rows, j):
        return np.array([self.fn(i, j) for i in rows], dtype=np.float64)


class KernelOracle:
    """Entry oracle K(p_i, q_j) over a point cloud, counted in EVALS (aca.py:73)."""

    def __init__(self, kernel: KernelSpec, cloud):
        self.kernel = kernel
        self.cloud = cloud

    @property
    def fused(self) -> bool:
        return self.kernel.kind != KIND_CUSTOM

    def row(self, i, cols):
        from .kernels import raw_block

        EVALS.add(len(cols))
        return raw_block(self.kernel, self.cloud.points_p[[i]], self.cloud.points_q[np.asarray(cols)])[0]

    def col(self, rows, j):
        from .kernels import raw_block

        EVALS.add(len(rows))
        return raw_block(self.kernel, self.cloud.points_p[np.asarray(rows)], self.cloud.points_q[[j]])[:, 0]


def _empty_result(rows, cols, converged=True):
    k0 = np.empty(0, dtype=np.int64)
    return ACAResult(row_pivots=k0, col_pivots=k0.copy(), row_pivots_local=k0.copy(), col_pivots_local=k0.copy(),
                     u_factor=np.zeros((len(rows), 0)), v_factor=np.zeros((len(cols), 0)), rank=0,
                     pivot_lu=(np.zeros((0, 0)), np.zeros((0, 0))), converged=converged)


def _finish(rows, cols, U, V, rp, cp, k, converged, n_evals=0):
    rp = np.asarray(rp[:k], dtype=np.int64)
    cp = np.asarray(cp[:k], dtype=np.int64)
    U = np.ascontiguousarray(U[:, :k])
    V = np.ascontiguousarray(V[:, :k])
    low = np.tril(U[rp, :])
    up = np.triu(V[cp, :].T)
    np.fill_diagonal(up, 1.0)
    return ACAResult(row_pivots=rows[rp], col_pivots=cols[cp], row_pivots_local=rp, col_pivots_local=cp,
                     u_factor=U, v_factor=V, rank=int(k), pivot_lu=(low, up), converged=bool(converged),
                     n_evals=int(n_evals))


def aca_kernel(kind: int, a: float, X: np.ndarray, Y: np.ndarray, eps: float, cap: int):
    """GPU twin of _core.pyx:70 aca_kernel: (U, V, rp, cp, converged, nevals)."""
    X = _lib.f64(X)
    Y = _lib.f64(Y)
    m, n = X.shape[0], Y.shape[0]
    d = X.shape[1]
    cap = int(cap)
    U = np.zeros((m, max(cap, 1)))
    V = np.zeros((n, max(cap, 1)))
    rp = np.zeros(max(cap, 1), dtype=np.int64)
    cp = np.zeros(max(cap, 1), dtype=np.int64)
    conv = ctypes.c_int()
    nev = ctypes.c_int64()
    rank = ctypes.c_int64()
    _lib.check(_lib.lib().h2b_aca_kernel(int(kind), float(a), _lib.dptr(X), m, _lib.dptr(Y), n, d, float(eps), cap,
                                         _lib.dptr(U), _lib.dptr(V), _lib.iptr(rp), _lib.iptr(cp), ctypes.byref(conv),
                                         ctypes.byref(nev), ctypes.byref(rank)))
    k = rank.value
    return (np.ascontiguousarray(U[:, :k]), np.ascontiguousarray(V[:, :k]), rp[:k].copy(), cp[:k].copy(),
            bool(conv.value), int(nev.value))


def partial_aca(rows, cols, oracle, epsilon: float, max_rank: int | None = None) -> ACAResult:
    """Run partially pivoted ACA on the block A[rows, cols] (aca.py:122).

    ``oracle`` must be a ``KernelOracle`` over a built-in kernel; Python
    callables cannot run on the GPU engine and are refused.
    """
    if not epsilon > 0:
        raise ValueError("epsilon must be positive")
    rows = np.asarray(rows, dtype=np.int64)
    cols = np.asarray(cols, dtype=np.int64)
    m, n = rows.size, cols.size
    if m == 0 or n == 0:
        return _empty_result(rows, cols)
    hard_cap = min(m, n)
    cap = hard_cap if max_rank is None else min(hard_cap, int(max_rank))
    if cap == 0:
        return _empty_result(rows, cols, converged=False)
    if not isinstance(oracle, KernelOracle) or not oracle.fused:
        raise NotImplementedError("the B200 engine runs ACA only over a KernelOracle with a built-in kernel")
    kernel = oracle.kernel
    X = oracle.cloud.points_p[rows]
    Y = oracle.cloud.points_q[cols]
    U, V, rp, cp, converged, n_evals = aca_kernel(kernel.kind, kernel.device_param, X, Y, epsilon, cap)
    EVALS.add(n_evals)
    return _finish(rows, cols, U, V, rp, cp, rp.size, converged, n_evals)


def apply_pivot_inverse(result: ACAResult, rhs: np.ndarray) -> np.ndarray:
    """Apply A[tau, sigma]^{-1} to ``rhs`` via the stored triangular factors (aca.py:264)."""
    low, up = result.pivot_lu
    k = result.rank
    rhs = np.asarray(rhs, dtype=np.float64)
    if rhs.shape[0] != k:
        raise ValueError(f"rhs has {rhs.shape[0]} rows, expected {k}")
    if k == 0:
        return rhs.copy()
    b = rhs if rhs.ndim > 1 else rhs[:, None]
    diag = np.abs(np.diag(low))
    keep = k
    bad = np.flatnonzero(diag < PIVOT_RTOL * diag.max())
    if bad.size:
        keep = int(bad[0])
        warnings.warn(f"near-singular pivot block: keeping {keep} of {k} pivots", RuntimeWarning, stacklevel=2)
    out = np.zeros_like(b)
    if keep:
        y = solve_triangular(low[:keep, :keep], b[:keep], lower=True)
        out[:keep] = solve_triangular(up[:keep, :keep], y, lower=False, unit_diagonal=True)
    return out[:, 0] if rhs.ndim == 1 else out


def row_interpolator(result: ACAResult) -> np.ndarray:
    """A[:, sigma] A[tau, sigma]^{-1} == U L^{-1}, pivot rows pinned to I (aca.py:297)."""
    low, _ = result.pivot_lu
    k = result.rank
    if k == 0:
        return np.zeros((result.u_factor.shape[0], 0))
    P = solve_triangular(low.T, result.u_factor.T, lower=False).T
    P[result.row_pivots_local] = np.eye(k)
    return P


def col_interpolator(result: ACAResult) -> np.ndarray:
    """(A[tau, sigma]^{-1} A[tau, :])^T == V R^{-T}, pivot rows pinned to I (aca.py:311)."""
    _, up = result.pivot_lu
    k = result.rank
    if k == 0:
        return np.zeros((result.v_factor.shape[0], 0))
    Q = solve_triangular(up, result.v_factor.T, lower=False, unit_diagonal=True).T
    Q[result.col_pivots_local] = np.eye(k)
    return Q
