"""H2 compression by nested cross approximation, on the GPU.

Same surface as h2cross/compress.py.  ``assemble`` (compress.py:285) calls
h2b_assemble: one bottom-up level sweep, every cell's ACA run as one CTA,
interpolation operators formed from the ACA factors on the device (no extra
kernel entries, Remark 2).  Coupling blocks S_{X,Y} = K(t_in^X, s_out^Y) and
near-field blocks are not stored — the matvec regenerates them in registers —
so ``H2Matrix.couplings`` / ``.nearfield`` are lazy views that evaluate a
block on the GPU when it is indexed.
"""

from __future__ import annotations

import ctypes
import time
from collections.abc import Mapping
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .geometry import Cell, HierTree
from .kernels import EVALS, KernelSpec, raw_block

_EMPTY = np.empty(0, dtype=np.int64)

TOP_COMPRESSED_LEVEL = 2  # compress.py:40


@dataclass
class PivotSet:
    """Per-cell pivot index sets (global point indices)."""

    t_in: np.ndarray = field(default_factory=lambda: _EMPTY)
    s_in: np.ndarray = field(default_factory=lambda: _EMPTY)
    t_out: np.ndarray = field(default_factory=lambda: _EMPTY)
    s_out: np.ndarray = field(default_factory=lambda: _EMPTY)

    @property
    def rank_in(self) -> int:
        return self.t_in.size

    @property
    def rank_out(self) -> int:
        return self.s_out.size

    def max_cardinality(self) -> int:
        return max(self.t_in.size, self.s_in.size, self.t_out.size, self.s_out.size)


@dataclass
class TransferOps:
    """Per-cell basis/translation operators (compress.py:65)."""

    l2p: np.ndarray | None = None
    p2m: np.ndarray | None = None
    l2l: dict = field(default_factory=dict)
    m2m: dict = field(default_factory=dict)


@dataclass
class Candidates:
    t_in: np.ndarray
    s_in: np.ndarray
    t_out: np.ndarray
    s_out: np.ndarray
    in_slices: list = field(default_factory=list)
    out_slices: list = field(default_factory=list)


@dataclass
class H2Stats:
    n_targets: int = 0
    n_sources: int = 0
    max_rank: int = 0
    memory_bytes: int = 0
    assembly_seconds: float = 0.0
    entry_evaluations: int = 0
    evals_pivots: int = 0
    evals_transfers: int = 0
    evals_couplings: int = 0
    evals_nearfield: int = 0
    cells_visited: int = 0
    aca_warnings: int = 0
    aca_unconverged: int = 0


class _H2Handle:
    def __init__(self, ptr):
        self.ptr = ptr

    def __del__(self):
        if self.ptr:
            _lib.lib().h2b_h2_free(self.ptr)
            self.ptr = None


H2_FIELDS = {"k_in": 0, "k_out": 1, "t_in": 2, "s_in": 3, "t_out": 4, "s_out": 5, "nevals": 6, "converged": 7,
             "m_in": 8, "n_out": 9}


class _PivotView(Mapping):
    """Cell -> PivotSet, read lazily from the device representation."""

    def __init__(self, h2):
        self._h2 = h2
        self._cache = {}

    def _level(self, level):
        if level not in self._cache:
            h2 = self._h2
            kin = h2.array(level, "k_in")
            kout = h2.array(level, "k_out")
            pin = np.concatenate([[0], np.cumsum(kin)])
            pout = np.concatenate([[0], np.cumsum(kout)])
            self._cache[level] = (pin, pout, h2.array(level, "t_in"), h2.array(level, "s_in"),
                                  h2.array(level, "t_out"), h2.array(level, "s_out"))
        return self._cache[level]

    def __getitem__(self, cell):
        if not isinstance(cell, Cell) or cell._ref_index < 0 or cell.level < TOP_COMPRESSED_LEVEL \
                or cell.level > self._h2.tree.depth:
            raise KeyError(cell)
        pin, pout, ti, si, to, so = self._level(cell.level)
        i = cell._ref_index
        return PivotSet(t_in=ti[pin[i]:pin[i + 1]], s_in=si[pin[i]:pin[i + 1]], t_out=to[pout[i]:pout[i + 1]],
                        s_out=so[pout[i]:pout[i + 1]])

    def __iter__(self):
        tree = self._h2.tree
        for level in range(TOP_COMPRESSED_LEVEL, tree.depth + 1):
            yield from tree.nonempty_cells(level)

    def __len__(self):
        tree = self._h2.tree
        return sum(tree.ncells(level) for level in range(TOP_COMPRESSED_LEVEL, tree.depth + 1))


class _TransferView(Mapping):
    """Cell -> TransferOps built from the device interpolation operators."""

    def __init__(self, h2):
        self._h2 = h2

    def __getitem__(self, cell):
        h2 = self._h2
        if not isinstance(cell, Cell) or cell._ref_index < 0 or cell.level < TOP_COMPRESSED_LEVEL \
                or cell.level > h2.tree.depth:
            raise KeyError(cell)
        ops = TransferOps()
        P = h2.interp(cell.level, cell._ref_index, 0)
        Q = P if h2.symmetric_path else h2.interp(cell.level, cell._ref_index, 1)
        if cell.is_leaf:
            ops.l2p = P
            ops.p2m = Q
            return ops
        a = b = 0
        for child in cell.children:
            if child.is_empty:
                continue
            ps = h2.pivots[child]
            ops.l2l[child] = np.ascontiguousarray(P[a:a + ps.t_in.size])
            ops.m2m[child] = np.ascontiguousarray(Q[b:b + ps.s_out.size].T)
            a += ps.t_in.size
            b += ps.s_out.size
        return ops

    def __iter__(self):
        return iter(self._h2.pivots)

    def __len__(self):
        return len(self._h2.pivots)


class _BlockView(Mapping):
    """(X, Y) -> dense kernel block, evaluated on the GPU when indexed."""

    def __init__(self, h2, near: bool):
        self._h2 = h2
        self._near = near

    def _pair_ok(self, x, y):
        h2 = self._h2
        if self._near:
            return x.is_leaf and x.t_idx.size and y.s_idx.size and y in x.neighbors
        if x.level < TOP_COMPRESSED_LEVEL or y not in x.interaction_list:
            return False
        px, py = h2.pivots.get(x), h2.pivots.get(y)
        return px is not None and py is not None and px.t_in.size > 0 and py.s_out.size > 0

    def __getitem__(self, key):
        x, y = key
        if not self._pair_ok(x, y):
            raise KeyError(key)
        h2 = self._h2
        cloud = h2.tree.cloud
        if self._near:
            return raw_block(h2.kernel, cloud.points_p[x.t_idx], cloud.points_q[y.s_idx])
        return raw_block(h2.kernel, cloud.points_p[h2.pivots[x].t_in], cloud.points_q[h2.pivots[y].s_out])

    def __iter__(self):
        tree = self._h2.tree
        if self._near:
            for x in tree.leaves():
                if x.t_idx.size == 0:
                    continue
                for y in x.neighbors:
                    if y.s_idx.size:
                        yield (x, y)
        else:
            for level in range(TOP_COMPRESSED_LEVEL, tree.depth + 1):
                for x in tree.nonempty_cells(level):
                    for y in x.interaction_list:
                        if self._pair_ok(x, y):
                            yield (x, y)

    def __len__(self):
        return sum(1 for _ in self)


class H2Matrix:
    """Assembled H2 representation, resident on the GPU (compress.py:107)."""

    def __init__(self, tree: HierTree, kernel: KernelSpec, handle: _H2Handle):
        self.tree = tree
        self.kernel = kernel
        self._handle = handle
        self._arrays = {}
        st = self.native_stats()
        self._symmetric = bool(st[6])
        self.pivots = _PivotView(self)
        self.transfers = _TransferView(self)
        self.couplings = _BlockView(self, near=False)
        self.nearfield = _BlockView(self, near=True)
        self.stats = H2Stats(n_targets=tree.cloud.n_targets, n_sources=tree.cloud.n_sources)

    @property
    def handle(self):
        return self._handle.ptr

    def native_stats(self) -> np.ndarray:
        st = np.zeros(10, dtype=np.int64)
        _lib.check(_lib.lib().h2b_h2_stats(self.handle, _lib.iptr(st)))
        return st

    def array(self, level: int, name: str) -> np.ndarray:
        key = (level, name)
        if key not in self._arrays:
            L = _lib.lib()
            w = H2_FIELDS[name]
            n = _lib.check(L.h2b_h2_get_i64(self.handle, level, w, None))
            out = np.empty(n, dtype=np.int64)
            if n:
                _lib.check(L.h2b_h2_get_i64(self.handle, level, w, _lib.iptr(out)))
            self._arrays[key] = out
        return self._arrays[key]

    def interp(self, level: int, cell_index: int, which: int = 0) -> np.ndarray:
        L = _lib.lib()
        cols = ctypes.c_int64()
        rows = _lib.check(L.h2b_h2_get_interp(self.handle, level, int(cell_index), which, ctypes.byref(cols), None))
        out = np.empty((rows, cols.value))
        if out.size:
            _lib.check(L.h2b_h2_get_interp(self.handle, level, int(cell_index), which, ctypes.byref(cols),
                                           _lib.dptr(out)))
        return out

    @property
    def shape(self):
        return (self.tree.cloud.n_targets, self.tree.cloud.n_sources)

    @property
    def symmetric_path(self) -> bool:
        return self._symmetric

    def compressed_levels(self):
        return range(TOP_COMPRESSED_LEVEL, self.tree.depth + 1)

    def pivot_set(self, cell) -> PivotSet:
        return self.pivots.get(cell) or PivotSet()

    def matvec(self, w):
        from .matvec import h2_matvec

        return h2_matvec(self, w)

    def __matmul__(self, w):
        return self.matvec(w)

    def memory_bytes(self) -> int:
        """Device bytes held by the representation (pivots, coordinates, transfer operators, matvec scratch).

        Not comparable with the reference's figure: the engine stores no coupling and no near-field blocks (it
        regenerates their entries in registers); ``reference_memory_bytes`` is the reference's count.
        """
        return int(self.native_stats()[5])

    def reference_memory_bytes(self) -> int:
        """Bytes the reference's representation of this matrix holds (compress.py:142 memory_bytes, before its
        apply plan is built): stored coupling and near-field blocks, dense transfer operators, pivot index arrays."""
        st = self.native_stats()
        total = 8 * (int(st[1]) + int(st[2]))
        for level in self.compressed_levels():
            k_in, k_out = self.array(level, "k_in"), self.array(level, "k_out")
            m_in, n_out = self.array(level, "m_in"), self.array(level, "n_out")
            total += 8 * int((m_in * k_in).sum() + (n_out * k_out).sum())
            total += 8 * int(2 * k_in.sum() + 2 * k_out.sum())
        return total


def candidate_sets(cell: Cell, pivots: dict) -> Candidates:
    """Build the four pivot search spaces for one cell (compress.py:159).

    Host view helper (the engine builds the same sets on the device).
    """
    il = [c for c in cell.interaction_list if not c.is_empty]
    if cell.is_leaf:
        s_in = [c.s_idx for c in il]
        t_out = [c.t_idx for c in il]
        return Candidates(t_in=cell.t_idx, s_in=np.concatenate(s_in) if s_in else _EMPTY,
                          t_out=np.concatenate(t_out) if t_out else _EMPTY, s_out=cell.s_idx)
    t_in_parts, in_slices, s_out_parts, out_slices = [], [], [], []
    pos_in = pos_out = 0
    for child in cell.children:
        ps = pivots.get(child)
        if ps is None:
            continue
        t_in_parts.append(ps.t_in)
        in_slices.append((child, pos_in, pos_in + ps.t_in.size))
        pos_in += ps.t_in.size
        s_out_parts.append(ps.s_out)
        out_slices.append((child, pos_out, pos_out + ps.s_out.size))
        pos_out += ps.s_out.size
    s_in_parts, t_out_parts = [], []
    for member in il:
        for child in member.children:
            ps = pivots.get(child)
            if ps is None:
                continue
            s_in_parts.append(ps.s_out)
            t_out_parts.append(ps.t_in)

    def cat(parts):
        return np.concatenate(parts) if parts else _EMPTY

    return Candidates(t_in=cat(t_in_parts), s_in=cat(s_in_parts), t_out=cat(t_out_parts), s_out=cat(s_out_parts),
                      in_slices=in_slices, out_slices=out_slices)


def _native_assemble(tree: HierTree, kernel: KernelSpec, epsilon_nca: float, force_general: bool,
                     max_rank: int | None) -> H2Matrix:
    if not epsilon_nca > 0:
        raise ValueError("epsilon must be positive")
    kernel.require_device()
    h = ctypes.c_void_p()
    _lib.check(_lib.lib().h2b_assemble(tree.handle, kernel.kind, kernel.device_param, float(epsilon_nca),
                                       int(bool(force_general) or not kernel.is_symmetric),
                                       -1 if max_rank is None else int(max_rank), None, ctypes.byref(h)))
    return H2Matrix(tree, kernel, _H2Handle(h.value))


def _fill_stats(h2: H2Matrix, seconds: float) -> H2Stats:
    st = h2.native_stats()
    s = h2.stats
    s.evals_pivots = int(st[0])
    s.evals_couplings = int(st[1])
    s.evals_nearfield = int(st[2])
    s.max_rank = int(st[3])
    s.cells_visited = int(st[4])
    s.memory_bytes = int(st[5])
    s.evals_transfers = 0
    s.entry_evaluations = s.evals_pivots + s.evals_couplings + s.evals_nearfield
    s.assembly_seconds = seconds
    s.aca_unconverged = int(st[9])
    return s


def select_pivots(tree: HierTree, kernel: KernelSpec, epsilon_nca: float, force_general: bool = False,
                  max_rank: int | None = None):
    """Single bottom-up pass choosing pivots and transfer operators (compress.py:216).

    Returns (pivots, transfers, stats) as lazy views over the device result.
    """
    t0 = time.perf_counter()
    h2 = _native_assemble(tree, kernel, epsilon_nca, force_general, max_rank)
    stats = _fill_stats(h2, time.perf_counter() - t0)
    EVALS.add(stats.evals_pivots)
    return h2.pivots, h2.transfers, stats


def assemble(tree: HierTree, kernel: KernelSpec, epsilon_nca: float, force_general: bool = False,
             max_rank: int | None = None) -> H2Matrix:
    """Build the H2 representation on the GPU (compress.py:285)."""
    t0 = time.perf_counter()
    h2 = _native_assemble(tree, kernel, epsilon_nca, force_general, max_rank)
    stats = _fill_stats(h2, time.perf_counter() - t0)
    EVALS.add(stats.entry_evaluations)
    return h2
