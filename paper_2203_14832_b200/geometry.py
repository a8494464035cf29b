"""Uniform 2^d spatial tree with neighbor and interaction lists (GPU-built).

Same public surface as h2cross/geometry.py (PointCloud, Cell, HierTree,
admissible, build_tree, compute_lists).  ``build_tree`` runs entirely on the
GPU (libh2b200.so h2b_tree_build, replacing geometry.py:230): Morton codes
from the reference's exact bin recurrence, one radix sort, per-level cells,
and CSR neighbour / interaction lists.  The returned ``HierTree`` keeps the
device tree and materialises the reference's Python view (``levels`` dicts of
``Cell`` objects, including empty cells) lazily, only when it is touched.
"""

from __future__ import annotations

import ctypes
import io
import itertools
import math
from dataclasses import dataclass

import numpy as np

from . import _lib

FULL_GRID_CELL_CAP = 1 << 21  # geometry.py:33
WIDTH_UNDERFLOW = 2.0**-50  # geometry.py:36


@dataclass
class PointCloud:
    """Target points P (indexed by I) and source points Q (indexed by J)."""

    points_p: np.ndarray
    points_q: np.ndarray
    shared: bool = False

    def __post_init__(self):
        self.points_p = np.ascontiguousarray(np.atleast_2d(self.points_p), dtype=np.float64)
        self.points_q = np.ascontiguousarray(np.atleast_2d(self.points_q), dtype=np.float64)
        if self.points_p.ndim != 2 or self.points_q.ndim != 2:
            raise ValueError("points must be 2-d arrays of shape (n, d)")
        if self.points_p.shape[1] != self.points_q.shape[1]:
            raise ValueError("target and source points must share a dimension")
        if self.points_p.shape[1] == 0:
            raise ValueError("points must have at least one coordinate")

    @classmethod
    def from_points(cls, points, sources=None) -> "PointCloud":
        pts = np.atleast_2d(np.asarray(points, dtype=np.float64))
        if sources is None:
            return cls(pts, pts, shared=True)
        return cls(pts, np.atleast_2d(np.asarray(sources, dtype=np.float64)), shared=False)

    @classmethod
    def from_csv(cls, path, dim: int, sources_path=None) -> "PointCloud":
        pts = load_points_csv(path, dim)
        if sources_path is None:
            return cls(pts, pts, shared=True)
        return cls(pts, load_points_csv(sources_path, dim), shared=False)

    @property
    def dim(self) -> int:
        return self.points_p.shape[1]

    @property
    def n_targets(self) -> int:
        return self.points_p.shape[0]

    @property
    def n_sources(self) -> int:
        return self.points_q.shape[0]


def load_points_csv(path, dim: int) -> np.ndarray:
    data = np.loadtxt(path, delimiter=",", ndmin=2, dtype=np.float64)
    if data.shape[1] < dim:
        raise ValueError(f"{path}: expected at least {dim} columns, found {data.shape[1]}")
    return np.ascontiguousarray(data[:, :dim])


_EMPTY_IDX = np.empty(0, dtype=np.int64)


class Cell:
    """One box of the tree (geometry.py:96)."""

    __slots__ = ("level", "multi_index", "center", "half_width", "parent", "children", "t_idx", "s_idx",
                 "neighbors", "interaction_list", "is_leaf", "over_capacity", "_ref_index")

    def __init__(self, level, multi_index, center, half_width, parent=None):
        self.level = level
        self.multi_index = multi_index
        self.center = center
        self.half_width = half_width
        self.parent = parent
        self.children = []
        self.t_idx = _EMPTY_IDX
        self.s_idx = _EMPTY_IDX
        self.neighbors = []
        self.interaction_list = []
        self.is_leaf = False
        self.over_capacity = False
        self._ref_index = -1  # position among the level's nonempty cells (engine export order)

    @property
    def n_targets(self):
        return self.t_idx.size

    @property
    def n_sources(self):
        return self.s_idx.size

    @property
    def is_empty(self):
        return self.t_idx.size == 0 and self.s_idx.size == 0

    def key(self):
        return (self.level, self.multi_index)

    def __repr__(self):
        return f"Cell(level={self.level}, mi={self.multi_index}, nt={self.n_targets}, ns={self.n_sources})"


def boxes_admissible(center_x, hw_x, center_y, hw_y, eta: float) -> bool:
    """Closed-form admissibility for two axis-aligned hypercubes (geometry.py:147)."""
    d = len(center_x)
    diam = 2.0 * max(hw_x, hw_y) * math.sqrt(d)
    gap = np.maximum(np.abs(np.asarray(center_x) - np.asarray(center_y)) - (hw_x + hw_y), 0.0)
    dist = math.sqrt(float(np.dot(gap, gap)))
    return diam <= eta * dist


def admissible(x: Cell, y: Cell, eta: float) -> bool:
    """True iff max(diam(X), diam(Y)) <= eta * dist(X, Y)."""
    return boxes_admissible(x.center, x.half_width, y.center, y.half_width, eta)


class _TreeHandle:
    """Owns the native tree (freed when the last Python reference goes)."""

    def __init__(self, ptr):
        self.ptr = ptr

    def __del__(self):
        if self.ptr:
            _lib.lib().h2b_tree_free(self.ptr)
            self.ptr = None


TREE_FIELDS = {"key": 0, "mi": 1, "t_ptr": 2, "t_idx": 3, "s_ptr": 4, "s_idx": 5, "nb_ptr": 6, "nb_idx": 7,
               "il_ptr": 8, "il_idx": 9, "parent": 10, "ch_ptr": 11, "ch_idx": 12}


class HierTree:
    """Finished tree: device-resident, with a lazily built reference view."""

    def __init__(self, cloud: PointCloud, handle: _TreeHandle, eta: float, nu: int):
        self.cloud = cloud
        self.eta = float(eta)
        self.nu = int(nu)
        self._handle = handle
        depth = ctypes.c_int()
        over = ctypes.c_int()
        mid = np.zeros(cloud.dim)
        half = ctypes.c_double()
        _lib.check(_lib.lib().h2b_tree_info(handle.ptr, ctypes.byref(depth), ctypes.byref(over), _lib.dptr(mid),
                                            ctypes.byref(half)))
        self._depth = depth.value
        self._over = bool(over.value)
        self.mid = mid
        self.half = half.value
        self._levels = None
        self._arrays = {}

    # ---- native access -------------------------------------------------
    @property
    def handle(self):
        return self._handle.ptr

    def ncells(self, level: int) -> int:
        """Number of nonempty cells at a level."""
        return int(_lib.lib().h2b_tree_ncells(self.handle, level))

    def array(self, level: int, name: str) -> np.ndarray:
        """Per-level engine export in reference cell order (nonempty cells by multi-index)."""
        key = (level, name)
        if key not in self._arrays:
            L = _lib.lib()
            w = TREE_FIELDS[name]
            n = _lib.check(L.h2b_tree_get(self.handle, level, w, None))
            out = np.empty(n, dtype=np.int64)
            if n:
                _lib.check(L.h2b_tree_get(self.handle, level, w, _lib.iptr(out)))
            self._arrays[key] = out
        return self._arrays[key]

    # ---- reference surface -----------------------------------------------
    @property
    def depth(self) -> int:
        return self._depth

    @property
    def levels(self):
        if self._levels is None:
            self._levels = _materialize(self)
        return self._levels

    @property
    def root(self) -> Cell:
        return self.levels[0][(0,) * self.cloud.dim]

    def cells(self, level: int):
        """Cells of one level in multi-index order."""
        return [self.levels[level][mi] for mi in sorted(self.levels[level])]

    def nonempty_cells(self, level: int):
        return [c for c in self.cells(level) if not c.is_empty]

    def leaves(self):
        return self.cells(self.depth)

    @property
    def over_capacity(self) -> bool:
        return self._over

    def stats_report(self) -> str:
        """Plain-text summary: depth, cells per level, leaf occupancy histogram (geometry.py:189)."""
        out = io.StringIO()
        cloud = self.cloud
        d = cloud.dim
        print(f"points: {cloud.n_targets} targets, {cloud.n_sources} sources, dim {d}", file=out)
        print(f"depth: {self.depth}", file=out)
        print(f"eta: {self.eta:g}  nu: {self.nu}", file=out)
        for k in range(self.depth + 1):
            nonempty = self.ncells(k)
            print(f"level {k}: {_n_materialized(self, k)} cells, {nonempty} nonempty", file=out)
        tp = self.array(self.depth, "t_ptr")
        occ = np.diff(tp)
        sp = self.array(self.depth, "s_ptr")
        occ = occ[(np.diff(tp) > 0) | (np.diff(sp) > 0)]
        if occ.size:
            print(f"leaf occupancy (targets): min {occ.min()}  mean {occ.mean():.1f}  max {occ.max()}", file=out)
            edges = np.linspace(0, occ.max() + 1, num=min(9, occ.max() + 2), dtype=np.int64)
            hist, _ = np.histogram(occ, bins=edges)
            for lo, hi, h in zip(edges[:-1], edges[1:], hist):
                print(f"  [{lo}, {hi}): {h}", file=out)
        if self.over_capacity:
            print("warning: width underflow stopped subdivision; some leaves exceed nu", file=out)
        return out.getvalue()


def _n_materialized(tree: HierTree, level: int) -> int:
    if tree._levels is not None:
        return len(tree._levels[level])
    n_axis = 1 << level
    if n_axis ** tree.cloud.dim <= FULL_GRID_CELL_CAP:
        return n_axis ** tree.cloud.dim
    return len(tree.levels[level])


def _cell_center(tree: HierTree, level: int, mi) -> tuple:
    if level == 0:
        return tree.mid.copy(), tree.half
    width = tree.half * 2.0 ** (1 - level)
    lo0 = tree.mid - tree.half
    return lo0 + (np.array(mi, dtype=np.float64) + 0.5) * width, 0.5 * width


def _materialize(tree: HierTree):
    """Build the reference's per-level dicts of Cell objects from engine exports.

    Nonempty cells, their point sets and parent/child links come from the
    engine.  Empty cells are created where the reference creates them
    (geometry.py:284-300: the full grid while it has at most
    FULL_GRID_CELL_CAP cells, else the children of nonempty cells and of
    their neighbours); their lists are computed here by the reference rule.
    """
    d = tree.cloud.dim
    levels = []
    for level in range(tree.depth + 1):
        mi_arr = tree.array(level, "mi").reshape(-1, d)
        tp, ti = tree.array(level, "t_ptr"), tree.array(level, "t_idx")
        sp, si = tree.array(level, "s_ptr"), tree.array(level, "s_idx")
        cells = {}
        ne = []
        for i in range(mi_arr.shape[0]):
            mi = tuple(int(v) for v in mi_arr[i])
            c, hw = _cell_center(tree, level, mi)
            cell = Cell(level, mi, c, hw)
            cell.t_idx = ti[tp[i]:tp[i + 1]]
            cell.s_idx = si[sp[i]:sp[i + 1]]
            cell._ref_index = i
            cells[mi] = cell
            ne.append(cell)
        if level > 0:
            n_axis = 1 << level
            if n_axis**d <= FULL_GRID_CELL_CAP:
                parents = levels[level - 1].values()
            else:
                keep = set()
                for c in levels[level - 1].values():
                    if not c.is_empty:
                        keep.add(c)
                        keep.update(c.neighbors)
                parents = keep
            for par in parents:
                base = tuple(2 * m for m in par.multi_index)
                for off in itertools.product((0, 1), repeat=d):
                    mi = tuple(b + o for b, o in zip(base, off))
                    cell = cells.get(mi)
                    if cell is None:
                        c, hw = _cell_center(tree, level, mi)
                        cell = Cell(level, mi, c, hw)
                        cells[mi] = cell
                    cell.parent = par
                    par.children.append(cell)
        levels.append(cells)
        if level == 0:
            root = cells[(0,) * d]
            root.neighbors = [root]
            root.interaction_list = []
        else:
            _annotate(levels, level, tree.eta)
    for c in levels[tree.depth].values():
        c.is_leaf = True
        if tree.over_capacity and max(c.n_targets, c.n_sources) > tree.nu:
            c.over_capacity = True
    return levels


def _annotate(levels, level, eta):
    """geometry.py:322 _annotate_level on the materialised view."""
    for cell in levels[level].values():
        parent = cell.parent
        candidates = [ch for nb in parent.neighbors for ch in nb.children]
        nbrs, il = [], []
        for cand in candidates:
            if admissible(cell, cand, eta):
                il.append(cand)
            else:
                nbrs.append(cand)
        nbrs.sort(key=Cell.key)
        il.sort(key=Cell.key)
        cell.neighbors = nbrs
        cell.interaction_list = il


def build_tree(cloud: PointCloud, nu: int, eta: float) -> HierTree:
    """Build the uniform 2^d tree and its lists on the GPU (geometry.py:230).

    Raises ValueError for an empty cloud, ``nu`` < 1, or ``eta`` <= 0.
    """
    if cloud.n_targets == 0 or cloud.n_sources == 0:
        raise ValueError("empty point set")
    if nu < 1:
        raise ValueError("invalid leaf capacity")
    if not eta > 0:
        raise ValueError("eta must be positive")
    if cloud.dim > 4:
        raise ValueError("the B200 engine supports dimensions 1..4")
    L = _lib.lib()
    h = ctypes.c_void_p()
    P = cloud.points_p
    Q = cloud.points_q
    _lib.check(L.h2b_tree_build(P.ctypes.data, P.shape[0], Q.ctypes.data, Q.shape[0], cloud.dim,
                                int(bool(cloud.shared)), int(nu), float(eta), 0, None, ctypes.byref(h)))
    return HierTree(cloud, _TreeHandle(h.value), eta, nu)


def compute_lists(tree: HierTree) -> HierTree:
    """(Re)compute neighbor and interaction lists at every level >= 1 (geometry.py:339).

    The engine computes the lists during ``build_tree``; on the Python view
    this re-derives them from the cell geometry, as the reference does.
    """
    levels = tree.levels
    levels[0][(0,) * tree.cloud.dim].neighbors = [levels[0][(0,) * tree.cloud.dim]]
    for level in range(1, tree.depth + 1):
        _annotate(levels, level, tree.eta)
    return tree
