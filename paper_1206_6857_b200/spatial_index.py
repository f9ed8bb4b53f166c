"""Device-resident kd-trees (mirror of spatial_index.py).

``build_tree`` runs the level-synchronous device build (fg_tree.cu), which
reproduces the reference's split rule and therefore its permutation and node
ranges (spatial_index.py:231-276).  The tree stays on the GPU; the
reference's host object model (``root``/``nodes``/``leaves``, per-node
fields, ``points``/``weights``/``perm``) is materialised lazily from the
device arrays the first time it is touched.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .kernel_math import index_set
from .series_expansion import FarFieldExpansion, LocalExpansion

_PLIMIT_SCHEDULE = {1: 8, 2: 8, 3: 6, 4: 4, 5: 4, 6: 2}


def default_plimit(dim: int) -> int:
    """Series-order cap per dimension (spatial_index.py:39-44)."""
    return _PLIMIT_SCHEDULE.get(dim, 1)


def engine_plimit(dim: int) -> int:
    """The engine's own series-order cap (``fg_engine_plimit``): what sweeps use
    when ``RunConfig.plimit`` is None.  10 at D = 3, ``default_plimit`` elsewhere."""
    return int(_lib.lib().fg_engine_plimit(int(dim)))


@dataclass
class PointStore:
    """(N, D) points with positive weights (spatial_index.py:47-80)."""

    points: np.ndarray
    weights: np.ndarray = field(default=None)

    def __post_init__(self):
        self.points = np.ascontiguousarray(self.points, dtype=float)
        if self.points.ndim != 2 or self.points.shape[0] == 0:
            raise ValueError("points must be a non-empty (N, D) array")
        if self.weights is None:
            self.weights = np.ones(self.points.shape[0])
        else:
            self.weights = np.ascontiguousarray(self.weights, dtype=float).reshape(-1)
            if self.weights.shape[0] != self.points.shape[0]:
                raise ValueError("weights length must match point count")
            if np.any(self.weights <= 0.0):
                raise ValueError("weights must be positive")

    @property
    def n(self) -> int:
        return self.points.shape[0]

    @property
    def dim(self) -> int:
        return self.points.shape[1]

    @property
    def total_weight(self) -> float:
        return float(self.weights.sum())


class Node:
    """Host view of one device node (spatial_index.py:83-141)."""

    __slots__ = ("index", "start", "end", "lo", "hi", "lo_t", "hi_t", "center", "count",
                 "weight", "inf_radius", "left", "right", "_tree", "tokens", "mass_lo",
                 "mass_hi", "pend_lo", "pend_hi", "est", "local", "local_used")

    def __init__(self, tree, index, start, end, lo, hi, center, weight, inf_radius):
        self._tree = tree
        self.index = index
        self.start = start
        self.end = end
        self.lo = lo
        self.hi = hi
        self.lo_t = tuple(lo.tolist())
        self.hi_t = tuple(hi.tolist())
        self.center = center
        self.count = end - start
        self.weight = weight
        self.inf_radius = inf_radius
        self.left = None
        self.right = None
        self.tokens = 0.0
        self.mass_lo = 0.0
        self.mass_hi = 0.0
        self.pend_lo = 0.0
        self.pend_hi = 0.0
        self.est = 0.0
        self.local = None
        self.local_used = False

    @property
    def is_leaf(self) -> bool:
        return self.left is None

    @property
    def moments(self):
        """Cached far-field expansion of this node (refresh_moments)."""
        return self._tree._node_moments(self.index)


class KdTree:
    """A kd-tree resident on the GPU (spatial_index.py:144-228)."""

    def __init__(self, handle, store: PointStore, leaf_threshold: int):
        self._h = handle
        self._store = store
        self.leaf_threshold = leaf_threshold
        n = ctypes.c_int64()
        dim = ctypes.c_int32()
        nn = ctypes.c_int64()
        tw = ctypes.c_double()
        lv = ctypes.c_int32()
        _lib.call("fg_tree_info", self._h, ctypes.byref(n), ctypes.byref(dim), ctypes.byref(nn),
                  ctypes.byref(tw), ctypes.byref(lv))
        self._n, self._dim, self.node_count = n.value, dim.value, nn.value
        self.total_weight = tw.value
        self.levels = lv.value
        self.moments_bandwidth = None
        self.moments_order = None
        self._export = None
        self._nodes = None
        self._points = None
        self._weights = None
        self._moments = None
        self.q_mass_lo = None
        self.q_mass_hi = None
        self._q_est = None
        self._run_values = None

    @property
    def q_est(self):
        """Per-point estimates in tree order (the reference's q_est), built lazily
        from the last run's values."""
        if self._q_est is None and self._run_values is not None:
            self._q_est = np.asarray(self._run_values)[self.perm]
        return self._q_est

    @q_est.setter
    def q_est(self, value):
        self._q_est = value
        self._run_values = None

    def _set_run_values(self, values):
        self._run_values = values
        self._q_est = None

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            try:
                _lib.lib().fg_tree_free(h)
            except Exception:
                pass
            self._h = None

    @property
    def handle(self):
        return self._h

    @property
    def n(self) -> int:
        return self._n

    @property
    def dim(self) -> int:
        return self._dim

    # ------------------------------------------------------ exported views
    def _exported(self):
        if self._export is None:
            nn, D = self.node_count, self._dim
            e = dict(perm=np.empty(self._n, np.int64), start=np.empty(nn, np.int64),
                     end=np.empty(nn, np.int64), lo=np.empty((nn, D)), hi=np.empty((nn, D)),
                     center=np.empty((nn, D)), weight=np.empty(nn),
                     inf_radius=np.empty(nn), left=np.empty(nn, np.int64),
                     right=np.empty(nn, np.int64))
            _lib.call("fg_tree_export", self._h,
                      *[_lib.ptr(e[k]) for k in ("perm", "start", "end", "lo", "hi", "center",
                                                  "weight", "inf_radius", "left", "right")])
            self._export = e
        return self._export

    def arrays(self) -> dict:
        """Preorder node arrays (perm, start, end, lo, hi, center, weight,
        inf_radius, left, right) -- the reference's Node fields as arrays."""
        return self._exported()

    @property
    def perm(self) -> np.ndarray:
        return self._exported()["perm"]

    @property
    def points(self) -> np.ndarray:
        if self._points is None:
            self._points = np.empty((self._n, self._dim))
            self._weights = np.empty(self._n)
            _lib.call("fg_tree_points", self._h, _lib.ptr(self._points), _lib.ptr(self._weights))
        return self._points

    @property
    def weights(self) -> np.ndarray:
        if self._weights is None:
            _ = self.points
        return self._weights

    @property
    def nodes(self) -> list:
        if self._nodes is None:
            e = self._exported()
            nodes = [Node(self, i, int(e["start"][i]), int(e["end"][i]), e["lo"][i], e["hi"][i],
                          e["center"][i], float(e["weight"][i]), float(e["inf_radius"][i]))
                     for i in range(self.node_count)]
            for i, nd in enumerate(nodes):
                if e["left"][i] >= 0:
                    nd.left = nodes[e["left"][i]]
                    nd.right = nodes[e["right"][i]]
            self._nodes = nodes
        return self._nodes

    @property
    def root(self) -> Node:
        return self.nodes[0]

    @property
    def leaves(self) -> list:
        return [nd for nd in self.nodes if nd.left is None]

    # ------------------------------------------------------------ moments
    def refresh_moments(self, h: float, plimit: int) -> None:
        """Rebuild every node's far-field moments for bandwidth h (device)."""
        _lib.call("fg_moments_refresh", self._h, float(h), int(plimit))
        self._moments_refreshed(h, plimit)

    def _moments_refreshed(self, h: float, plimit: int) -> None:
        self.moments_bandwidth = h
        self.moments_order = plimit
        self._moments = None

    def _node_moments(self, index: int):
        if self.moments_bandwidth is None:
            return None
        if self._moments is None:
            K = index_set(self._dim, self.moments_order).count
            out = np.empty((self.node_count, K))
            _lib.call("fg_moments_export", self._h, _lib.ptr(out), None, None, None)
            self._moments = out
        e = self._exported()
        return FarFieldExpansion(e["center"][index], self.moments_order,
                                 self._moments[index], self.moments_bandwidth)

    def moments_array(self) -> np.ndarray:
        """(nodes, K) moments in preorder numbering."""
        self._node_moments(0)
        return self._moments

    # -------------------------------------------------------- query state
    def reset_query_state(self, total_ref_weight: float, local_order: int | None = None,
                          bandwidth: float | None = None) -> None:
        """Zero the host mirror of the query-side state (spatial_index.py:199-228).

        The engine keeps its traversal state on the device for the duration
        of a run; this resets the reference-visible mirror fields.
        """
        w = float(total_ref_weight)
        coeff_count = index_set(self._dim, local_order).count if local_order else 0
        for node in self.nodes:
            node.tokens = 0.0
            node.mass_lo = 0.0
            node.mass_hi = w
            node.pend_lo = 0.0
            node.pend_hi = 0.0
            node.est = 0.0
            node.local_used = False
            node.local = None if local_order is None else LocalExpansion(
                node.center, local_order, np.zeros(coeff_count), bandwidth)
        self.q_mass_lo = np.zeros(self._n)
        self.q_mass_hi = np.full(self._n, w)
        self.q_est = np.zeros(self._n)


def build_tree(store: PointStore, leaf_threshold: int = 25) -> KdTree:
    """Device kd-tree build (spatial_index.py:231-276)."""
    if leaf_threshold < 1:
        raise ValueError("leaf threshold must be at least 1")
    pts = store.points
    w = store.weights
    h = ctypes.c_void_p()
    _lib.call("fg_tree_build", _lib.ptr(pts), _lib.ptr(w), pts.shape[0], pts.shape[1],
              int(leaf_threshold), ctypes.byref(h))
    return KdTree(h.value, store, leaf_threshold)


def build_tree_device(points, weights=None, leaf_threshold: int = 25) -> KdTree:
    """build_tree for inputs already resident on the GPU (CUDA tensors, float64).

    Validation (non-empty, positive weights, finite coordinates) runs on the
    device; the host mirror (``points``/``nodes``...) is still available lazily.
    """
    if leaf_threshold < 1:
        raise ValueError("leaf threshold must be at least 1")
    pts = _lib.as_f64(points)
    if pts.ndim != 2 or pts.shape[0] == 0:
        raise ValueError("points must be a non-empty (N, D) array")
    w = None if weights is None else _lib.as_f64(weights).reshape(-1)
    h = ctypes.c_void_p()
    with _lib.torch_stream(pts, w):
        _lib.call("fg_tree_build", _lib.ptr(pts), _lib.ptr(w), pts.shape[0], pts.shape[1],
                  int(leaf_threshold), ctypes.byref(h))
    return KdTree(h.value, None, leaf_threshold)


def min_sq_dist(a_lo, a_hi, b_lo, b_hi) -> float:
    gap = np.maximum(np.asarray(a_lo) - b_hi, np.asarray(b_lo) - a_hi)
    gap = np.maximum(gap, 0.0)
    return float(gap @ gap)


def max_sq_dist(a_lo, a_hi, b_lo, b_hi) -> float:
    span = np.maximum(np.asarray(a_hi) - b_lo, np.asarray(b_hi) - a_lo)
    return float(span @ span)


def box_sq_bounds(a_lo, a_hi, b_lo, b_hi) -> tuple[float, float]:
    return min_sq_dist(a_lo, a_hi, b_lo, b_hi), max_sq_dist(a_lo, a_hi, b_lo, b_hi)
