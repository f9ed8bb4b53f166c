"""Gaussian summation on the B200 (mirror of summation_engine.py).

``naive_sum`` runs the exhaustive FP64 kernel (fg_naive.cu);
``dfd_run``/``dfdo_run``/``dito_run`` run the fused traversal kernel
(fg_traverse.cu) with the reference's three mode flags
(summation_engine.py:458-480).  Results come back in original query order
as float64 NumPy arrays (or in a caller-provided CUDA tensor via ``out=``).
Every run guarantees max_q |G_est - G| / G <= epsilon.
"""

from __future__ import annotations

import ctypes
import time
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .spatial_index import KdTree, default_plimit, engine_plimit

_ALGORITHMS = ("naive", "dfd", "dfdo", "dito")


@dataclass
class RunConfig:
    """summation_engine.py:57-78."""

    bandwidth: float
    epsilon: float = 0.01
    algorithm: str = "dito"
    plimit: int | None = None
    leaf_threshold: int = 25

    def __post_init__(self):
        if self.bandwidth <= 0.0:
            raise ValueError("bandwidth must be positive")
        if self.epsilon < 0.0:
            raise ValueError("epsilon must be non-negative")
        if self.algorithm not in _ALGORITHMS:
            raise ValueError(f"unknown algorithm {self.algorithm!r}")


@dataclass
class TraversalCounters:
    """summation_engine.py:81-104, plus the pairs evaluated exactly in FP64 and
    the pairs evaluated in FP32 with a charged error bound."""

    pair_visits: int = 0
    base_cases: int = 0
    fd_prunes: int = 0
    hermite_prunes: int = 0
    local_prunes: int = 0
    h2l_prunes: int = 0
    exact_pairs: int = 0
    fp32_pairs: int = 0
    hermite_evals: int = 0
    hermite_terms: int = 0
    local_evals: int = 0

    @property
    def prunes(self) -> int:
        return self.fd_prunes + self.hermite_prunes + self.local_prunes + self.h2l_prunes

    def as_dict(self) -> dict:
        return {
            "pair_visits": self.pair_visits,
            "base_cases": self.base_cases,
            "fd_prunes": self.fd_prunes,
            "hermite_prunes": self.hermite_prunes,
            "local_prunes": self.local_prunes,
            "h2l_prunes": self.h2l_prunes,
        }

    @classmethod
    def _from_c(cls, c: _lib.fg_counters) -> "TraversalCounters":
        return cls(c.pair_visits, c.base_cases, c.fd_prunes, c.hermite_prunes, c.local_prunes,
                   c.h2l_prunes, c.exact_pairs, c.fp32_pairs, c.hermite_evals,
                   c.hermite_terms, c.local_evals)


@dataclass
class ResultVector:
    """summation_engine.py:107-119."""

    values: np.ndarray
    seconds: float
    counters: TraversalCounters = field(default_factory=TraversalCounters)
    audit: list | None = None


def naive_sum(queries, references, weights, h, out=None) -> ResultVector:
    """Exact FP64 sums G(x_q) = sum_r w_r exp(-|x_q - x_r|^2 / 2h^2) on the GPU.

    summation_engine.py:122-154.  ``h`` may be a scalar or a sequence of
    bandwidths (then ``values`` has shape (len(h), M)).  Inputs may be NumPy
    arrays or CUDA tensors; ``out`` may be a CUDA tensor to keep the result
    on the device.
    """
    t0 = time.perf_counter()
    q = _lib.as_f64(queries)
    if q.ndim == 1:
        q = q.reshape(1, -1)
    r = _lib.as_f64(references)
    if r.ndim == 1:
        r = r.reshape(-1, q.shape[1])
    w = _lib.as_f64(weights).reshape(-1)
    m, dim = q.shape
    n = r.shape[0]
    if r.shape[1] != dim or w.shape[0] != n:
        raise ValueError("shape mismatch between queries, references and weights")
    hs = np.atleast_1d(np.asarray(h, dtype=float))
    if np.any(hs <= 0.0):
        raise ValueError("bandwidth must be positive")
    shapes = [(hs.shape[0], m)] + ([(m,)] if hs.shape[0] == 1 else [])
    vals = _lib.check_out(out, shapes) if out is not None else np.empty((hs.shape[0], m))
    with _lib.torch_stream(q, r, w, vals):
        _lib.call("fg_naive_sum", _lib.ptr(q), m, _lib.ptr(r), _lib.ptr(w), n, dim,
                  _lib.ptr(hs), hs.shape[0], _lib.ptr(vals))
    if out is None and np.ndim(h) == 0:
        vals = vals[0]
    counters = TraversalCounters(exact_pairs=int(m) * int(n) * int(hs.shape[0]))
    return ResultVector(vals, time.perf_counter() - t0, counters)


# fg_audit_event (include/fastgauss_b200.h)
AUDIT_DTYPE = np.dtype([("kind", np.int32), ("qblock", np.int32), ("seq", np.int32),
                        ("lane", np.int32), ("w_ref", np.float64), ("bound", np.float64),
                        ("mass_lo", np.float64), ("token_flow", np.float64)])
AUDIT_KINDS = ("base", "fd", "hermite", "local", "h2l")


def query_block_ranges(qtree: KdTree) -> tuple:
    """(starts, counts) of the query blocks in tree order."""
    nb = query_block_count(qtree)
    starts = np.empty(nb, np.int32)
    counts = np.empty(nb, np.int32)
    _lib.call("fg_query_block_ranges", qtree.handle, _lib.ptr(starts), _lib.ptr(counts))
    return starts, counts


def query_block_nodes(qtree: KdTree) -> np.ndarray:
    """Preorder node index (Node.index) of every query block: the deepest node
    containing its run of tree-order points."""
    nb = query_block_count(qtree)
    starts = np.empty(nb, np.int32)
    counts = np.empty(nb, np.int32)
    _lib.call("fg_query_block_ranges", qtree.handle, _lib.ptr(starts), _lib.ptr(counts))
    e = qtree.arrays()
    # the deepest node containing each block's range (node ranges nest)
    depth_order = np.argsort(e["end"] - e["start"], kind="stable")
    out = np.full(nb, -1, np.int64)
    for v in depth_order[::-1]:  # largest first; later (smaller) nodes overwrite
        lo = np.searchsorted(starts, e["start"][v], side="left")
        hi = np.searchsorted(starts, e["end"][v], side="left")
        sel = np.arange(lo, hi)
        sel = sel[starts[sel] + counts[sel] <= e["end"][v]]
        out[sel] = v
    return out


def _audit_run(config: RunConfig, qtree: KdTree, rtree: KdTree, mode: str, plimit: int,
               vals) -> tuple:
    """One run with the device ledger (fg_run_audit); returns the ledger in the
    reference's tuple form (kind, query node index, W_R, bound, mass_lo at the
    decision, token flow), ordered by query node, step and item."""
    cnt = _lib.fg_counters()
    secs = ctypes.c_double()
    cap = 1 << 16
    while True:
        ev = np.empty(cap, AUDIT_DTYPE)
        n = ctypes.c_int64()
        _lib.call("fg_run_audit", qtree.handle, rtree.handle, float(config.bandwidth),
                  float(config.epsilon), _lib.MODES[mode], int(plimit), _lib.ptr(vals),
                  ctypes.byref(cnt), ctypes.byref(secs), ev.ctypes.data, cap, ctypes.byref(n))
        if n.value <= cap:
            break
        cap = n.value
    ev = ev[:n.value]
    ev = ev[np.lexsort((ev["lane"], ev["seq"], ev["qblock"]))]
    nodes = query_block_nodes(qtree)
    ledger = AuditLedger(
        (AUDIT_KINDS[k], int(nodes[b]), float(w), float(bd), float(ml), float(fl))
        for k, b, w, bd, ml, fl in zip(ev["kind"], ev["qblock"], ev["w_ref"], ev["bound"],
                                       ev["mass_lo"], ev["token_flow"]))
    ledger.blocks = np.asarray(ev["qblock"], dtype=np.int64)
    return cnt, secs.value, ledger, ev


class AuditLedger(list):
    """The ledger tuples (reference form: kind, query node, W_R, bound,
    mass_lo, token flow) plus ``blocks``: the query block of every event (the
    unit each bound is charged against; several blocks may share a node)."""

    blocks = None


def _run_tree_algorithm(config: RunConfig, qtree: KdTree, rtree: KdTree, mode: str,
                        audit: bool, out=None, block_range=None) -> ResultVector:
    """summation_engine.py:431-455 on the device."""
    if audit and block_range is not None:
        raise ValueError("the audit ledger records full runs")
    plimit = config.plimit if config.plimit is not None else default_plimit(qtree.dim)
    if mode == "dito" and (rtree.moments_bandwidth != config.bandwidth or
                           rtree.moments_order is None or rtree.moments_order < plimit):
        raise RuntimeError("reference moments missing or stale; call refresh_moments "
                           "for this bandwidth first")
    vals = _lib.check_out(out, [(qtree.n,)]) if out is not None else np.empty(qtree.n)
    if audit:
        cnt, secs, ledger, _ = _audit_run(config, qtree, rtree, mode, plimit, vals)
        if out is None:
            qtree._set_run_values(vals)
        return ResultVector(vals, secs, TraversalCounters._from_c(cnt), ledger)
    cnt = _lib.fg_counters()
    secs = ctypes.c_double()
    with _lib.torch_stream(vals):
        if block_range is None:
            _lib.call("fg_run", qtree.handle, rtree.handle, float(config.bandwidth),
                      float(config.epsilon), _lib.MODES[mode], int(plimit), _lib.ptr(vals),
                      ctypes.byref(cnt), ctypes.byref(secs))
        else:
            b0, b1, stride = block_range
            _lib.call("fg_run_range", qtree.handle, rtree.handle, float(config.bandwidth),
                      float(config.epsilon), _lib.MODES[mode], int(plimit), int(b0), int(b1),
                      int(stride), _lib.ptr(vals), ctypes.byref(cnt), ctypes.byref(secs))
    if out is None:
        qtree._set_run_values(vals)
    return ResultVector(vals, secs.value, TraversalCounters._from_c(cnt), None)


def dfd_run(config: RunConfig, qtree: KdTree, rtree: KdTree, audit: bool = False,
            out=None) -> ResultVector:
    """Finite-difference dual-tree summation (no tokens, no series)."""
    return _run_tree_algorithm(config, qtree, rtree, "dfd", audit, out)


def dfdo_run(config: RunConfig, qtree: KdTree, rtree: KdTree, audit: bool = False,
             out=None) -> ResultVector:
    """Finite-difference dual-tree summation with error tokens."""
    return _run_tree_algorithm(config, qtree, rtree, "dfdo", audit, out)


def dito_run(config: RunConfig, qtree: KdTree, rtree: KdTree, audit: bool = False,
             out=None) -> ResultVector:
    """Series-accelerated dual-tree summation with error tokens.

    Requires ``rtree.refresh_moments(bandwidth, plimit)`` for this bandwidth.
    """
    return _run_tree_algorithm(config, qtree, rtree, "dito", audit, out)


def sweep_run(config: RunConfig, qtree: KdTree, rtree: KdTree, bandwidths,
              out=None, block_range=None) -> list:
    """Run ``config.algorithm`` at every bandwidth in one device call.

    The per-bandwidth loop of run_sweep (cli_harness.py:246-283): for DITO each
    bandwidth refreshes ``rtree``'s moments first (they are left at the last
    bandwidth).  ``config.bandwidth`` is ignored.  Returns one ResultVector per
    bandwidth; with ``out`` (a CUDA tensor of shape (len(bandwidths), M)) the
    values stay on the device and each ResultVector holds a row view.
    ``block_range`` = (begin, end, stride) restricts the sweep to those query
    blocks (sharding; the other entries of ``out`` are kept).
    """
    if config.algorithm == "naive":
        raise ValueError("sweep_run runs the tree algorithms; use naive_sum for naive")
    hs = np.ascontiguousarray(np.atleast_1d(np.asarray(bandwidths, dtype=float)))
    if hs.size == 0 or np.any(hs <= 0.0):
        raise ValueError("bandwidths must be positive")
    # the engine's own order cap unless the caller fixes one (any order keeps
    # eps): 0 lets the engine apply engine_plimit(dim), lowered if the moment
    # sets of that order would not fit the device's memory
    plimit = config.plimit if config.plimit is not None else 0
    nh = hs.shape[0]
    shapes = [(nh, qtree.n)] + ([(qtree.n,)] if nh == 1 else [])
    vals = _lib.check_out(out, shapes) if out is not None else (
        np.empty((nh, qtree.n)) if block_range is None else np.zeros((nh, qtree.n)))
    cnt = (_lib.fg_counters * nh)()
    secs = np.zeros(nh)
    with _lib.torch_stream(vals):
        if block_range is None:
            _lib.call("fg_run_sweep", qtree.handle, rtree.handle, _lib.ptr(hs), nh,
                      float(config.epsilon), _lib.MODES[config.algorithm], int(plimit),
                      _lib.ptr(vals), cnt, _lib.ptr(secs))
        else:
            b0, b1, stride = block_range
            _lib.call("fg_run_sweep_range", qtree.handle, rtree.handle, _lib.ptr(hs), nh,
                      float(config.epsilon), _lib.MODES[config.algorithm], int(plimit),
                      int(b0), int(b1), int(stride), _lib.ptr(vals), cnt, _lib.ptr(secs))
    if config.algorithm == "dito":
        # the order the engine left the moments at (its own cap may have been
        # lowered to fit the device's memory)
        order = ctypes.c_int32(0)
        _lib.call("fg_moments_export", rtree.handle, None, None, None, ctypes.byref(order))
        rtree._moments_refreshed(float(hs[-1]),
                                 int(order.value) or int(plimit) or engine_plimit(qtree.dim))
    rows = vals.reshape(nh, qtree.n)
    return [ResultVector(rows[j], float(secs[j]), TraversalCounters._from_c(cnt[j]), None)
            for j in range(nh)]


def query_block_count(qtree: KdTree) -> int:
    """Number of query blocks (<= 64 points each; the unit of query sharding)."""
    nb = ctypes.c_int64()
    _lib.call("fg_query_blocks", qtree.handle, ctypes.byref(nb))
    return nb.value


def run_blocks(config: RunConfig, qtree: KdTree, rtree: KdTree, block_begin: int,
               block_end: int, block_stride: int = 1, out=None) -> ResultVector:
    """Run ``config.algorithm`` on query blocks block_begin, block_begin +
    block_stride, ... (< block_end) only; other entries of ``out`` are kept."""
    vals = out if out is not None else np.zeros(qtree.n)
    res = _run_tree_algorithm(config, qtree, rtree, config.algorithm, False, vals,
                              (block_begin, block_end, block_stride))
    return res


def dito_post(qtree: KdTree) -> None:
    """Push node-level estimates and local polynomials of the host mirror
    state down to the points (summation_engine.py:253-281).

    The device engine applies this pass inside each run; this function serves
    callers that populate the mirror state (``reset_query_state`` fields)
    themselves.  Shifts and evaluations run on the device.
    """
    from .series_expansion import add_local, eval_local, translate_l2l

    if qtree.q_est is None:
        raise RuntimeError("query state not initialised; call reset_query_state first")
    pts = qtree.points
    stack = [qtree.root]
    while stack:
        node = stack.pop()
        if node.is_leaf:
            if node.est != 0.0:
                qtree.q_est[node.start:node.end] += node.est
            if node.local_used:
                qtree.q_est[node.start:node.end] += eval_local(node.local,
                                                               pts[node.start:node.end])
            continue
        for child in (node.left, node.right):
            child.est += node.est
            if node.local_used:
                add_local(child.local, translate_l2l(node.local, child.center))
                child.local_used = True
        node.est = 0.0
        stack.append(node.right)
        stack.append(node.left)
