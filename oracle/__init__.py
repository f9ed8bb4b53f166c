"""CPU oracle for the fastgauss hot path -- TEST INFRASTRUCTURE ONLY.

A plain-C restatement (``fg_oracle.c``) of the reference package
``fastgauss`` (``/root/reference/pkg/src/fastgauss``), wrapped with ctypes.
Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (its
``cpu_baseline`` leg and ``--impl reference``) may import this module, and
only as the checker / CPU baseline: the B200 product path in
``paper_1206_6857_b200`` never calls it.

Pinning: ``tests/test_oracle_pins.py`` checks this oracle against the golden
vectors in ``tests/golden/`` (made by ``tests/golden/make_golden.py`` from the
unmodified reference) and against the reference's own known-answer tests.
"""

from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "libfg_oracle.so")
_lib = None

_D = ctypes.POINTER(ctypes.c_double)
_I64 = ctypes.POINTER(ctypes.c_int64)
_I32 = ctypes.POINTER(ctypes.c_int)


def build() -> str:
    """Compile the oracle library in-tree (make)."""
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        L = ctypes.CDLL(_LIB_PATH)
        L.fgo_build_tree.restype = ctypes.c_void_p
        L.fgo_build_tree.argtypes = [_D, _D, ctypes.c_int64, ctypes.c_int, ctypes.c_int]
        L.fgo_tree_free.argtypes = [ctypes.c_void_p]
        L.fgo_tree_nnodes.restype = ctypes.c_int64
        L.fgo_tree_nnodes.argtypes = [ctypes.c_void_p]
        L.fgo_tree_export.argtypes = [ctypes.c_void_p] + [ctypes.c_void_p] * 10
        L.fgo_refresh_moments.argtypes = [ctypes.c_void_p, ctypes.c_double, ctypes.c_int]
        L.fgo_moments_count.argtypes = [ctypes.c_void_p]
        L.fgo_tree_export_moments.argtypes = [ctypes.c_void_p, _D]
        L.fgo_run.restype = ctypes.c_int
        L.fgo_run.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_double,
                              ctypes.c_double, ctypes.c_int, ctypes.c_int, _D, _I64]
        L.fgo_run_sharded.restype = ctypes.c_int
        L.fgo_run_sharded.argtypes = [_D, ctypes.c_int64, ctypes.c_void_p, ctypes.c_int,
                                      ctypes.c_double, ctypes.c_double, ctypes.c_int,
                                      ctypes.c_int, ctypes.c_int, _D, _I64]
        L.fgo_naive_sum.argtypes = [_D, ctypes.c_int64, _D, _D, ctypes.c_int64,
                                    ctypes.c_int, ctypes.c_double, _D]
        L.fgo_naive_sum_mt.argtypes = [_D, ctypes.c_int64, _D, _D, ctypes.c_int64,
                                       ctypes.c_int, ctypes.c_double, _D, ctypes.c_int]
        L.fgo_naive_sum_comp_mt.argtypes = L.fgo_naive_sum_mt.argtypes
        L.fgo_best_method.argtypes = [ctypes.c_double] * 5 + [ctypes.c_int64] * 2 + [
            ctypes.c_int, ctypes.c_double, ctypes.c_double, ctypes.c_int,
            _I32, _I32, _D, _D]
        L.fgo_series_floor_constant.restype = ctypes.c_double
        L.fgo_series_floor_constant.argtypes = [ctypes.c_int, ctypes.c_int]
        L.fgo_tail_tables.argtypes = [ctypes.c_int, ctypes.c_int, _D, _D, _D]
        L.fgo_iset_count.restype = ctypes.c_int
        L.fgo_iset_count.argtypes = [ctypes.c_int, ctypes.c_int]
        L.fgo_iset_export.argtypes = [ctypes.c_int, ctypes.c_int, _I32, _I32, _D, _I32, _I32]
        L.fgo_hermite_ladder.argtypes = [_D, ctypes.c_int64, ctypes.c_int, _D]
        L.fgo_power_table.argtypes = [_D, ctypes.c_int64, ctypes.c_int, _D]
        L.fgo_accumulate_far_field.argtypes = [_D, _D, ctypes.c_int64, ctypes.c_int, _D,
                                               ctypes.c_int, ctypes.c_double, _D]
        L.fgo_accumulate_local_direct.argtypes = L.fgo_accumulate_far_field.argtypes
        L.fgo_eval_far_field.argtypes = [_D, _D, ctypes.c_int, ctypes.c_int, ctypes.c_double,
                                         _D, ctypes.c_int64, _D]
        L.fgo_eval_local.argtypes = L.fgo_eval_far_field.argtypes
        L.fgo_translate_h2h.argtypes = [_D, _D, _D, ctypes.c_int, ctypes.c_int,
                                        ctypes.c_double, _D]
        L.fgo_translate_l2l.argtypes = L.fgo_translate_h2h.argtypes
        L.fgo_translate_h2l.argtypes = [_D, _D, _D, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                        ctypes.c_double, _D]
        _lib = L
    return _lib


def _dp(a):
    return a.ctypes.data_as(_D)


def _f64(a, shape=None):
    a = np.ascontiguousarray(a, dtype=np.float64)
    if shape is not None:
        a = a.reshape(shape)
    return a


# ----------------------------------------------------------------- engine
def naive_sum(queries, references, weights, h, threads: int = 1, compensated: bool = False):
    """summation_engine.py:122-154 restated (exact FP64 sums).  ``compensated``
    sums the same terms with Neumaier compensation (full-size fixtures)."""
    q = _f64(queries)
    if q.ndim == 1:
        q = q.reshape(1, -1)
    r = _f64(references)
    w = _f64(weights).reshape(-1)
    out = np.empty(q.shape[0])
    if compensated:
        lib().fgo_naive_sum_comp_mt(_dp(q), q.shape[0], _dp(r), _dp(w), r.shape[0], q.shape[1],
                                    float(h), _dp(out), int(threads))
    elif threads == 1:
        lib().fgo_naive_sum(_dp(q), q.shape[0], _dp(r), _dp(w), r.shape[0], q.shape[1],
                            float(h), _dp(out))
    else:
        lib().fgo_naive_sum_mt(_dp(q), q.shape[0], _dp(r), _dp(w), r.shape[0], q.shape[1],
                               float(h), _dp(out), int(threads))
    return out


class Tree:
    """spatial_index.py:144-276 restated: a kd-tree built by the C oracle."""

    def __init__(self, points, weights=None, leaf_threshold: int = 25):
        p = _f64(points)
        w = np.ones(p.shape[0]) if weights is None else _f64(weights).reshape(-1)
        self._keep = (p, w)
        self.dim = p.shape[1]
        self.n = p.shape[0]
        self.h = lib().fgo_build_tree(_dp(p), _dp(w), p.shape[0], p.shape[1], leaf_threshold)
        if not self.h:
            raise ValueError("oracle build_tree rejected its input")

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None:
            _lib.fgo_tree_free(self.h)
            self.h = None

    def export(self):
        L = lib()
        nn = L.fgo_tree_nnodes(self.h)
        D = self.dim
        out = dict(
            perm=np.empty(self.n, np.int64), start=np.empty(nn, np.int64),
            end=np.empty(nn, np.int64), lo=np.empty((nn, D)), hi=np.empty((nn, D)),
            center=np.empty((nn, D)), weight=np.empty(nn), inf_radius=np.empty(nn),
            left=np.empty(nn, np.int64), right=np.empty(nn, np.int64))
        L.fgo_tree_export(self.h, *[out[k].ctypes.data for k in
                                    ("perm", "start", "end", "lo", "hi", "center", "weight",
                                     "inf_radius", "left", "right")])
        return out

    def refresh_moments(self, h: float, plimit: int):
        lib().fgo_refresh_moments(self.h, float(h), int(plimit))

    def moments(self):
        L = lib()
        nn = L.fgo_tree_nnodes(self.h)
        K = L.fgo_moments_count(self.h)
        out = np.empty((nn, K))
        L.fgo_tree_export_moments(self.h, _dp(out))
        return out


_MODES = {"dfd": 1, "dfdo": 2, "dito": 3}


def run(algorithm: str, qtree: Tree, rtree: Tree, h: float, eps: float, plimit=None):
    """summation_engine.py:431-480 restated (depth-first dual-tree traversal)."""
    vals = np.empty(qtree.n)
    cnt = np.zeros(6, np.int64)
    st = lib().fgo_run(qtree.h, rtree.h, float(h), float(eps), _MODES[algorithm],
                       int(plimit or 0), _dp(vals), cnt.ctypes.data_as(_I64))
    if st == 2:
        raise RuntimeError("reference moments missing or stale")
    return vals, cnt


def run_sharded(algorithm, queries, rtree: Tree, h, eps, plimit=None, threads=0,
                leaf_threshold=25):
    """The unmodified DFS algorithm on `threads` disjoint query shards (CPU baseline)."""
    q = _f64(queries)
    vals = np.empty(q.shape[0])
    cnt = np.zeros(6, np.int64)
    st = lib().fgo_run_sharded(_dp(q), q.shape[0], rtree.h, leaf_threshold, float(h),
                               float(eps), _MODES[algorithm], int(plimit or 0), int(threads),
                               _dp(vals), cnt.ctypes.data_as(_I64))
    if st == 2:
        raise RuntimeError("reference moments missing or stale")
    return vals, cnt


# ---------------------------------------------------------------- series
def iset(dim, order):
    L = lib()
    K = L.fgo_iset_count(dim, order)
    digits = np.empty((K, dim), np.int32)
    deg = np.empty(K, np.int32)
    fact = np.empty(K)
    npairs = ctypes.c_int(0)
    L.fgo_iset_export(dim, order, digits.ctypes.data_as(_I32), deg.ctypes.data_as(_I32),
                      _dp(fact), ctypes.byref(npairs), None)
    pairs = np.empty((npairs.value, 3), np.int32)
    L.fgo_iset_export(dim, order, None, None, None, ctypes.byref(npairs),
                      pairs.ctypes.data_as(_I32))
    return digits, deg, fact, pairs


def hermite_ladder(t, max_order):
    t = _f64(t)
    out = np.empty(t.shape + (max_order + 1,))
    lib().fgo_hermite_ladder(_dp(t.reshape(-1)), t.size, max_order, _dp(out))
    return out


def power_table(u, max_power):
    u = _f64(u)
    out = np.empty(u.shape + (max_power + 1,))
    lib().fgo_power_table(_dp(u.reshape(-1)), u.size, max_power, _dp(out))
    return out


def accumulate_far_field(points, weights, center, order, h):
    c = _f64(center).reshape(-1)
    p = _f64(points).reshape(-1, c.shape[0])
    w = _f64(weights).reshape(-1)
    out = np.empty(lib().fgo_iset_count(c.shape[0], order))
    lib().fgo_accumulate_far_field(_dp(p), _dp(w), p.shape[0], c.shape[0], _dp(c), order,
                                   float(h), _dp(out))
    return out


def accumulate_local_direct(points, weights, center, order, h):
    c = _f64(center).reshape(-1)
    p = _f64(points).reshape(-1, c.shape[0])
    w = _f64(weights).reshape(-1)
    out = np.empty(lib().fgo_iset_count(c.shape[0], order))
    lib().fgo_accumulate_local_direct(_dp(p), _dp(w), p.shape[0], c.shape[0], _dp(c), order,
                                      float(h), _dp(out))
    return out


def eval_far_field(coeffs, center, order, h, x):
    c = _f64(center).reshape(-1)
    x = _f64(x).reshape(-1, c.shape[0])
    co = _f64(coeffs)
    out = np.empty(x.shape[0])
    lib().fgo_eval_far_field(_dp(co), _dp(c), c.shape[0], order, float(h), _dp(x),
                             x.shape[0], _dp(out))
    return out


def eval_local(coeffs, center, order, h, x):
    c = _f64(center).reshape(-1)
    x = _f64(x).reshape(-1, c.shape[0])
    co = _f64(coeffs)
    out = np.empty(x.shape[0])
    lib().fgo_eval_local(_dp(co), _dp(c), c.shape[0], order, float(h), _dp(x), x.shape[0],
                         _dp(out))
    return out


def translate_h2h(coeffs, old_c, new_c, order, h):
    o = _f64(old_c).reshape(-1)
    n = _f64(new_c).reshape(-1)
    co = _f64(coeffs)
    out = np.empty(lib().fgo_iset_count(o.shape[0], order))
    lib().fgo_translate_h2h(_dp(co), _dp(o), _dp(n), o.shape[0], order, float(h), _dp(out))
    return out


def translate_l2l(coeffs, old_c, new_c, order, h):
    o = _f64(old_c).reshape(-1)
    n = _f64(new_c).reshape(-1)
    co = _f64(coeffs)
    out = np.empty(lib().fgo_iset_count(o.shape[0], order))
    lib().fgo_translate_l2l(_dp(co), _dp(o), _dp(n), o.shape[0], order, float(h), _dp(out))
    return out


def translate_h2l(coeffs, src_c, dst_c, src_order, dst_order, h):
    s = _f64(src_c).reshape(-1)
    d = _f64(dst_c).reshape(-1)
    co = _f64(coeffs)
    out = np.empty(lib().fgo_iset_count(s.shape[0], dst_order))
    lib().fgo_translate_h2l(_dp(co), _dp(s), _dp(d), s.shape[0], src_order, dst_order,
                            float(h), _dp(out))
    return out


def best_method(min_sq, max_sq, r_ref, r_query, w_ref, n_query, n_ref, dim, h, maxerr,
                plimit):
    m = ctypes.c_int(0)
    p = ctypes.c_int(0)
    b = ctypes.c_double(0)
    c = ctypes.c_double(0)
    lib().fgo_best_method(min_sq, max_sq, r_ref, r_query, w_ref, n_query, n_ref, dim, h,
                          maxerr, plimit, ctypes.byref(m), ctypes.byref(p), ctypes.byref(b),
                          ctypes.byref(c))
    names = {0: "exhaustive", 2: "hermite", 3: "local", 4: "h2l"}
    return names[m.value], (p.value or None), b.value, c.value


def series_floor_constant(dim, plimit):
    return lib().fgo_series_floor_constant(dim, plimit)


def max_rel_error(estimates, exact):
    """cli_harness.py:216-226 restated."""
    exact = np.asarray(exact, dtype=float)
    estimates = np.asarray(estimates, dtype=float)
    err = np.zeros_like(exact)
    pos = exact > 0.0
    err[pos] = np.abs(estimates[pos] - exact[pos]) / exact[pos]
    if np.any(~pos & (estimates != 0.0)):
        return float("inf")
    return float(err.max()) if err.size else 0.0
