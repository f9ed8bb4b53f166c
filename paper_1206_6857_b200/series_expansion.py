"""Far-field / local expansions on the device (mirror of series_expansion.py).

Same names, arguments and error behaviour as the reference module
(/root/reference/pkg/src/fastgauss/series_expansion.py); every numeric
operation runs in the engine's CUDA kernels (fg_series.cu) through the C ABI.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from . import _lib
from .kernel_math import index_set

_SQRT2 = math.sqrt(2.0)


@dataclass
class FarFieldExpansion:
    """A_alpha = sum_r (w_r/alpha!) ((x_r - c)/sqrt(2h^2))^alpha  (:36-51)."""

    center: np.ndarray
    order: int
    coeffs: np.ndarray
    bandwidth: float

    @property
    def dim(self) -> int:
        return self.center.shape[0]


@dataclass
class LocalExpansion:
    """Polynomial coefficients B_beta in the scaled offset from ``center`` (:54-69)."""

    center: np.ndarray
    order: int
    coeffs: np.ndarray
    bandwidth: float

    @property
    def dim(self) -> int:
        return self.center.shape[0]


def _accumulate(kind, points, weights, center, order, h):
    if order < 1:
        raise ValueError("truncation order must be at least 1")
    center = np.ascontiguousarray(center, dtype=float).reshape(-1)
    dim = center.shape[0]
    points = np.ascontiguousarray(points, dtype=float).reshape(-1, dim)
    weights = np.ascontiguousarray(weights, dtype=float).reshape(-1)
    count = index_set(dim, order).count
    out = np.zeros(count)
    off = np.array([0, points.shape[0]], dtype=np.int64)
    if points.shape[0]:
        _lib.call("fg_series_accumulate", kind, _lib.ptr(points), _lib.ptr(weights),
                  _lib.ptr(off), 1, dim, _lib.ptr(center), order, float(h), _lib.ptr(out))
    return center, out


def accumulate_far_field(points, weights, center, order: int, h: float) -> FarFieldExpansion:
    """series_expansion.py:76-92 on the device."""
    c, coeffs = _accumulate(0, points, weights, center, order, h)
    return FarFieldExpansion(c, order, coeffs, h)


def accumulate_local_direct(points, weights, center, order: int, h: float) -> LocalExpansion:
    """series_expansion.py:110-126 on the device."""
    c, coeffs = _accumulate(1, points, weights, center, order, h)
    return LocalExpansion(c, order, coeffs, h)


def _eval(kind, exp, x, order):
    p = exp.order if order is None else order
    x = np.asarray(x, dtype=float)
    scalar = x.ndim == 1
    pts = np.ascontiguousarray(x.reshape(-1, exp.dim))
    coeffs = np.ascontiguousarray(exp.coeffs, dtype=float)
    out = np.empty(pts.shape[0])
    off = np.array([0, pts.shape[0]], dtype=np.int64)
    center = np.ascontiguousarray(exp.center, dtype=float)
    _lib.call("fg_series_eval", kind, _lib.ptr(coeffs), coeffs.shape[0], _lib.ptr(center), 1,
              exp.dim, p, float(exp.bandwidth), _lib.ptr(pts), _lib.ptr(off), _lib.ptr(out))
    return out[0] if scalar else out.reshape(x.shape[:-1])


def eval_far_field(exp: FarFieldExpansion, x, order: int | None = None):
    """series_expansion.py:95-107 (EVALM) on the device."""
    return _eval(0, exp, x, order)


def eval_local(exp: LocalExpansion, x, order: int | None = None):
    """series_expansion.py:129-136 (EVALL) on the device."""
    return _eval(1, exp, x, order)


def _translate(kind, exp, new_center, order_src, order):
    new_center = np.ascontiguousarray(new_center, dtype=float).reshape(-1)
    if new_center.shape != exp.center.shape:
        raise ValueError("center dimension mismatch")
    coeffs = np.ascontiguousarray(exp.coeffs, dtype=float)
    out = np.empty(index_set(exp.dim, order).count)
    src = np.ascontiguousarray(exp.center, dtype=float)
    _lib.call("fg_series_translate", kind, _lib.ptr(coeffs), coeffs.shape[0], _lib.ptr(src),
              _lib.ptr(new_center), 1, exp.dim, order_src, order, float(exp.bandwidth),
              _lib.ptr(out))
    return new_center, out


def translate_h2h(exp: FarFieldExpansion, new_center) -> FarFieldExpansion:
    """series_expansion.py:139-157 (exact moment shift) on the device."""
    c, out = _translate(0, exp, new_center, exp.order, exp.order)
    return FarFieldExpansion(c, exp.order, out, exp.bandwidth)


def add_far_field(dst: FarFieldExpansion, src: FarFieldExpansion) -> None:
    """series_expansion.py:160-164."""
    if dst.order != src.order or dst.bandwidth != src.bandwidth:
        raise ValueError("expansion order/bandwidth mismatch")
    dst.coeffs += src.coeffs


def translate_h2l(exp: FarFieldExpansion, dest_center, dest_order: int,
                  src_order: int | None = None) -> LocalExpansion:
    """series_expansion.py:167-194 on the device."""
    if dest_order < 1:
        raise ValueError("truncation order must be at least 1")
    p_src = exp.order if src_order is None else src_order
    c, out = _translate(2, exp, dest_center, p_src, dest_order)
    return LocalExpansion(c, dest_order, out, exp.bandwidth)


def translate_l2l(exp: LocalExpansion, new_center) -> LocalExpansion:
    """series_expansion.py:197-217 (exact polynomial shift) on the device."""
    c, out = _translate(1, exp, new_center, exp.order, exp.order)
    return LocalExpansion(c, exp.order, out, exp.bandwidth)


def add_local(dst: LocalExpansion, src: LocalExpansion) -> None:
    """series_expansion.py:220-228: a lower-order src fills the leading prefix."""
    if src.order > dst.order or dst.bandwidth != src.bandwidth:
        raise ValueError("expansion order/bandwidth mismatch")
    dst.coeffs[: src.coeffs.shape[0]] += src.coeffs
