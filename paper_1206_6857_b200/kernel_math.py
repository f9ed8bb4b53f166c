"""Multi-index combinatorics (graded-lex index sets) and small constants.

The reference's kernel_math.py (:20-36 factorials/binomials, :111-136
enumeration, :139-209 MultiIndexSet) is the table-building half of its series
algebra.  Here the tables come from the engine itself (``fg_iset_export``,
the host half of the tables the kernels use; no GPU needed), so the host
mirror and the device agree by construction.  The numeric series work
(Hermite ladders, products) runs on the GPU.
"""

from __future__ import annotations

import ctypes
import math
from functools import lru_cache

import numpy as np

from . import _lib

_MAX_FACTORIAL = 34
_FACTORIALS = np.array([float(math.factorial(n)) for n in range(_MAX_FACTORIAL + 1)])


def factorial(n: int) -> float:
    return _FACTORIALS[n]


def binomial(n: int, k: int) -> int:
    return math.comb(n, k)


def _engine_tables(dim: int, order: int):
    if dim <= 0:
        raise ValueError("dimension must be positive")
    if order <= 0:
        raise ValueError("truncation order must be positive")
    K = ctypes.c_int32()
    npairs = ctypes.c_int32()
    _lib.call("fg_iset_export", dim, order, ctypes.byref(K), None, None, None, None,
              ctypes.byref(npairs), None)
    k, n = K.value, npairs.value
    digits = np.empty((k, dim), np.int32)
    degrees = np.empty(k, np.int32)
    fact = np.empty(k)
    prefix = np.empty(order + 1, np.int32)
    pairs = np.empty((max(n, 1), 3), np.int32)
    _lib.call("fg_iset_export", dim, order, None, _lib.ptr(digits), _lib.ptr(degrees),
              _lib.ptr(fact), _lib.ptr(prefix), None, _lib.ptr(pairs))
    return digits, degrees, fact, prefix, pairs[:n]


def enumerate_multi_indices(dim: int, order: int) -> list[tuple[int, ...]]:
    """All multi-indices with |alpha| < order in graded-lex order (by degree,
    then leading digit descending)."""
    digits = _engine_tables(dim, order)[0]
    return [tuple(int(v) for v in row) for row in digits]


class MultiIndexSet:
    """Digits, degrees, alpha!, prefix counts and shift pairs of an index set."""

    def __init__(self, dim: int, order: int):
        digits, degrees, fact, prefix, pairs = _engine_tables(dim, order)
        self.dim = dim
        self.order = order
        self.count = digits.shape[0]
        self.digits = digits.astype(np.intp)
        self.degrees = degrees.astype(np.intp)
        self.fact = fact
        self.inv_fact = 1.0 / fact
        self.position = {tuple(int(v) for v in row): k for k, row in enumerate(digits)}
        self.prefix_counts = prefix.astype(np.intp)
        self.shift_pairs = tuple(pairs[:, c].astype(np.intp) for c in range(3))

    def count_below(self, p: int) -> int:
        return int(self.prefix_counts[p])


@lru_cache(maxsize=None)
def index_set(dim: int, order: int) -> MultiIndexSet:
    return MultiIndexSet(dim, order)
