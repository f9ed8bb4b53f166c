"""Multi-index combinatorics (graded-lex index sets) and small constants.

Restates the table-building half of the reference's kernel_math.py
(:20-36 factorials/binomials, :111-136 enumeration, :139-209 MultiIndexSet
tables).  These are integer metadata consumed by the device kernels; the
numeric series work (Hermite ladders, products) runs on the GPU.
"""

from __future__ import annotations

import math
from functools import lru_cache

import numpy as np

_MAX_FACTORIAL = 34
_FACTORIALS = np.array([float(math.factorial(n)) for n in range(_MAX_FACTORIAL + 1)])


def factorial(n: int) -> float:
    return _FACTORIALS[n]


def binomial(n: int, k: int) -> int:
    return math.comb(n, k)


def _compositions(total: int, dims: int):
    # leading digit descending within a degree (kernel_math.py:111-119)
    if dims == 1:
        yield (total,)
        return
    for head in range(total, -1, -1):
        for rest in _compositions(total - head, dims - 1):
            yield (head,) + rest


def enumerate_multi_indices(dim: int, order: int) -> list[tuple[int, ...]]:
    """All multi-indices with |alpha| < order in graded-lex order."""
    if dim <= 0:
        raise ValueError("dimension must be positive")
    if order <= 0:
        raise ValueError("truncation order must be positive")
    out = []
    for degree in range(order):
        out.extend(_compositions(degree, dim))
    return out


class MultiIndexSet:
    """Digits, degrees, alpha!, prefix counts and shift pairs of an index set."""

    def __init__(self, dim: int, order: int):
        indices = enumerate_multi_indices(dim, order)
        self.dim = dim
        self.order = order
        self.count = len(indices)
        self.digits = np.array(indices, dtype=np.intp).reshape(self.count, dim)
        self.degrees = self.digits.sum(axis=1)
        self.fact = _FACTORIALS[self.digits].prod(axis=1)
        self.inv_fact = 1.0 / self.fact
        self.position = {idx: k for k, idx in enumerate(indices)}
        self.prefix_counts = np.searchsorted(self.degrees, np.arange(order + 1))
        self._pairs = None

    def count_below(self, p: int) -> int:
        return int(self.prefix_counts[p])

    @property
    def shift_pairs(self):
        if self._pairs is None:
            a_idx, b_idx, s_idx = [], [], []
            for a in range(self.count):
                for b in range(self.count):
                    if self.degrees[a] + self.degrees[b] >= self.order:
                        continue
                    a_idx.append(a)
                    b_idx.append(b)
                    s_idx.append(self.position[tuple(self.digits[a] + self.digits[b])])
            self._pairs = tuple(np.array(v, dtype=np.intp) for v in (a_idx, b_idx, s_idx))
        return self._pairs


@lru_cache(maxsize=None)
def index_set(dim: int, order: int) -> MultiIndexSet:
    return MultiIndexSet(dim, order)
