"""Truncation-error bounds and the approximation selector (mirror of error_bounds.py).

``best_method`` (error_bounds.py:168-230) is evaluated by the same device
routine the traversal kernel uses (fg_series.cuh: best_method_dev), batched
through the C ABI.  The closed-form single-bound helpers and the tail-table
constants (:73-159) are scalar host formulas kept for API parity.
"""

from __future__ import annotations

import math
from dataclasses import dataclass
from enum import Enum
from functools import lru_cache

import numpy as np

from . import _lib

_SQRT2 = math.sqrt(2.0)


class Method(Enum):
    EXHAUSTIVE = "exhaustive"
    FINITE_DIFF = "fd"
    HERMITE = "hermite"
    LOCAL = "local"
    H2L = "h2l"


_CODES = {0: Method.EXHAUSTIVE, 2: Method.HERMITE, 3: Method.LOCAL, 4: Method.H2L}


@dataclass
class MethodChoice:
    method: Method
    order: int | None
    bound: float
    cost: float


@dataclass
class NodePairGeometry:
    """Squared box distances, radii already divided by h, node statistics (:53-70)."""

    min_sqdist: float
    max_sqdist: float
    r_ref: float
    r_query: float
    weight_ref: float
    n_query: int
    n_ref: int
    dim: int
    bandwidth: float


@lru_cache(maxsize=None)
def _tail_tables(dim: int, plimit: int):
    """count[p] = C(D+p-1, D-1), denom[p], cross[p] = C(D+p-1, D)  (:73-92)."""
    count = np.zeros(plimit + 1)
    denom = np.ones(plimit + 1)
    cross = np.zeros(plimit + 1)
    for p in range(1, plimit + 1):
        count[p] = math.comb(dim + p - 1, dim - 1)
        q, r = divmod(p, dim)
        denom[p] = math.sqrt(math.factorial(q) ** (dim - r) * math.factorial(q + 1) ** r)
        cross[p] = math.comb(dim + p - 1, dim)
    return count, denom, cross


def _prefactor(geom):
    return math.exp(-0.25 * geom.min_sqdist / (geom.bandwidth * geom.bandwidth))


def fd_bound(geom: NodePairGeometry) -> float:
    inv = -0.5 / (geom.bandwidth * geom.bandwidth)
    spread = math.exp(geom.min_sqdist * inv) - math.exp(geom.max_sqdist * inv)
    return 0.5 * geom.weight_ref * max(spread, 0.0)


def hermite_bound(p: int, geom: NodePairGeometry) -> float:
    count, denom, _ = _tail_tables(geom.dim, max(p, 1))
    return geom.weight_ref * _prefactor(geom) * count[p] * geom.r_ref ** p / denom[p]


def local_bound(p: int, geom: NodePairGeometry) -> float:
    count, denom, _ = _tail_tables(geom.dim, max(p, 1))
    return geom.weight_ref * _prefactor(geom) * count[p] * geom.r_query ** p / denom[p]


def h2l_bound(p: int, geom: NodePairGeometry) -> float:
    count, denom, cross = _tail_tables(geom.dim, max(p, 1))
    pref = _prefactor(geom) * count[p] / denom[p]
    sq = _SQRT2 * geom.r_query
    step = 1.0 if sq <= 1.0 else sq ** (p - 1)
    return geom.weight_ref * (pref * geom.r_query ** p
                              + pref * (_SQRT2 * geom.r_ref) ** p * cross[p] * step)


@lru_cache(maxsize=None)
def series_floor_constant(dim: int, plimit: int) -> float:
    count, denom, _ = _tail_tables(dim, plimit)
    return float(min(count[p] / denom[p] for p in range(1, plimit + 1)))


def best_method_batch(geoms, maxerrs, plimit: int):
    """Vectorised best_method over many geometries of one dimension (device)."""
    geoms = list(geoms)
    if not geoms:
        return []
    dim = geoms[0].dim
    rows = np.array([[g.min_sqdist, g.max_sqdist, g.r_ref, g.r_query, g.weight_ref,
                      g.n_query, g.n_ref, g.bandwidth, m] for g, m in zip(geoms, maxerrs)],
                    dtype=float)
    out = np.empty((len(geoms), 4))
    _lib.call("fg_best_method", _lib.ptr(rows), len(geoms), dim, int(plimit), _lib.ptr(out))
    return [MethodChoice(_CODES[int(o[0])], int(o[1]) or None, float(o[2]), float(o[3]))
            for o in out]


def best_method(geom: NodePairGeometry, maxerr: float, plimit: int) -> MethodChoice:
    """Cheapest feasible series method, else exhaustive (:168-230), on the device."""
    return best_method_batch([geom], [maxerr], plimit)[0]
