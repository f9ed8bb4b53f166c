"""Callers of the hot path: the parity metric, the LSCV score
that Config 4 measures, and least-squares cross-validation bandwidth selection,
all running their kernel sums on the device engine.

Restates cli_harness.py:101-157 (select_bandwidth + score) and :216-226
(max_rel_error).  The score arithmetic on the two sums is O(n) host work, as in
the reference; the sums themselves are device runs.
"""

from __future__ import annotations

import math

import numpy as np

from .spatial_index import KdTree, PointStore, build_tree
from .summation_engine import RunConfig, sweep_run


def max_rel_error(estimates, exact) -> float:
    """max_q |est - exact| / exact, exact zeros must be matched (cli_harness.py:216-226)."""
    exact = np.asarray(exact, dtype=float)
    estimates = np.asarray(estimates, dtype=float)
    err = np.zeros_like(exact)
    pos = exact > 0.0
    err[pos] = np.abs(estimates[pos] - exact[pos]) / exact[pos]
    if np.any(~pos & (estimates != 0.0)):
        return float("inf")
    return float(err.max()) if err.size else 0.0


def lscv_scores(tree: KdTree, hs, epsilon: float = 1e-3, algorithm: str = "dfd") -> list:
    """LSCV scores of a Gaussian KDE with unit weights (cli_harness.py:128-137):

        (2 pi 2h^2)^(-D/2) sum G_{sqrt2 h} / n^2
          - 2 (2 pi h^2)^(-D/2) (sum G_h - n) / (n (n-1))

    for every h in ``hs``; all 2 len(hs) monochromatic sums run as one device
    sweep (the self term is removed by `- n`).
    """
    n, dim = tree.n, tree.dim
    hs = [float(h) for h in hs]
    bws = [b for h in hs for b in (math.sqrt(2.0) * h, h)]
    res = sweep_run(RunConfig(bandwidth=bws[0], epsilon=epsilon, algorithm=algorithm), tree,
                    tree, bws)
    out = []
    for i, h in enumerate(hs):
        conv, near = res[2 * i].values, res[2 * i + 1].values
        norm_conv = (2.0 * math.pi * 2.0 * h * h) ** (-0.5 * dim)
        norm_near = (2.0 * math.pi * h * h) ** (-0.5 * dim)
        integral_sq = norm_conv * float(conv.sum()) / (n * n)
        leave_one_out = norm_near * 2.0 * float(near.sum() - n) / (n * (n - 1))
        out.append(integral_sq - leave_one_out)
    return out


def lscv_score(tree: KdTree, h: float, epsilon: float = 1e-3, algorithm: str = "dfd") -> float:
    """LSCV score at one bandwidth (see :func:`lscv_scores`)."""
    return lscv_scores(tree, [h], epsilon, algorithm)[0]


def select_bandwidth(points, seed: int = 0, epsilon: float = 1e-3, max_points: int = 2000,
                     algorithm: str = "dfd") -> float:
    """LSCV bandwidth: 14-point geometric grid over [1e-3, 0.5] x diameter, then a
    golden-section search in log h down to width 0.02 (cli_harness.py:101-157)."""
    points = np.asarray(points, dtype=float)
    if points.ndim == 1:
        points = points.reshape(-1, 1)
    if points.shape[0] < 2:
        raise ValueError("bandwidth selection needs at least two points")
    lo = points.min(axis=0)
    hi = points.max(axis=0)
    if np.all(hi == lo):
        raise ValueError("all points identical; no finite bandwidth minimizes LSCV")
    if points.shape[0] > max_points:
        idx = np.random.default_rng(seed).choice(points.shape[0], max_points, replace=False)
        points = points[idx]
    scale = float(np.linalg.norm(hi - lo))
    tree = build_tree(PointStore(points))

    def score(h):
        return lscv_score(tree, h, epsilon, algorithm)

    grid = np.geomspace(1e-3 * scale, 0.5 * scale, 14)
    scores = lscv_scores(tree, grid, epsilon, algorithm)  # the whole grid in one sweep
    best = int(np.argmin(scores))
    a = math.log(grid[max(best - 1, 0)])
    b = math.log(grid[min(best + 1, len(grid) - 1)])
    invphi = 0.5 * (math.sqrt(5.0) - 1.0)
    c = b - invphi * (b - a)
    d = a + invphi * (b - a)
    fc, fd = lscv_scores(tree, [math.exp(c), math.exp(d)], epsilon, algorithm)
    while b - a > 0.02:
        if fc < fd:
            b, d, fd = d, c, fc
            c = b - invphi * (b - a)
            fc = score(math.exp(c))
        else:
            a, c, fc = c, d, fd
            d = a + invphi * (b - a)
            fd = score(math.exp(d))
    return math.exp(0.5 * (a + b))


def telescoping_audit(ledger, qtree: KdTree, exact, epsilon: float) -> dict:
    """Theorem-2 telescoping check over an audit ledger and the
    accounting invariant, per query node of the ledger:

    * worst_ratio = max over query blocks of  sum(bound) / (eps * min_q G(q)),
      G the exact sums (original order); <= 1 is the guarantee.  Every bound
      is an absolute error bound for every query of its block;
    * weight_error = max relative deviation of sum(W_R) from n_blocks * W:
      every reference's weight is settled exactly once per query block.
    """
    from .summation_engine import query_block_nodes, query_block_ranges

    e = qtree.arrays()
    exact_tree = np.asarray(exact, dtype=float)[e["perm"]]
    blocks = getattr(ledger, "blocks", None)
    if blocks is not None:
        # per query block: its own queries' minimum exact sum, one settlement of
        # every reference weight
        starts, counts = query_block_ranges(qtree)
        total_w = float(e["weight"][0])
        bsum = np.bincount(blocks, weights=[t[3] for t in ledger], minlength=len(starts))
        wsum = np.bincount(blocks, weights=[t[2] for t in ledger], minlength=len(starts))
        used = np.unique(blocks)
        worst, werr = 0.0, 0.0
        for b in used:
            g = float(exact_tree[starts[b]:starts[b] + counts[b]].min())
            if bsum[b] > 0.0:
                worst = max(worst, bsum[b] / (epsilon * g) if g > 0.0 else float("inf"))
            werr = max(werr, abs(wsum[b] - total_w) / total_w)
        return {"worst_ratio": worst, "weight_error": werr, "query_nodes": len(used)}
    blocks_per_node = np.bincount(query_block_nodes(qtree), minlength=len(e["start"]))
    bound = {}
    wsum = {}
    for kind, v, w_ref, bd, _, _ in ledger:
        bound[v] = bound.get(v, 0.0) + bd
        wsum[v] = wsum.get(v, 0.0) + w_ref
    total_w = float(e["weight"][0])
    worst, werr = 0.0, 0.0
    for v, b in bound.items():
        g = float(exact_tree[e["start"][v]:e["end"][v]].min())
        k = int(blocks_per_node[v])
        if b > 0.0:
            worst = max(worst, b / (k * epsilon * g) if g > 0.0 else float("inf"))
        werr = max(werr, abs(wsum[v] - k * total_w) / (k * total_w))
    return {"worst_ratio": worst, "weight_error": werr, "query_nodes": len(bound)}
