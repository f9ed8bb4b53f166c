"""Series orders above the reference's default cap (default_plimit(3) = 6).

The engine evaluates Hermite far fields at D = 3 up to order 12 (its own cap,
fg_engine_plimit; RunConfig.plimit is honoured as given, error_bounds.py:107-117
holds for every order).  The series operators are checked against the oracle at
those orders, and whole runs against exhaustive summation (<= eps) and against
the reference's depth-first DITO run at the SAME order cap (<= 2 eps, oracle
port, counters pinned to the reference).
"""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def fg():
    import paper_1206_6857_b200 as fg

    return fg


def clustered(seed, n):
    rng = np.random.default_rng(seed)
    centres = rng.random((12, 3))
    k = rng.integers(0, 12, n)
    pts = centres[k] + rng.normal(0.0, 0.04, (n, 3))
    pts[: n // 10] = rng.random((n // 10, 3))
    return pts, rng.uniform(0.5, 1.5, n)


def test_engine_order_cap(fg):
    assert fg.engine_plimit(3) == 12
    for d in (1, 2, 4, 5, 6, 7, 9, 16):
        assert fg.engine_plimit(d) == fg.default_plimit(d)


@pytest.mark.parametrize("order", [7, 9, 10, 11, 12])
def test_series_operators_at_high_order(fg, oracle, order):
    rng = np.random.default_rng(order)
    h = 0.3
    pts = 0.5 + 0.08 * rng.standard_normal((300, 3))
    w = rng.uniform(0.5, 1.5, 300)
    c = pts.mean(0)
    x = 0.5 + 0.6 * rng.standard_normal((200, 3))
    far = fg.accumulate_far_field(pts, w, c, order, h)
    ref = oracle.accumulate_far_field(pts, w, c, order, h)
    np.testing.assert_allclose(far.coeffs, ref, rtol=1e-11, atol=1e-14)
    np.testing.assert_allclose(fg.eval_far_field(far, x), oracle.eval_far_field(ref, c, order, h, x),
                               rtol=1e-10, atol=1e-14)
    cq = c + 0.05
    loc = fg.accumulate_local_direct(pts, w, cq, order, h)
    np.testing.assert_allclose(loc.coeffs, oracle.accumulate_local_direct(pts, w, cq, order, h),
                               rtol=1e-11, atol=1e-14)


@pytest.mark.parametrize("plimit", [7, 8, 10, 11, 12])
@pytest.mark.parametrize("eps", [1e-2, 1e-4])
def test_runs_at_high_order_within_eps(fg, oracle, plimit, eps):
    pts, w = clustered(40 + plimit, 6000)
    tree = fg.build_tree(fg.PointStore(pts, w), 25)
    ref_tree = oracle.Tree(pts, w, 25)
    used = 0
    for h in (0.05, 0.15, 0.4):
        exact = oracle.naive_sum(pts, pts, w, h, threads=0)
        tree.refresh_moments(h, plimit)
        res = fg.dito_run(fg.RunConfig(bandwidth=h, epsilon=eps, plimit=plimit), tree, tree)
        assert oracle.max_rel_error(res.values, exact) <= eps
        used += res.counters.hermite_prunes
        # the reference's own DITO at the same order cap (depth-first, oracle port)
        ref_tree.refresh_moments(h, plimit)
        ref_vals, _ = oracle.run("dito", ref_tree, ref_tree, h, eps, plimit=plimit)
        assert oracle.max_rel_error(res.values, ref_vals) <= 2 * eps
    assert used > 0


def test_far_field_only_run_is_accurate(fg, oracle):
    """At a bandwidth far above the data's extent every reference node is settled
    by a Hermite expansion; the truncation bounds are far below eps there, so
    the row machine's sums must agree with exhaustive summation to ~1e-9."""
    pts, w = clustered(7, 20000)
    tree = fg.build_tree(fg.PointStore(pts, w), 25)
    for h in (2.0, 5.0):
        res = fg.sweep_run(fg.RunConfig(bandwidth=h, epsilon=1e-3), tree, tree, [h])[0]
        assert res.counters.hermite_prunes > 0 and res.counters.base_cases == 0
        exact = fg.naive_sum(pts, pts, w, h).values
        assert oracle.max_rel_error(res.values, exact) <= 1e-7


def test_tight_eps_uses_the_high_orders(fg, oracle):
    """eps = 1e-6 at moderate bandwidths: only high orders are admissible for
    nodes of useful size; the sweep (engine order cap) stays within eps."""
    pts, w = clustered(11, 12000)
    tree = fg.build_tree(fg.PointStore(pts, w), 25)
    hs = [0.1, 0.25, 0.6]
    res = fg.sweep_run(fg.RunConfig(bandwidth=hs[0], epsilon=1e-6), tree, tree, hs)
    low = fg.sweep_run(fg.RunConfig(bandwidth=hs[0], epsilon=1e-6, plimit=6), tree, tree, hs)
    for h, r, r6 in zip(hs, res, low):
        exact = oracle.naive_sum(pts, pts, w, h, threads=0)
        assert oracle.max_rel_error(r.values, exact) <= 1e-6
        assert oracle.max_rel_error(r6.values, exact) <= 1e-6
        # the higher cap never evaluates more pairs exactly
        assert (r.counters.exact_pairs + r.counters.fp32_pairs
                <= r6.counters.exact_pairs + r6.counters.fp32_pairs)


@pytest.mark.parametrize("plimit", [6, 12])
def test_moments_by_h2h_match_the_oracle(fg, oracle, plimit):
    """Nodes of more than 256 points take their moments from their children
    (H2H level pass), smaller ones and large LEAVES (identical points) from
    their points: every node's moments against the oracle's (leaf moments +
    H2H, spatial_index.py:171-197), in preorder like the reference."""
    rng = np.random.default_rng(3)
    pts = np.concatenate([rng.random((6000, 3)), np.tile([[0.31, 0.62, 0.17]], (700, 1)),
                          0.8 + 0.01 * rng.standard_normal((3000, 3))])
    w = rng.uniform(0.5, 1.5, len(pts))
    tree = fg.build_tree(fg.PointStore(pts, w), 25)
    ref = oracle.Tree(pts, w, 25)
    for h in (0.07, 0.4):
        tree.refresh_moments(h, plimit)
        ref.refresh_moments(h, plimit)
        m, r = tree.moments_array(), ref.moments()
        assert m.shape == r.shape
        scale = np.abs(r).max(axis=1, keepdims=True) + 1e-300
        assert np.max(np.abs(m - r) / scale) <= 1e-10
