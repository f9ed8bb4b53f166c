"""Pin the CPU oracle (oracle/) before trusting it as the parity checker.

Two kinds of pins:
* golden vectors produced by the unmodified reference (tests/golden/*.npz,
  made by tests/golden/make_golden.py);
* the reference's own known-answer tests (tests/test_kernel_math.py,
  tests/test_spatial_index.py, tests/test_error_bounds.py in
  /root/reference/pkg/tests), restated here.
"""

import math

import numpy as np
import pytest

from conftest import golden


def rel(a, b):
    a = np.asarray(a, float)
    b = np.asarray(b, float)
    scale = np.maximum(np.abs(b), 1e-300)
    return float(np.max(np.abs(a - b) / scale)) if a.size else 0.0


# ------------------------------------------------------- known answers
def test_kernel_known_answers(oracle):
    # tests/test_kernel_math.py:66-72: K(0)=1, K(2h^2)=e^-1
    out = oracle.naive_sum(np.zeros((1, 1)), np.zeros((1, 1)), np.ones(1), 0.7)
    assert out[0] == 1.0
    h = 0.7
    out = oracle.naive_sum(np.array([[math.sqrt(2.0) * h]]), np.zeros((1, 1)), np.ones(1), h)
    assert abs(out[0] - 0.36787944117144233) <= 1e-14


def test_multi_index_enumeration(oracle):
    # tests/test_kernel_math.py:21-26 known answers and C(D+p-1, D) counts
    d, _, _, _ = oracle.iset(2, 2)
    assert d.tolist() == [[0, 0], [1, 0], [0, 1]]
    d, deg, fact, _ = oracle.iset(3, 3)
    assert d[:4].tolist() == [[0, 0, 0], [1, 0, 0], [0, 1, 0], [0, 0, 1]]
    assert d[4:7].tolist() == [[2, 0, 0], [1, 1, 0], [1, 0, 1]]
    for D in (1, 2, 3, 5):
        for p in (1, 2, 4, 8):
            dg, deg, fact, pairs = oracle.iset(D, p)
            assert dg.shape[0] == math.comb(D + p - 1, D)
            assert np.all(np.diff(deg) >= 0)
            np.testing.assert_array_equal(
                fact, [np.prod([math.factorial(int(x)) for x in row]) for row in dg])
            # shift pairs: digits_a + digits_b == digits_s, degree < order
            s = pairs
            np.testing.assert_array_equal(dg[s[:, 0]] + dg[s[:, 1]], dg[s[:, 2]])


def test_hermite_ladder_vs_numpy_hermval(oracle):
    # tests/test_kernel_math.py:158-171
    t = np.linspace(-3, 3, 41)
    lad = oracle.hermite_ladder(t, 8)
    for n in range(9):
        c = np.zeros(n + 1)
        c[n] = 1.0
        ref = np.polynomial.hermite.hermval(t, c) * np.exp(-t * t)
        np.testing.assert_allclose(lad[:, n], ref, rtol=1e-10, atol=1e-12)


def test_power_table(oracle):
    u = np.array([0.5, -2.0, 3.0])
    tab = oracle.power_table(u, 4)
    np.testing.assert_array_equal(tab, u[:, None] ** np.arange(5))


def test_plimit_floor_and_tail_tables(oracle):
    g = golden("bounds.npz")
    for D, pl, val in g["floor"]:
        assert oracle.series_floor_constant(int(D), int(pl)) == pytest.approx(val, rel=1e-15)


def test_best_method_golden(oracle):
    g = golden("bounds.npz")
    names = {0: "exhaustive", 2: "hermite", 3: "local", 4: "h2l"}
    for row in g["rows"]:
        (mn, mx, rr, rq, wr, nq, nr, D, h, maxerr, pl, code, order, bound, cost) = row
        m, p, b, c = oracle.best_method(mn, mx, rr, rq, wr, int(nq), int(nr), int(D), h,
                                        maxerr, int(pl))
        assert m == names[int(code)]
        assert (p or 0) == int(order)
        assert b == pytest.approx(bound, rel=1e-12, abs=1e-300)
        assert c == pytest.approx(cost, rel=1e-12)


def test_series_golden(oracle):
    g = golden("series.npz")
    for k in range(int(g["count"])):
        D, p, h = g[f"c{k}_meta"]
        D, p = int(D), int(p)
        pts, w, x = g[f"c{k}_pts"], g[f"c{k}_w"], g[f"c{k}_x"]
        c, c2, cq = g[f"c{k}_c"], g[f"c{k}_c2"], g[f"c{k}_cq"]
        far = oracle.accumulate_far_field(pts, w, c, p, h)
        assert rel(far, g[f"c{k}_far"]) <= 1e-12 or np.allclose(far, g[f"c{k}_far"],
                                                                 rtol=1e-12, atol=1e-15)
        np.testing.assert_allclose(oracle.eval_far_field(far, c, p, h, x), g[f"c{k}_evalm"],
                                   rtol=1e-12, atol=1e-15)
        loc = oracle.accumulate_local_direct(pts, w, cq, p, h)
        np.testing.assert_allclose(loc, g[f"c{k}_loc"], rtol=1e-12, atol=1e-15)
        np.testing.assert_allclose(oracle.eval_local(loc, cq, p, h, x), g[f"c{k}_evall"],
                                   rtol=1e-12, atol=1e-15)
        np.testing.assert_allclose(oracle.translate_h2h(far, c, c2, p, h), g[f"c{k}_h2h"],
                                   rtol=1e-12, atol=1e-15)
        np.testing.assert_allclose(oracle.translate_h2l(far, c, cq, p, p, h), g[f"c{k}_h2l"],
                                   rtol=1e-12, atol=1e-15)
        np.testing.assert_allclose(oracle.translate_l2l(loc, cq, c2, p, h), g[f"c{k}_l2l"],
                                   rtol=1e-12, atol=1e-15)
        np.testing.assert_allclose(oracle.hermite_ladder(x[:, 0], 2 * p), g[f"c{k}_ladder"],
                                   rtol=1e-13, atol=1e-15)


@pytest.mark.parametrize("name", ["uniform3", "dup", "ident", "small", "leaf1",
                                  "C2", "C3", "C4", "C5"])
def test_tree_golden(oracle, name):
    g = golden(f"tree_{name}.npz")
    t = oracle.Tree(g["points"], g["weights"], int(g["leaf"]))
    ex = t.export()
    for key in ("perm", "start", "end", "left", "right"):
        np.testing.assert_array_equal(ex[key], g[key])
    np.testing.assert_array_equal(ex["lo"], g["lo"])
    np.testing.assert_array_equal(ex["hi"], g["hi"])
    np.testing.assert_allclose(ex["center"], g["center"], rtol=1e-13, atol=1e-15)
    np.testing.assert_allclose(ex["inf_radius"], g["inf_radius"], rtol=1e-12, atol=1e-15)
    np.testing.assert_allclose(ex["weight"], g["weight"], rtol=1e-12)


@pytest.mark.parametrize("D", [2, 3, 5])
def test_moments_golden(oracle, D):
    g = golden(f"moments_D{D}.npz")
    t = oracle.Tree(g["points"], g["weights"], int(g["leaf"]))
    for h, ref in zip(g["bandwidths"], g["moments"]):
        t.refresh_moments(h, int(g["plimit"]))
        m = t.moments()
        scale = np.abs(ref).max(axis=1, keepdims=True) + 1e-30
        assert np.max(np.abs(m - ref) / scale) <= 1e-12


@pytest.mark.parametrize("name", ["mono_D1", "mono_D2", "mono_D3", "mono_D5", "mono_D7",
                                  "bi_D3"])
def test_runs_golden(oracle, name):
    """The oracle's depth-first dfd/dfdo/dito reproduce the reference's decisions
    (identical counters) and values to rounding."""
    g = golden(f"run_{name}.npz")
    pts, w, qs = g["points"], g["weights"], g["queries"]
    rt = oracle.Tree(pts, w, 25)
    qt = rt if int(g["mono"]) else oracle.Tree(qs, None, 25)
    D = pts.shape[1]
    pl = {1: 8, 2: 8, 3: 6, 4: 4, 5: 4, 6: 2}.get(D, 1)
    for j, h in enumerate(g["bandwidths"]):
        naive = oracle.naive_sum(qs, pts, w, h)
        assert rel(naive, g["naive"][j]) <= 1e-13
        rt.refresh_moments(h, pl)
        for eps in (0.01, 0.001, 0.0):
            for alg in ("dfd", "dfdo", "dito"):
                vals, cnt = oracle.run(alg, qt, rt, h, eps)
                np.testing.assert_array_equal(cnt, g[f"{alg}_{eps}_counters"][j])
                assert rel(vals, g[f"{alg}_{eps}_values"][j]) <= 1e-12
                assert oracle.max_rel_error(vals, naive) <= max(eps, 1e-12)


def test_config1_golden(oracle):
    from paper_1206_6857_b200.configs import config

    g = golden("config1.npz")
    wl = config(1)
    rt = oracle.Tree(wl.references, wl.weights, 25)
    qt = oracle.Tree(wl.queries, None, 25)
    rt.refresh_moments(0.05, 8)
    vals, cnt = oracle.run("dito", qt, rt, 0.05, 0.01)
    np.testing.assert_array_equal(cnt, g["dito_counters"])
    assert rel(vals, g["dito"]) <= 1e-12
    sub = slice(0, 500)
    naive = oracle.naive_sum(wl.queries[sub], wl.references, wl.weights, 0.05)
    assert rel(naive, g["naive"][sub]) <= 1e-13


def test_lscv_exact_terms(oracle):
    g = golden("lscv.npz")
    for D in (2, 3):
        pts = g[f"D{D}_points"]
        n = pts.shape[0]
        for h, (t1, t2) in zip(g[f"D{D}_hs"], g[f"D{D}_terms"]):
            conv = oracle.naive_sum(pts, pts, np.ones(n), np.sqrt(2.0) * h, threads=0)
            near = oracle.naive_sum(pts, pts, np.ones(n), h, threads=0)
            nc = (2 * np.pi * 2 * h * h) ** (-0.5 * D)
            nn = (2 * np.pi * h * h) ** (-0.5 * D)
            assert nc * conv.sum() / n ** 2 == pytest.approx(t1, rel=1e-12)
            assert 2 * nn * (near.sum() - n) / (n * (n - 1)) == pytest.approx(t2, rel=1e-12)
