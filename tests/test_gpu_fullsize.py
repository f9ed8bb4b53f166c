"""Full-size parity at BASELINE.json's sizes.

* The exhaustive kernel (K1) at FULL N for configs 2-5, every bandwidth, on a
  seeded 1024-query subsample, against the oracle's naive_sum fixture
  (tests/golden/make_fullsize.py): <= 1e-12 relative per query.
* The DITO sweep over ALL M queries of configs 2-4 (and a seeded 2^16-query
  sample of C5) within the config's eps of the exhaustive kernel at every
  bandwidth (the kernel being pinned by the first test).
* The DITO sweep on the BASELINE.md section 3 subsample within 2 eps of the
  reference's own depth-first DITO (oracle port, fixture) -- both are
  eps-approximations with different traversal orders.
"""

import os

import numpy as np
import pytest

from conftest import golden

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def fg():
    import paper_1206_6857_b200 as fg

    return fg


def rel(a, b):
    a = np.asarray(a, float)
    b = np.asarray(b, float)
    return float(np.max(np.abs(a - b) / np.abs(b))) if a.size else 0.0


_SWEEPS = {}


def _sweep(fg, index):
    """The whole DITO sweep of config `index` at full size (cached per module)."""
    if index not in _SWEEPS:
        from paper_1206_6857_b200.configs import config

        wl = config(index)
        rt = fg.build_tree(fg.PointStore(wl.references, wl.weights), 25)
        hs = list(wl.bandwidths)
        res = fg.sweep_run(fg.RunConfig(bandwidth=hs[0], epsilon=wl.epsilon), rt, rt, hs)
        _SWEEPS.clear()  # keep one config's values resident at a time
        _SWEEPS[index] = (wl, np.stack([r.values for r in res]), res)
    return _SWEEPS[index]


@pytest.mark.parametrize("index", [2, 3, 4, 5])
def test_naive_full_n_matches_oracle(fg, index):
    """K1 over all N references at every bandwidth vs the oracle (1e-12)."""
    from paper_1206_6857_b200.configs import config

    g = golden(f"full_C{index}.npz")
    wl = config(index)
    np.testing.assert_array_equal(g["hs"], np.array(wl.bandwidths))
    got = fg.naive_sum(wl.query_points()[g["idx"]], wl.references, wl.weights,
                       list(g["hs"])).values
    assert got.shape == g["naive"].shape
    assert rel(got, g["naive"]) <= 1e-12


@pytest.mark.parametrize("index", [2, 3, 4, 5])
def test_dito_sweep_all_queries_within_eps(fg, index):
    """Every query of the full-size sweep within eps of the exhaustive sums
    (C5: a seeded 2^16-query sample; its exhaustive leg alone is 2.6e14 pairs
    over all M)."""
    wl, vals, _ = _sweep(fg, index)
    if index == 5:
        sel = np.sort(np.random.default_rng(65536).choice(wl.m, 1 << 16, replace=False))
    else:
        sel = np.arange(wl.m)
    qp = wl.query_points()[sel]
    for j, h in enumerate(wl.bandwidths):
        exact = fg.naive_sum(qp, wl.references, wl.weights, h).values
        v = vals[j][sel]
        assert np.all(np.isfinite(v)) and np.all(v > 0.0)
        assert rel(v, exact) <= wl.epsilon, (index, j, h)


@pytest.mark.parametrize("index", [2, 3, 4, 5])
def test_dito_sweep_within_2eps_of_reference_dito(fg, index):
    """GPU DITO vs the reference's DFS DITO (oracle port, fixture) on the
    section-3 subsample: <= 2 eps; the fixture itself is <= eps of naive."""
    g = golden(f"full_C{index}.npz")
    wl, vals, _ = _sweep(fg, index)
    eps = float(g["epsilon"])
    assert eps == wl.epsilon
    assert rel(g["dito"], g["naive"]) <= eps
    got = vals[:, g["idx"]]
    assert rel(got, g["naive"]) <= eps
    assert rel(got, g["dito"]) <= 2 * eps


def test_query_block_partition_matches_host_rule(fg):
    """fg_query_block_ranges == distributed.query_block_ranges (the host
    restatement the multi-rank CPU tests use) on assorted trees."""
    from paper_1206_6857_b200 import distributed as D
    from paper_1206_6857_b200.configs import config
    from paper_1206_6857_b200.summation_engine import query_block_ranges

    rng = np.random.default_rng(11)
    cases = [(rng.random((1, 3)), 25), (rng.random((50, 2)), 25), (rng.random((5000, 3)), 10),
             (np.repeat(rng.random((30, 2)), 90, axis=0), 25), (rng.random((3000, 5)), 1),
             (config(2).references, 25)]
    for pts, leaf in cases:
        t = fg.build_tree(fg.PointStore(pts), leaf)
        e = t.arrays()
        host = D.query_block_ranges(e["start"], e["end"], e["left"], e["right"])
        s, c = query_block_ranges(t)
        assert list(zip(s.tolist(), c.tolist())) == host


def test_two_threads_own_trees_bit_exact(fg):
    """concurrent traversals on distinct query trees from two host
    threads (each on its own engine stream: the per-thread default stream,
    then a private torch stream) reproduce the serial results bit for bit."""
    import threading

    import torch

    rng = np.random.default_rng(21)
    data = [(rng.random((20000, 3)), rng.uniform(0.5, 1.5, 20000)),
            (rng.normal(size=(15000, 3)), None)]
    hs = [[0.01, 0.05, 0.2], [0.1, 0.3, 1.0]]

    def work(k, use_torch_stream):
        pts, w = data[k]
        tree = fg.build_tree(fg.PointStore(pts, w), 25)
        cfg = fg.RunConfig(bandwidth=hs[k][0], epsilon=0.01)
        out = []
        for _ in range(3):
            if use_torch_stream:
                s = torch.cuda.Stream()
                with torch.cuda.stream(s):
                    dev = torch.zeros((3, tree.n), dtype=torch.float64, device="cuda")
                    fg.sweep_run(cfg, tree, tree, hs[k], out=dev)
                    s.synchronize()
                    out.append(dev.cpu().numpy())
            else:
                out.append(np.stack([r.values for r in fg.sweep_run(cfg, tree, tree, hs[k])]))
            tree.refresh_moments(hs[k][1], fg.default_plimit(3))
            out.append(fg.dito_run(fg.RunConfig(bandwidth=hs[k][1], epsilon=0.01),
                                   tree, tree).values)
        return out

    serial = [work(0, False), work(1, False)]
    for use_ts in (False, True):
        got = [None, None]
        errs = []

        def run(k):
            try:
                got[k] = work(k, use_ts)
            except Exception as e:  # surfaced below
                errs.append(e)

        ths = [threading.Thread(target=run, args=(k,)) for k in (0, 1)]
        for t in ths:
            t.start()
        for t in ths:
            t.join()
        assert not errs, errs
        for k in (0, 1):
            for a, b in zip(got[k], serial[k]):
                np.testing.assert_array_equal(a, b)


def test_counters_parity_and_token_dominance(fg, oracle):
    """(f)3 and SPEC.md:571 (criterion 4) on paired runs (same tree, DFD vs DFDO):
    the token scheme settles more by pruning, so DFDO needs no more node-pair
    visits, base cases or exactly evaluated pairs than DFD -- for the engine
    and for the reference DFS (oracle) alike.  The literal "DFDO prune count
    >= DFD" does NOT hold for the reference DFS either (one coarse DFDO prune
    replaces many fine DFD prunes): profiles/r02_counters.jsonl has 17 of 54
    (config, bandwidth) rows where the reference DFS prunes fewer times under
    DFDO, while visits and base cases dominate in all 54."""
    rng = np.random.default_rng(31)
    for D in (3, 7):
        pts = rng.normal(size=(20000, D)) * rng.uniform(0.5, 2.0, D)
        tree = fg.build_tree(fg.PointStore(pts), 25)
        otree = oracle.Tree(pts, None, 25)
        for h in (0.05, 0.2, 0.6):
            c, o = {}, {}
            for alg in ("dfd", "dfdo"):
                r = getattr(fg, f"{alg}_run")(fg.RunConfig(bandwidth=h, epsilon=0.01),
                                              tree, tree)
                c[alg] = r.counters
                _, o[alg] = oracle.run(alg, otree, otree, h, 0.01)
            assert c["dfdo"].pair_visits <= c["dfd"].pair_visits, (D, h)
            assert c["dfdo"].base_cases <= c["dfd"].base_cases, (D, h)
            assert (c["dfdo"].exact_pairs + c["dfdo"].fp32_pairs <=
                    c["dfd"].exact_pairs + c["dfd"].fp32_pairs), (D, h)
            assert o["dfdo"][0] <= o["dfd"][0] and o["dfdo"][1] <= o["dfd"][1], (D, h)
            for alg in ("dfd", "dfdo"):
                k = c[alg]
                assert k.exact_pairs + k.fp32_pairs <= 20000 * 20000
                assert k.pair_visits >= k.fd_prunes + k.base_cases
