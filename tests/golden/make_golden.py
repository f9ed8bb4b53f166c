"""Generate golden vectors by running the UNMODIFIED reference package.

Run in the build container (where /root/reference exists):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

It imports ``fastgauss`` from /root/reference/pkg/src, runs it on seeded
inputs and stores inputs + outputs as compressed .npz fixtures next to this
script.  The fixtures pin the CPU oracle (oracle/) and the B200 engine; no
test reads /root/reference at run time.
"""

import os
import sys

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", ".."))
import fastgauss as fg  # noqa: E402
from fastgauss import kernel_math as km  # noqa: E402
from fastgauss.cli_harness import max_rel_error  # noqa: E402

from paper_1206_6857_b200.configs import config  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))


def tree_arrays(t):
    nodes = t.nodes
    return dict(
        perm=t.perm.astype(np.int64),
        start=np.array([n.start for n in nodes], np.int64),
        end=np.array([n.end for n in nodes], np.int64),
        lo=np.array([n.lo for n in nodes]),
        hi=np.array([n.hi for n in nodes]),
        center=np.array([n.center for n in nodes]),
        weight=np.array([n.weight for n in nodes]),
        inf_radius=np.array([n.inf_radius for n in nodes]),
        left=np.array([-1 if n.left is None else n.left.index for n in nodes], np.int64),
        right=np.array([-1 if n.right is None else n.right.index for n in nodes], np.int64),
    )


def counters(res):
    c = res.counters
    return np.array([c.pair_visits, c.base_cases, c.fd_prunes, c.hermite_prunes,
                     c.local_prunes, c.h2l_prunes], np.int64)


def make_trees():
    out = {}
    cases = []
    rng = np.random.default_rng(7)
    cases.append(("uniform3", rng.random((3000, 3)), rng.uniform(0.5, 2.0, 3000), 25))
    cases.append(("dup", fg.PointStore(np.repeat(rng.random((40, 2)), 30, axis=0)).points,
                   None, 25))
    cases.append(("ident", np.tile([0.3, 0.7], (100, 1)), None, 25))
    cases.append(("small", rng.random((10, 3)), None, 25))
    cases.append(("leaf1", rng.random((200, 2)), None, 1))
    for i in (2, 3, 4, 5):
        wl = config(i, scale={2: 0.05, 3: 0.02, 4: 0.01, 5: 0.002}[i])
        cases.append((f"C{i}", wl.references, wl.weights, 25))
    for name, pts, w, leaf in cases:
        t = fg.build_tree(fg.PointStore(pts, w), leaf)
        arr = tree_arrays(t)
        arr["points"] = np.asarray(pts, dtype=float)
        arr["weights"] = t.weights[np.argsort(t.perm)]
        arr["leaf"] = np.int64(leaf)
        np.savez_compressed(os.path.join(HERE, f"tree_{name}.npz"), **arr)
        out[name] = len(t.nodes)
    return out


def make_moments():
    rng = np.random.default_rng(8)
    for D, n in [(2, 400), (3, 600), (5, 500)]:
        pts = rng.random((n, D))
        w = rng.uniform(0.5, 2.0, n)
        t = fg.build_tree(fg.PointStore(pts, w), 20)
        pl = fg.default_plimit(D)
        hs = [0.05, 0.3, 1.7]
        moms = []
        for h in hs:
            t.refresh_moments(h, pl)
            moms.append(np.array([nd.moments.coeffs for nd in t.nodes]))
        np.savez_compressed(os.path.join(HERE, f"moments_D{D}.npz"), points=pts, weights=w,
                            leaf=np.int64(20), plimit=np.int64(pl), bandwidths=np.array(hs),
                            moments=np.array(moms))


def make_runs():
    """End-to-end: naive + dfd/dfdo/dito on seeded small inputs."""
    rng = np.random.default_rng(9)
    cases = []
    for D, n, hs in [(1, 1500, [0.01, 0.3]), (2, 2500, [0.02, 0.1, 0.5, 2.0]),
                     (3, 2500, [0.03, 0.2, 0.6]), (5, 1500, [0.1, 0.5, 1.5]),
                     (7, 1200, [0.3, 1.0, 3.0])]:
        pts = rng.random((n, D))
        w = rng.uniform(0.5, 1.5, n)
        cases.append((f"mono_D{D}", pts, w, None, hs))
    # bichromatic with different M and N
    pts = rng.random((1800, 3))
    qs = rng.random((700, 3)) * 1.2 - 0.1
    cases.append(("bi_D3", pts, np.ones(1800), qs, [0.05, 0.4]))
    for name, pts, w, qs, hs in cases:
        store = fg.PointStore(pts, w)
        rt = fg.build_tree(store, 25)
        qt = rt if qs is None else fg.build_tree(fg.PointStore(qs), 25)
        qpts = pts if qs is None else qs
        rec = dict(points=pts, weights=w, queries=qpts, mono=np.int64(qs is None),
                   bandwidths=np.array(hs))
        for eps in (0.01, 0.001, 0.0):
            for alg in ("dfd", "dfdo", "dito"):
                vals, cnts = [], []
                for h in hs:
                    rt.refresh_moments(h, fg.default_plimit(pts.shape[1]))
                    res = getattr(fg, alg + "_run")(fg.RunConfig(bandwidth=h, epsilon=eps),
                                                   qt, rt)
                    vals.append(res.values)
                    cnts.append(counters(res))
                rec[f"{alg}_{eps}_values"] = np.array(vals)
                rec[f"{alg}_{eps}_counters"] = np.array(cnts)
        rec["naive"] = np.array([fg.naive_sum(qpts, pts, w, h).values for h in hs])
        np.savez_compressed(os.path.join(HERE, f"run_{name}.npz"), **rec)


def make_c1():
    """Config 1 in full: naive and dito at h=0.05, eps=0.01."""
    wl = config(1)
    rt = fg.build_tree(fg.PointStore(wl.references, wl.weights), 25)
    qt = fg.build_tree(fg.PointStore(wl.queries), 25)
    rt.refresh_moments(0.05, fg.default_plimit(2))
    naive = fg.naive_sum(wl.queries, wl.references, wl.weights, 0.05).values
    res = fg.dito_run(fg.RunConfig(bandwidth=0.05, epsilon=0.01), qt, rt)
    np.savez_compressed(os.path.join(HERE, "config1.npz"), naive=naive, dito=res.values,
                        dito_counters=counters(res),
                        dito_err=np.float64(max_rel_error(res.values, naive)))


def make_subsamples():
    """Configs 2-5 at reduced N: naive oracle sums on a seeded query subsample."""
    for i, scale, mq in [(2, 0.1, 400), (3, 0.05, 300), (4, 0.02, 200), (5, 0.005, 300)]:
        wl = config(i, scale=scale)
        rng = np.random.default_rng(2000 + i)
        idx = np.sort(rng.choice(wl.n, mq, replace=False))
        qs = wl.references[idx]
        naive = np.array([fg.naive_sum(qs, wl.references, wl.weights, h).values
                          for h in wl.bandwidths])
        np.savez_compressed(os.path.join(HERE, f"sub_C{i}.npz"), scale=np.float64(scale),
                            query_index=idx, bandwidths=np.array(wl.bandwidths), naive=naive,
                            epsilon=np.float64(wl.epsilon))


def make_series():
    rng = np.random.default_rng(10)
    rec = {}
    k = 0
    for D in (1, 2, 3, 5):
        for p in (1, 2, 4, 6):
            n = int(rng.integers(2, 20))
            h = float(rng.uniform(0.1, 1.5))
            pts = rng.random((n, D)) * 0.5
            w = rng.uniform(0.2, 2.0, n)
            c = pts.mean(axis=0)
            x = rng.random((7, D)) * 0.5 + float(rng.uniform(0, 2))
            c2 = c + rng.uniform(-0.3, 0.3, D)
            cq = x.mean(axis=0)
            far = fg.accumulate_far_field(pts, w, c, p, h)
            loc = fg.accumulate_local_direct(pts, w, cq, p, h)
            rec[f"c{k}_meta"] = np.array([D, p, h])
            rec[f"c{k}_pts"] = pts
            rec[f"c{k}_w"] = w
            rec[f"c{k}_x"] = x
            rec[f"c{k}_c"] = c
            rec[f"c{k}_c2"] = c2
            rec[f"c{k}_cq"] = cq
            rec[f"c{k}_far"] = far.coeffs
            rec[f"c{k}_evalm"] = np.atleast_1d(fg.eval_far_field(far, x))
            rec[f"c{k}_loc"] = loc.coeffs
            rec[f"c{k}_evall"] = np.atleast_1d(fg.eval_local(loc, x))
            rec[f"c{k}_h2h"] = fg.translate_h2h(far, c2).coeffs
            rec[f"c{k}_h2l"] = fg.translate_h2l(far, cq, p).coeffs
            rec[f"c{k}_l2l"] = fg.translate_l2l(loc, c2).coeffs
            rec[f"c{k}_ladder"] = km.hermite_ladder(x[:, 0], 2 * p)
            k += 1
    rec["count"] = np.int64(k)
    np.savez_compressed(os.path.join(HERE, "series.npz"), **rec)


def make_bounds():
    rng = np.random.default_rng(11)
    rows = []
    codes = {fg.Method.EXHAUSTIVE: 0, fg.Method.HERMITE: 2, fg.Method.LOCAL: 3,
             fg.Method.H2L: 4}
    for _ in range(400):
        D = int(rng.integers(1, 8))
        pl = int(rng.integers(1, 9))
        h = float(rng.uniform(0.05, 2.0))
        geom = fg.NodePairGeometry(
            min_sqdist=float(rng.uniform(0, 4)) * h * h,
            max_sqdist=float(rng.uniform(4, 20)) * h * h,
            r_ref=float(rng.uniform(0, 1.5)), r_query=float(rng.uniform(0, 1.5)),
            weight_ref=float(rng.uniform(0.1, 50)), n_query=int(rng.integers(1, 200)),
            n_ref=int(rng.integers(1, 200)), dim=D, bandwidth=h)
        maxerr = float(10 ** rng.uniform(-6, 1))
        ch = fg.best_method(geom, maxerr, pl)
        rows.append([geom.min_sqdist, geom.max_sqdist, geom.r_ref, geom.r_query,
                     geom.weight_ref, geom.n_query, geom.n_ref, D, h, maxerr, pl,
                     codes[ch.method], ch.order or 0, ch.bound, ch.cost])
    floor = []
    for D in range(1, 9):
        for pl in range(1, 9):
            floor.append([D, pl, fg.error_bounds.series_floor_constant(D, pl)])
    np.savez_compressed(os.path.join(HERE, "bounds.npz"), rows=np.array(rows),
                        floor=np.array(floor))


def make_lscv():
    """LSCV selection (cli_harness.py:101-157) and exact scores on seeded data."""
    from fastgauss.cli_harness import select_bandwidth

    rng = np.random.default_rng(12)
    rec = {}
    for D, n in ((2, 1500), (3, 1200)):
        means = rng.uniform(0, 1, (3, D))
        pts = means[rng.integers(0, 3, n)] + 0.08 * rng.standard_normal((n, D))
        h_sel = select_bandwidth(pts, seed=0)
        hs = np.geomspace(0.01, 0.3, 5)
        exact = []
        for h in hs:
            conv = fg.naive_sum(pts, pts, np.ones(n), np.sqrt(2.0) * h).values
            near = fg.naive_sum(pts, pts, np.ones(n), h).values
            nc = (2 * np.pi * 2 * h * h) ** (-0.5 * D)
            nn = (2 * np.pi * h * h) ** (-0.5 * D)
            exact.append([nc * conv.sum() / n ** 2, 2 * nn * (near.sum() - n) / (n * (n - 1))])
        rec[f"D{D}_points"] = pts
        rec[f"D{D}_h_select"] = np.float64(h_sel)
        rec[f"D{D}_hs"] = hs
        rec[f"D{D}_terms"] = np.array(exact)
    np.savez_compressed(os.path.join(HERE, "lscv.npz"), **rec)


def make_cli():
    """Report formats, CSV ingestion and the dataset generators of the reference's
    cli_harness.py / datasets.py, rendered by the reference itself."""
    import json
    import tempfile

    from fastgauss import cli_harness as ch
    from fastgauss import datasets as ds

    rec = {"reports": [], "loads": [], "datasets": {}}
    rows = [("naive", 0.5, 0.05, 0.12345, 0.0, {}),
            ("dfd", 0.5, 0.05, 0.0123456, 0.00123, {"pair_visits": 10, "base_cases": 3,
                                                    "fd_prunes": 4, "hermite_prunes": 0,
                                                    "local_prunes": 0, "h2l_prunes": 0}),
            ("naive", 1.0, 0.1, 0.2, 0.0, {}),
            ("dfd", 1.0, 0.1, 1.5e-4, 2.5e-7, {"pair_visits": 7, "base_cases": 1,
                                               "fd_prunes": 5, "hermite_prunes": 2,
                                               "local_prunes": 1, "h2l_prunes": 0})]
    for verified in (True, False):
        rrows = [ch.SweepRow(a, m, h, s, (e if verified else None), c) for a, m, h, s, e, c in rows]
        totals = {"naive": 0.32345, "dfd": 0.0124956}
        rep = ch.SweepReport(0.1, 0.01, "ref.csv", None, (0.5, 1.0), ("naive", "dfd"), rrows,
                             totals, verified)
        rec["reports"].append({
            "verified": verified,
            "rows": [[a, m, h, s, (e if verified else None), c] for a, m, h, s, e, c in rows],
            "totals": totals,
            "table": ch._format_table(rep), "csv": ch._format_csv(rep),
            "json": json.dumps(ch.report_to_dict(rep), indent=2) + "\n"})
    cases = {
        "plain": ("0.1,0.2\n0.3,0.4\n\n0.5,0.6\n", {}),
        "header": ("x,y\n1,2\n3,4\n", {"header": True}),
        "weights": ("0,0,2\n1,1,0.5\n", {"has_weights": True}),
        "rescale": ("1,5,2\n3,5,4\n2,5,8\n", {"rescale": True}),
        "ragged": ("1,2\n3\n", {}),
        "nonnumeric": ("1,2\n3,abc\n", {}),
        "empty": ("\n\n", {}),
        "bad_weights": ("0,0,-1\n1,1,1\n", {"has_weights": True}),
        "weights_one_col": ("1\n2\n", {"has_weights": True}),
    }
    with tempfile.TemporaryDirectory() as td:
        for name, (text, kw) in cases.items():
            path = os.path.join(td, "data.csv")
            with open(path, "w") as fh:
                fh.write(text)
            entry = {"name": name, "text": text, "kw": kw}
            try:
                st = ch.load_points(path, **kw)
                entry["points"] = st.points.tolist()
                entry["weights"] = st.weights.tolist()
            except ch.LoadError as exc:
                entry["error"] = str(exc).replace(path, "<path>")
            rec["loads"].append(entry)
    rec["datasets"] = {
        "uniform": ds.uniform_points(5, 3, 7).tolist(),
        "clustered": ds.clustered_points(6, 2, 3).tolist(),
        "hierarchical": ds.hierarchical_clusters(6, 2, 4).tolist(),
        "duplicated": ds.duplicated_points(10, 2, 5).tolist(),
    }
    with open(os.path.join(HERE, "cli.json"), "w") as fh:
        json.dump(rec, fh, indent=1)


if __name__ == "__main__":
    which = sys.argv[1:] or ["trees", "moments", "series", "bounds", "runs", "subsamples",
                             "c1", "lscv", "cli"]
    if "cli" in which:
        make_cli()
    if "trees" in which:
        print("trees", make_trees())
    if "moments" in which:
        make_moments()
    if "series" in which:
        make_series()
    if "bounds" in which:
        make_bounds()
    if "runs" in which:
        make_runs()
    if "subsamples" in which:
        make_subsamples()
    if "c1" in which:
        make_c1()
    if "lscv" in which:
        make_lscv()
    print("done")
