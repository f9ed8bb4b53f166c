"""Per-bandwidth report of the engine on a config: time, counters, exact-pair
share, and max relative error vs the GPU exhaustive kernel on a query subsample.

  python tools/sweep_report.py --config 2 [--scale 1.0] [--algo dito] [--ref-leaf 32]
"""
import argparse
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--scale", type=float, default=1.0)
    ap.add_argument("--algo", default="dito")
    ap.add_argument("--ref-leaf", type=int, default=0)
    ap.add_argument("--sub", type=int, default=2000)
    ap.add_argument("--plimit", type=int, default=0, help="series order cap (default: default_plimit(D))")
    ap.add_argument("--hmin", type=float, default=0.0, help="skip bandwidths below this")
    ap.add_argument("--naive", action="store_true", help="also time the full exhaustive kernel")
    ap.add_argument("--sweep", action="store_true",
                    help="one sweep_run over all bandwidths (after a warm-up sweep)")
    args = ap.parse_args()
    import paper_1206_6857_b200 as fg
    from paper_1206_6857_b200 import _lib
    from paper_1206_6857_b200.configs import config
    import oracle

    if args.ref_leaf:
        _lib.call("fg_set_engine_params", args.ref_leaf, 0, -1)
    wl = config(args.config, scale=args.scale)
    qp = wl.query_points()
    t0 = time.perf_counter()
    rt = fg.build_tree(fg.PointStore(wl.references, wl.weights), 25)
    qt = rt if wl.monochromatic else fg.build_tree(fg.PointStore(wl.queries), 25)
    t_build = time.perf_counter() - t0
    rng = np.random.default_rng(0)
    idx = np.sort(rng.choice(wl.m, min(args.sub, wl.m), replace=False))
    pl = args.plimit or fg.default_plimit(wl.dim)
    print(f"{wl.name} N={wl.n} D={wl.dim} build {t_build*1e3:.1f} ms nodes={rt.node_count} "
          f"levels={rt.levels}")
    if args.sweep:
        cfg = fg.RunConfig(bandwidth=wl.bandwidths[0], epsilon=wl.epsilon, algorithm=args.algo)
        fg.sweep_run(cfg, qt, rt, wl.bandwidths)
        t0 = time.perf_counter()
        results = fg.sweep_run(cfg, qt, rt, wl.bandwidths)
        wall = time.perf_counter() - t0
        for h, res in zip(wl.bandwidths, results):
            exact = fg.naive_sum(qp[idx], wl.references, wl.weights, h).values
            c = res.counters
            print(json.dumps(dict(h=round(h, 6), kern_ms=round(res.seconds * 1e3, 3),
                                  err=float(f"{oracle.max_rel_error(res.values[idx], exact):.3e}"),
                                  exact_share=float(f"{c.exact_pairs / (wl.m * wl.n):.4f}"),
                                  fp32_share=float(f"{c.fp32_pairs / (wl.m * wl.n):.4f}"),
                                  visits=c.pair_visits, dh=c.hermite_prunes)), flush=True)
        tot = sum(r.seconds for r in results)
        print(f"sweep kernel ms {tot*1e3:.2f}, wall ms {wall*1e3:.2f}; effective pairs/s "
              f"{wl.m * wl.n * len(wl.bandwidths) / wall:.3e}")
        return
    tot = 0.0
    for h in wl.bandwidths:
        if h < args.hmin:
            continue
        t0 = time.perf_counter()
        rt.refresh_moments(h, pl)
        t_ref = time.perf_counter() - t0
        run = {"dfd": fg.dfd_run, "dfdo": fg.dfdo_run, "dito": fg.dito_run}[args.algo]
        t0 = time.perf_counter()
        res = run(fg.RunConfig(bandwidth=h, epsilon=wl.epsilon, plimit=pl), qt, rt)
        t_run = time.perf_counter() - t0
        exact = fg.naive_sum(qp[idx], wl.references, wl.weights, h).values
        err = oracle.max_rel_error(res.values[idx], exact)
        c = res.counters
        share = c.exact_pairs / (wl.m * wl.n)
        tot += res.seconds
        line = dict(h=round(h, 6), kern_ms=round(res.seconds * 1e3, 3),
                    wall_ms=round(t_run * 1e3, 2), refresh_ms=round(t_ref * 1e3, 2),
                    err=float(f"{err:.3e}"), exact_share=float(f"{share:.4f}"),
                    fp32_share=float(f"{c.fp32_pairs / (wl.m * wl.n):.4f}"),
                    visits=c.pair_visits, base=c.base_cases, fd=c.fd_prunes,
                    dh=c.hermite_prunes, dl=c.local_prunes, h2l=c.h2l_prunes,
                    pair_rate=float(f"{c.exact_pairs / max(res.seconds, 1e-9):.3e}"))
        if args.naive:
            t0 = time.perf_counter()
            fg.naive_sum(qp, wl.references, wl.weights, h)
            line["naive_ms"] = round((time.perf_counter() - t0) * 1e3, 2)
        print(json.dumps(line), flush=True)
    print(f"total kernel ms {tot*1e3:.2f}; effective pairs/s "
          f"{wl.m * wl.n * len(wl.bandwidths) / tot:.3e}")


if __name__ == "__main__":
    main()
