"""Run one engine call (for ncu captures): config, bandwidth index, algorithm.

  python tools/one_run.py --config 2 --bw 6 [--reps 2]
The first rep is a warm-up; ncu should skip it (-s 1 on the traverse kernel).
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--scale", type=float, default=1.0)
    ap.add_argument("--bw", type=int, default=6)
    ap.add_argument("--algo", default="dito")
    ap.add_argument("--reps", type=int, default=2)
    ap.add_argument("--naive", action="store_true")
    ap.add_argument("--ref-leaf", type=int, default=0)
    ap.add_argument("--plimit", type=int, default=0, help="series order cap (default: the engine's)")
    args = ap.parse_args()
    import paper_1206_6857_b200 as fg
    from paper_1206_6857_b200.configs import config

    if args.ref_leaf:
        from paper_1206_6857_b200 import _lib
        _lib.call("fg_set_engine_params", args.ref_leaf, 0, -1)
    wl = config(args.config, scale=args.scale)
    h = wl.bandwidths[args.bw]
    if args.naive:
        for _ in range(args.reps):
            fg.naive_sum(wl.query_points(), wl.references, wl.weights, h)
        return
    rt = fg.build_tree(fg.PointStore(wl.references, wl.weights), 25)
    qt = rt if wl.monochromatic else fg.build_tree(fg.PointStore(wl.queries), 25)
    pl = args.plimit or fg.engine_plimit(wl.dim)
    rt.refresh_moments(h, pl)
    run = {"dfd": fg.dfd_run, "dfdo": fg.dfdo_run, "dito": fg.dito_run}[args.algo]
    for _ in range(args.reps):
        res = run(fg.RunConfig(bandwidth=h, epsilon=wl.epsilon, plimit=pl), qt, rt)
    print(f"h={h:.5g} kernel {res.seconds*1e3:.3f} ms counters {res.counters}")


if __name__ == "__main__":
    main()
