"""Run sweep_run on a config (for ncu captures of the single sweep launch).

  python tools/one_sweep.py --config 2 [--reps 2]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--reps", type=int, default=2)
    ap.add_argument("--plimit", type=int, default=None)
    args = ap.parse_args()
    import paper_1206_6857_b200 as fg
    from paper_1206_6857_b200.configs import config

    wl = config(args.config)
    rt = fg.build_tree(fg.PointStore(wl.references, wl.weights), 25)
    qt = rt if wl.monochromatic else fg.build_tree(fg.PointStore(wl.queries), 25)
    cfg = fg.RunConfig(bandwidth=wl.bandwidths[0], epsilon=wl.epsilon, plimit=args.plimit)
    best = None
    for i in range(args.reps):
        res = fg.sweep_run(cfg, qt, rt, wl.bandwidths)
        ms = sum(r.seconds for r in res) * 1e3
        if i > 0 or args.reps == 1:
            best = ms if best is None else min(best, ms)
    print("sweep kernel ms", best, "(min over reps after the first)")


if __name__ == "__main__":
    main()
