"""Per-bandwidth single-run kernel ms for several reference base-item sizes.

  python tools/leaf_scan.py --config 4 --leaves 64,128,256 [--scale 1.0]
Prints one row per bandwidth: h, h / median block radius, ms per leaf size,
and the FP32 pair share of the last size.
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=4)
    ap.add_argument("--leaves", default="64,128,256")
    ap.add_argument("--scale", type=float, default=1.0)
    ap.add_argument("--bws", default="")
    args = ap.parse_args()
    import paper_1206_6857_b200 as fg
    from paper_1206_6857_b200 import _lib
    from paper_1206_6857_b200.configs import config

    wl = config(args.config, scale=args.scale)
    leaves = [int(v) for v in args.leaves.split(",")]
    rt = fg.build_tree(fg.PointStore(wl.references, wl.weights), 25)
    qt = rt if wl.monochromatic else fg.build_tree(fg.PointStore(wl.queries), 25)
    pl = fg.default_plimit(wl.dim)
    bws = range(len(wl.bandwidths)) if not args.bws else [int(v) for v in args.bws.split(",")]
    print("h " + " ".join(f"L{v}" for v in leaves))
    for j in bws:
        h = wl.bandwidths[j]
        rt.refresh_moments(h, pl)
        row = []
        for leaf in leaves:
            _lib.call("fg_set_engine_params", leaf, 0, -1)
            cfg = fg.RunConfig(bandwidth=h, epsilon=wl.epsilon)
            fg.dito_run(cfg, qt, rt)
            res = fg.dito_run(cfg, qt, rt)
            row.append(res.seconds * 1e3)
        c = res.counters
        print(f"{h:.4g} " + " ".join(f"{v:.2f}" for v in row) +
              f"  fp32 {c.fp32_pairs / (wl.m * wl.n):.3f} visits {c.pair_visits}", flush=True)
    _lib.call("fg_set_engine_params", -1, 0, -1)


if __name__ == "__main__":
    main()
