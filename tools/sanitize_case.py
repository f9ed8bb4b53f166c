"""Small engine workload for compute-sanitizer (racecheck / synccheck /
memcheck): device tree build (build_coop_kernel), moments, a DITO sweep and a
DFDO run through traverse_kernel (FP32 record-pair batches with bulk copies,
FP64 items, Hermite ring), the far-field pass, and the exhaustive kernel.

  compute-sanitizer --tool racecheck python tools/sanitize_case.py --dim 3
"""
import argparse
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--dim", type=int, default=3)
    ap.add_argument("--n", type=int, default=3000)
    args = ap.parse_args()
    import paper_1206_6857_b200 as fg

    rng = np.random.default_rng(args.dim)
    pts = np.concatenate([rng.normal(0.3, 0.05, (args.n // 2, args.dim)),
                          rng.random((args.n - args.n // 2, args.dim))])
    w = rng.uniform(0.5, 1.5, args.n)
    tree = fg.build_tree(fg.PointStore(pts, w), 25)
    hs = [0.02, 0.1, 0.5]
    cfg = fg.RunConfig(bandwidth=hs[0], epsilon=0.001)
    res = fg.sweep_run(cfg, tree, tree, hs)
    tree.refresh_moments(0.1, fg.default_plimit(args.dim))
    r2 = fg.dfdo_run(fg.RunConfig(bandwidth=0.1, epsilon=0.01), tree, tree)
    ex = fg.naive_sum(pts[:200], pts, w, hs).values
    err = max(float(np.max(np.abs(res[j].values[:200] - ex[j]) / ex[j])) for j in range(3))
    print(f"D={args.dim} n={args.n} sweep max err {err:.3e}, dfdo visits {r2.counters.pair_visits}")


if __name__ == "__main__":
    main()
