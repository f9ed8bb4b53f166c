import os, sys, numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1206_6857_b200 as fg
import oracle
from paper_1206_6857_b200.configs import config
wl = config(4)
rng = np.random.default_rng(0)
idx = np.sort(rng.choice(wl.m, 500, replace=False))
qp = wl.query_points()[idx]
for j in (14, 15, 16, 17, 18):
    h = wl.bandwidths[j]
    g = fg.naive_sum(qp, wl.references, wl.weights, h).values
    print(j, h, "zeros", (g == 0).sum(), "nonfinite", (~np.isfinite(g)).sum(), "min", g.min())
    if (g == 0).any():
        k = np.where(g == 0)[0][:3]
        ex = oracle.naive_sum(qp[k], wl.references, wl.weights, h, threads=0)
        print("   oracle at zeros", ex)
    sub = slice(0, 20)
    ex = oracle.naive_sum(qp[sub], wl.references, wl.weights, h, threads=0)
    print("   rel err first 20", np.max(np.abs(g[sub] - ex) / ex))
