"""Wall-clock breakdown of one bench step (build, refresh, runs) after warm-up."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_1206_6857_b200 as fg
from paper_1206_6857_b200.configs import config
from paper_1206_6857_b200.spatial_index import build_tree_device
from paper_1206_6857_b200.summation_engine import query_block_count

wl = config(int(sys.argv[1]) if len(sys.argv) > 1 else 2)
pts = torch.from_numpy(wl.references).cuda()
w = torch.from_numpy(wl.weights).cuda()
out = torch.zeros(wl.m, dtype=torch.float64, device="cuda")
pl = fg.default_plimit(wl.dim)
for rep in range(3):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    tree = build_tree_device(pts, w, 25)
    torch.cuda.synchronize(); t1 = time.perf_counter()
    nb = query_block_count(tree)
    torch.cuda.synchronize(); t2 = time.perf_counter()
    tr = tk = 0.0
    kern = 0.0
    for h in wl.bandwidths:
        a = time.perf_counter()
        tree.refresh_moments(h, pl)
        torch.cuda.synchronize(); b = time.perf_counter()
        res = fg.dito_run(fg.RunConfig(bandwidth=h, epsilon=wl.epsilon), tree, tree, out=out)
        torch.cuda.synchronize(); c = time.perf_counter()
        tr += b - a; tk += c - b; kern += res.seconds
    del tree
    torch.cuda.synchronize(); t3 = time.perf_counter()
    print(f"rep {rep}: build {1e3*(t1-t0):.2f} ms, qblocks {1e3*(t2-t1):.2f} ms, refresh {1e3*tr:.2f} ms, "
          f"runs {1e3*tk:.2f} ms (kernels {1e3*kern:.2f}), total {1e3*(t3-t0):.2f} ms, levels {0}")
