import sys, numpy as np
sys.path.insert(0, '.')
import paper_1206_6857_b200 as fg
from paper_1206_6857_b200.configs import config
from paper_1206_6857_b200.summation_engine import query_block_ranges
for c in (2, 3, 4, 5):
    wl = config(c)
    t = fg.build_tree(fg.PointStore(wl.references, wl.weights), 25)
    st, cn = query_block_ranges(t)
    e = t.arrays()
    P = wl.references[e["perm"]]
    rads = []
    for s0, c0 in zip(st, cn):
        x = P[s0:s0 + c0]
        ctr = x.mean(0)
        rads.append(np.abs(x - ctr).max())
    rb = float(np.median(rads))
    print(c, "blocks", len(st), "median r_b", rb, "h/r_b", [round(h / rb, 3) for h in wl.bandwidths])
