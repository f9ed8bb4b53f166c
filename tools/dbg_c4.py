import os, sys, numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1206_6857_b200 as fg
from paper_1206_6857_b200 import _lib
from paper_1206_6857_b200.configs import config
wl = config(4)
t = fg.build_tree(fg.PointStore(wl.references, wl.weights), 25)
h = wl.bandwidths[15]
print("h", h, "n", wl.n)
for fp32 in (1, 0):
    _lib.call("fg_set_engine_params", 0, 0, fp32)
    for alg, run in (("dfd", fg.dfd_run), ("dito", fg.dito_run)):
        t.refresh_moments(h, fg.default_plimit(7))
        r = run(fg.RunConfig(bandwidth=h, epsilon=0.01, algorithm=alg), t, t)
        v = r.values
        bad = ~np.isfinite(v)
        print(fp32, alg, "nonfinite", bad.sum(), "min", np.nanmin(v), "max", np.nanmax(v[np.isfinite(v)]), r.counters)
        if bad.any():
            idx = np.where(bad)[0][:5]
            print("  bad idx", idx, v[idx])
