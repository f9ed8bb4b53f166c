import os, sys, numpy as np
sys.path.insert(0, os.getcwd())
import paper_1206_6857_b200 as fg
from paper_1206_6857_b200.configs import config
c = int(sys.argv[1])
wl = config(c)
rt = fg.build_tree(fg.PointStore(wl.references, wl.weights), 25)
out = {}
for j, h in enumerate(wl.bandwidths):
    rt.refresh_moments(h, fg.default_plimit(wl.dim))
    path = f"gpurun_out/blk_c{c}_{j}.bin"
    if os.path.exists(path): os.remove(path)
    os.environ["FG_DEBUG_BLOCKS"] = path
    res = fg.dito_run(fg.RunConfig(bandwidth=h, epsilon=wl.epsilon), rt, rt)
    del os.environ["FG_DEBUG_BLOCKS"]
    a = np.fromfile(path, dtype=np.uint64).reshape(-1, 16)
    out[f"cyc{j}"] = a[:, 0].astype(float); out[f"vis{j}"] = a[:, 2].astype(float)
    out["rad"] = a[:, 3].view(np.float64)
    out[f"f32_{j}"] = a[:, 4].astype(float)
    out[f"ph{j}"] = a[:, 8:16].astype(float)
    os.remove(path)
    print(j, h, res.seconds)
np.savez(f"gpurun_out/blk_c{c}.npz", hs=np.array(wl.bandwidths), **out)
