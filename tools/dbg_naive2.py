import ctypes, os, sys, numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1206_6857_b200.configs import config
L = ctypes.CDLL(sys.argv[1])
P, I32, I64 = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64
L.fg_naive_sum.argtypes = [P, I64, P, P, I64, I32, P, I32, P]
wl = config(4)
rng = np.random.default_rng(0)
idx = np.sort(rng.choice(wl.m, 500, replace=False))
qp = np.ascontiguousarray(wl.query_points()[idx])
r = np.ascontiguousarray(wl.references); w = np.ascontiguousarray(wl.weights)
for j in (14, 15, 16, 17):
    hs = np.array([wl.bandwidths[j]]); out = np.empty(500)
    st = L.fg_naive_sum(qp.ctypes.data, 500, r.ctypes.data, w.ctypes.data, r.shape[0], 7, hs.ctypes.data, 1, out.ctypes.data)
    print(j, st, out.min(), out.max())
