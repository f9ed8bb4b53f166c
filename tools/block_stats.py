"""Summarise FG_DEBUG_BLOCKS dumps (per query block: cycles, steps, visits, pairs)."""
import sys
import numpy as np
a = np.fromfile(sys.argv[1], dtype=np.uint64).reshape(-1, 16)[:, :4].astype(float)
nb = int(sys.argv[2]) if len(sys.argv) > 2 else a.shape[0]
for r in range(a.shape[0] // nb):
    blk = a[r * nb:(r + 1) * nb]
    cyc, st, vis, pr = blk.T
    o = np.argsort(-cyc)
    print(f"run {r}: blocks {nb} cycles mean {cyc.mean():.3e} max {cyc.max():.3e} p99 {np.percentile(cyc,99):.3e} "
          f"sum/148/4 {cyc.sum()/148/16:.3e}; steps mean {st.mean():.1f} max {st.max():.0f}; "
          f"visits mean {vis.mean():.0f} max {vis.max():.0f}; pairs mean {pr.mean():.3e} max {pr.max():.3e}")
    print("   top blocks (cycles, steps, visits, pairs):", [tuple(int(v) for v in blk[i]) for i in o[:5]])
