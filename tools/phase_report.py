"""Per-bandwidth phase breakdown of single runs (needs an engine built with
-DFG_PHASE_PROF=1; tools/build_variant.sh ... EXTRA=-DFG_PHASE_PROF=1).

  FG_LIB=variants/phase.so python tools/phase_report.py --config 2
Phases: 0 step load + FD, 1 series selection, 2 descend, 3 FP32 bound,
4 FP32 batch, 5 FP64 items, 6 deferred series + post, 7 task setup.
"""
import argparse
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
NAMES = ["load+fd", "ser_sel", "descend", "f32bound", "f32batch", "fp64", "ser_eval", "setup"]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--bws", default="")
    args = ap.parse_args()
    import paper_1206_6857_b200 as fg
    from paper_1206_6857_b200.configs import config

    wl = config(args.config)
    rt = fg.build_tree(fg.PointStore(wl.references, wl.weights), 25)
    bws = range(len(wl.bandwidths)) if not args.bws else [int(v) for v in args.bws.split(",")]
    print("h ms | " + " ".join(f"{n:>9s}" for n in NAMES) + " | top-block share of kernel")
    for j in bws:
        h = wl.bandwidths[j]
        pl = fg.engine_plimit(wl.dim)
        rt.refresh_moments(h, pl)
        path = f"/tmp/phase_{os.getpid()}.bin"
        if os.path.exists(path):
            os.remove(path)
        os.environ["FG_DEBUG_BLOCKS"] = path
        res = fg.dito_run(fg.RunConfig(bandwidth=h, epsilon=wl.epsilon, plimit=pl), rt, rt)
        del os.environ["FG_DEBUG_BLOCKS"]
        a = np.fromfile(path, dtype=np.uint64).reshape(-1, 16).astype(float)
        os.remove(path)
        ph = a[:, 8:16]
        tot = ph.sum()
        top = int(np.argmax(a[:, 0]))
        kern_cyc = res.seconds * 1.965e9
        print(f"{h:.4g} {res.seconds*1e3:.2f} | " +
              " ".join(f"{100*v/tot:8.1f}%" for v in ph.sum(0)) +
              f" | top {a[top,0]:.3g} cyc ({a[top,0]/kern_cyc:.2f} of kernel), steps {a[top,1]:.0f}, "
              f"visits {a[top,2]:.0f}, f32 pairs {a[top,4]:.3g}; phases " +
              " ".join(f"{100*v/a[top,8:16].sum():.0f}" for v in a[top, 8:16]), flush=True)


if __name__ == "__main__":
    main()
