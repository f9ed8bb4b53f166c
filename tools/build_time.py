"""Time the device tree build (CUDA events) on a config's reference points.

  python tools/build_time.py --config 2 [--reps 10]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--reps", type=int, default=10)
    args = ap.parse_args()
    import torch
    import paper_1206_6857_b200 as fg
    from paper_1206_6857_b200.configs import config
    from paper_1206_6857_b200.spatial_index import build_tree_device

    wl = config(args.config)
    pts = torch.from_numpy(wl.references).cuda()
    w = torch.from_numpy(wl.weights).cuda()
    ts = []
    for _ in range(args.reps):
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        t = build_tree_device(pts, w, 25)
        e1.record()
        e1.synchronize()
        ts.append(e0.elapsed_time(e1))
        del t
    print(f"build ms: min {min(ts):.3f} median {sorted(ts)[len(ts) // 2]:.3f}")


if __name__ == "__main__":
    main()
