"""Kernel timeline of bench steps (torch.profiler / CUPTI): start offsets,
durations and the idle gaps between consecutive kernels of one step.

  python tools/step_timeline.py [--config 2]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=2)
    args = ap.parse_args()
    import torch
    from torch.profiler import ProfilerActivity, profile

    import paper_1206_6857_b200 as fg
    from paper_1206_6857_b200.configs import config
    from paper_1206_6857_b200.spatial_index import build_tree_device

    wl = config(args.config)
    pts = torch.from_numpy(wl.references).cuda()
    w = torch.from_numpy(wl.weights).cuda()
    vals = torch.zeros(len(wl.bandwidths), wl.m, dtype=torch.float64, device="cuda")

    def step():
        vals.zero_()
        tree = build_tree_device(pts, w, 25)
        cfg = fg.RunConfig(bandwidth=wl.bandwidths[0], epsilon=wl.epsilon)
        fg.sweep_run(cfg, tree, tree, wl.bandwidths, out=vals)
        torch.cuda.synchronize()

    for _ in range(3):
        step()
    with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
        step()
    evs = [e for e in prof.events() if e.device_type.name == "CUDA"]
    evs.sort(key=lambda e: e.time_range.start)
    t0 = evs[0].time_range.start
    prev = t0
    busy = 0.0
    for e in evs:
        s, d = e.time_range.start, e.time_range.elapsed_us()
        gap = s - prev
        print(f"{(s - t0) / 1e3:8.3f} ms  gap {gap:8.1f} us  dur {d:8.1f} us  {e.name[:70]}")
        prev = max(prev, e.time_range.end)
        busy += d
    print(f"span {(prev - t0) / 1e3:.3f} ms, kernels busy {busy / 1e3:.3f} ms")


if __name__ == "__main__":
    main()
