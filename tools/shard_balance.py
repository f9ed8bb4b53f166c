"""Per-rank cost of the multi-GPU query sharding, measured on one GPU.

For each world size N, runs every rank's shard of a config's whole DITO sweep
(``fg_run_sweep_range`` with the round-robin block deal of
``distributed.shard_blocks``) one after another on the same GPU and reports
each shard's device time.  The busiest shard bounds an N-GPU sweep, so
``full / (N * max shard)`` is the traversal's strong-scaling efficiency from
load balance alone (the replicated tree build and the final all-reduce are
not included).  Shards are also checked to sum bit-exactly to the full sweep.

    python tools/shard_balance.py --config 5 --worlds 2 4 8
"""

import argparse
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_1206_6857_b200 as fg  # noqa: E402
from paper_1206_6857_b200.summation_engine import query_block_count  # noqa: E402
from paper_1206_6857_b200.configs import config  # noqa: E402
from paper_1206_6857_b200.distributed import shard_blocks  # noqa: E402


def timed_sweep(cfg, qt, rt, hs, out, block_range=None):
    start, stop = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    start.record()
    fg.sweep_run(cfg, qt, rt, hs, out=out, block_range=block_range)
    stop.record()
    torch.cuda.synchronize()
    return start.elapsed_time(stop)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=5)
    ap.add_argument("--worlds", type=int, nargs="+", default=[2, 4, 8])
    ap.add_argument("--reps", type=int, default=3)
    args = ap.parse_args()

    wl = config(args.config)
    rt = fg.build_tree(fg.PointStore(wl.references, wl.weights), 25)
    qt = rt if wl.monochromatic else fg.build_tree(fg.PointStore(wl.queries), 25)
    hs = list(wl.bandwidths)
    cfg = fg.RunConfig(bandwidth=hs[0], epsilon=wl.epsilon)
    nb = query_block_count(qt)
    full = torch.zeros(len(hs), wl.m, dtype=torch.float64, device="cuda")
    timed_sweep(cfg, qt, rt, hs, full)  # warm-up
    t_full = min(timed_sweep(cfg, qt, rt, hs, full) for _ in range(args.reps))
    rows = []
    for world in args.worlds:
        acc = torch.zeros_like(full)
        times = []
        for rank in range(world):
            part = torch.zeros_like(full)
            br = shard_blocks(nb, rank, world)
            times.append(min(timed_sweep(cfg, qt, rt, hs, part, br) for _ in range(args.reps)))
            acc += part
        exact = bool(torch.equal(acc, full))
        rows.append({"world": world, "shard_ms": [round(t, 3) for t in times],
                     "max_ms": round(max(times), 3), "mean_ms": round(float(np.mean(times)), 3),
                     "efficiency": round(t_full / (world * max(times)), 4),
                     "shards_sum_bit_exact": exact})
    print(json.dumps({"config": wl.name, "query_blocks": nb, "bandwidths": len(hs),
                      "full_sweep_ms": round(t_full, 3), "worlds": rows}))


if __name__ == "__main__":
    main()
