#!/usr/bin/env python
"""Benchmark: effective Gaussian pair evaluations per second (M*N*bandwidths / T)
at eps=0.01 on BASELINE.json's configs[1] (C2: D=3, M=N=1e5, monochromatic,
10 bandwidths log-spaced 1e-3..1e2 x Silverman h), plus the FP64 roofline
fraction of the dominant kernel.

One step = one full sweep: device kd-tree build (amortised once per sweep, as
the reference's run_sweep does, cli_harness.py:246-283), then for every
bandwidth the moment refresh and a DITO run.  Prints ONE JSON line (rank 0).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Multi-GPU (torchrun, one rank per GPU): query blocks are dealt round-robin to
ranks (the reference tree is rebuilt on every rank, bit-identically), each
rank sums its blocks and one NCCL all-reduce over disjoint supports gathers
the result vector.  Total work is fixed: "scaling": "strong".
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

F_OF_D = {d: 3 * d + 34 for d in range(1, 9)}  # algorithmic FP64 flops per exact pair
METRIC = "effective Gaussian pair evals/sec (M·N/time) at ε=0.01; % of FP64 roofline"
UNIT = "pairs/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--cpu-seconds", type=float, default=10.0,
                    help="target CPU time of one bounded oracle sample")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    return ap.parse_args()


def workload(index):
    from paper_1206_6857_b200.configs import config

    return config(index)


def describe(wl):
    return (f"{wl.name}: D={wl.dim}, M=N={wl.n}, {wl.notes.get('mode')}, "
            f"{len(wl.bandwidths)} bandwidths, eps={wl.epsilon}, h_S={wl.h_star:.5g}")


# ------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md)."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc is not None:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for name, val in zip(names, parts[4:8]):
                if val.lower() == "active":
                    reasons.add(name)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx),
                "reasons": sorted(reasons), "samples": len(sm)}


def profiled_traffic():
    """dram read+write bytes per launch of the dominant kernel, from the
    committed `ncu --set full` summary (profiles/, one traversal launch of this
    same bench command: the whole 10-bandwidth sweep of one step).  Null when
    no summary is present."""
    import glob
    import re

    files = sorted(glob.glob(os.path.join(ROOT, "profiles", "r*_traverse_kernel_full.txt")))
    if not files:
        return None
    txt = open(files[-1]).read()
    tot = 0.0
    for key in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
        m = re.search(key + r"\s+([\d.]+)\s+(\w*byte)", txt)
        if not m:
            return None
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}[m.group(2)]
        tot += float(m.group(1)) * scale
    return {"bytes_per_launch": tot, "source": os.path.basename(files[-1]),
            "launch": "one C2 step's sweep launch (10 bandwidths)"}


# ------------------------------------------------------------ CPU side
def cpu_sample(wl, target_seconds, threads):
    """Bounded sample of the workload on the host with the oracle port of the
    reference's DFS DITO (oracle/fg_oracle.c: fgo_run_sharded): M' seeded query
    rows, bichromatic against the full reference tree (identical per-query sums
    to the monochromatic problem), every bandwidth, `threads` shards.
    Build + per-bandwidth refresh + run are timed, like run_sweep."""
    import oracle

    rng = np.random.default_rng(4242)
    qp = wl.query_points()
    mq = 256
    while True:
        idx = np.sort(rng.choice(qp.shape[0], min(mq, qp.shape[0]), replace=False))
        qs = qp[idx]
        t0 = time.perf_counter()
        rt = oracle.Tree(wl.references, wl.weights, 25)
        pl = {1: 8, 2: 8, 3: 6, 4: 4, 5: 4, 6: 2}.get(wl.dim, 1)
        for h in wl.bandwidths:
            rt.refresh_moments(h, pl)
            oracle.run_sharded("dito", qs, rt, h, wl.epsilon, threads=threads)
        dt = time.perf_counter() - t0
        if dt >= 0.4 * target_seconds or mq >= qp.shape[0]:
            break
        mq = int(min(qp.shape[0], mq * max(2.0, 0.8 * target_seconds / max(dt, 1e-3))))
    pairs = len(idx) * wl.n * len(wl.bandwidths)
    return pairs / dt, dt, len(idx)


def run_reference(args):
    """--impl reference: the reference algorithm (oracle port of its DFS DITO)
    on the host cores, same metric/config, bounded samples per step."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import oracle

    wl = workload(args.config)
    threads = os.cpu_count() or 1
    oracle.lib()
    # calibrate the per-step sample on a warm-up step
    _, _, mq = cpu_sample(wl, args.cpu_seconds, threads)
    rng = np.random.default_rng(4242)
    idx = np.sort(rng.choice(wl.m, mq, replace=False))
    qs = wl.query_points()[idx]
    pl = {1: 8, 2: 8, 3: 6, 4: 4, 5: 4, 6: 2}.get(wl.dim, 1)

    def step():
        rt = oracle.Tree(wl.references, wl.weights, 25)
        for h in wl.bandwidths:
            rt.refresh_moments(h, pl)
            oracle.run_sharded("dito", qs, rt, h, wl.epsilon, threads=threads)

    for _ in range(max(0, args.warmup - 1)):
        step()
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        step()
        times.append(time.perf_counter() - t0)
    total = sum(times)
    pairs = mq * wl.n * len(wl.bandwidths) * args.steps
    value = pairs / total
    sample = (f"{mq} of {wl.m} queries x {len(wl.bandwidths)} bandwidths per step vs the full "
              f"reference tree (bichromatic restatement of the monochromatic sums), "
              f"tree build + refresh + DFS DITO")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT,
        "n_gpus": int(os.environ.get("WORLD_SIZE", str(args.gpus))), "host_only": True,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * total / args.steps,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded; SURVEY Appendix C)",
        "config": {"workload": describe(wl), "sample_queries": mq},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "port",
                         "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------ GPU side
def run_ours(args):
    import torch
    import torch.distributed as dist

    import paper_1206_6857_b200 as fg
    from paper_1206_6857_b200 import _lib
    from paper_1206_6857_b200.spatial_index import build_tree_device
    from paper_1206_6857_b200.distributed import run_sharded, run_sharded_sweep

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    _lib.call("fg_set_device", local)
    stream = torch.cuda.Stream()
    _lib.set_stream(stream.cuda_stream)

    wl = workload(args.config)
    D = wl.dim
    pl = fg.default_plimit(D)
    dev = torch.device("cuda", local)
    pts_d = torch.from_numpy(wl.references).to(dev)
    w_d = torch.from_numpy(wl.weights).to(dev)
    vals_d = torch.zeros(len(wl.bandwidths), wl.m, dtype=torch.float64, device=dev)
    flush = torch.empty(int(512 * 2**20) // 4, dtype=torch.float32, device=dev)
    torch.cuda.synchronize()

    stats = {"kernel_s": 0.0, "pairs": 0, "pairs32": 0, "visits": 0}

    def step(record=True):
        vals_d.zero_()
        tree = build_tree_device(pts_d, w_d, 25)
        # the whole sweep in one engine call (moments for every bandwidth + one
        # traversal launch, one synchronisation); with N ranks each runs its
        # query blocks, then one NCCL all-reduce over disjoint supports gathers
        # every bandwidth's values -- inside the timed step
        cfg = fg.RunConfig(bandwidth=wl.bandwidths[0], epsilon=wl.epsilon, algorithm="dito")
        if world == 1:
            results = fg.sweep_run(cfg, tree, tree, wl.bandwidths, out=vals_d)
        else:
            results = run_sharded_sweep(cfg, tree, tree, wl.bandwidths, vals_d, rank, world)
        if record:
            for res in results:
                stats["kernel_s"] += res.seconds
                stats["pairs"] += res.counters.exact_pairs
                stats["pairs32"] += res.counters.fp32_pairs
                stats["visits"] += res.counters.pair_visits
        del tree

    with torch.cuda.stream(stream):
        for _ in range(args.warmup):
            step(record=False)
        stream.synchronize()
        lc0 = np.zeros(1, np.int64)
        _lib.call("fg_launch_count", _lib.ptr(lc0))
        times = []
        with ClockSampler(local) as clk:
            for _ in range(args.steps):
                flush.zero_()
                stream.synchronize()
                if world > 1:
                    dist.barrier()
                e0 = torch.cuda.Event(enable_timing=True)
                e1 = torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                step()
                e1.record(stream)
                e1.synchronize()
                times.append(e0.elapsed_time(e1) * 1e-3)
        lc1 = np.zeros(1, np.int64)
        _lib.call("fg_launch_count", _lib.ptr(lc1))
    total = sum(times)
    if world > 1:
        t = torch.tensor([total], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total = float(t.item())
    pairs_eff = wl.m * wl.n * len(wl.bandwidths)
    value = pairs_eff * args.steps / total

    # roofline of the dominant kernel (fused traversal + base-case kernel).
    # Its pair work has two legs: FP64 pairs bound by
    # the DFMA pipe at F(D) flops per pair, FP32 pairs bound by the SFU at one
    # ex2 per pair.  peak = the pair rate of the ideal kernel for this step's
    # FP64/FP32 mix; achieved = pairs evaluated / kernel time.
    peak = np.zeros(1)
    _lib.call("fg_fp64_peak", _lib.ptr(peak))
    peak_tf = float(peak[0])
    ex2 = np.zeros(1)
    _lib.call("fg_ex2_peak", _lib.ptr(ex2))
    ex2_gops = float(ex2[0])
    n64, n32, ks = stats["pairs"], stats["pairs32"], stats["kernel_s"]
    ideal_s = n64 * F_OF_D[D] / (peak_tf * 1e12) + n32 / (ex2_gops * 1e9)
    achieved = (n64 + n32) / ks / 1e9 if ks else 0.0
    peak_mix = (n64 + n32) / ideal_s / 1e9 if ideal_s else None
    roofline = {"bound": "fp64+sfu", "achieved": achieved, "peak": peak_mix, "unit": "Gpair/s",
                "frac": achieved / peak_mix if peak_mix else None,
                "traffic": profiled_traffic(),
                "kernel": f"traverse_kernel<{D}> (fused traversal + leaf base cases)",
                "legs": {"fp64": {"pairs_per_step": n64 / args.steps,
                                  "flops_per_pair": F_OF_D[D], "peak_tflops": peak_tf,
                                  "achieved_tflops_over_kernel_time":
                                      n64 * F_OF_D[D] / ks / 1e12 if ks else 0.0},
                         "fp32": {"pairs_per_step": n32 / args.steps, "ex2_per_pair": 1,
                                  "peak_ex2_gops": ex2_gops}},
                "kernel_share_of_step": ks / total if total else None,
                "visits_per_s_in_kernel": stats["visits"] / ks if ks else None,
                "peak_source": "measured: DFMA microbenchmark fg_fp64_peak and ex2.approx "
                               "microbenchmark fg_ex2_peak (burst)",
                "pair_share": {"fp64": n64 / (pairs_eff * args.steps),
                               "fp32": n32 / (pairs_eff * args.steps)}}

    # end to end through the public API with host buffers: the step's inputs
    # come from pinned host memory and all its value vectors go back into a
    # pinned host array (host <-> device copies inside the timed region)
    e2e = None
    if not args.no_e2e and world == 1:
        pts_h = torch.from_numpy(wl.references).pin_memory().numpy()
        w_h = torch.from_numpy(wl.weights).pin_memory().numpy()
        out_h = torch.empty((len(wl.bandwidths), wl.m), dtype=torch.float64,
                            pin_memory=True).numpy()

        def e2e_step():
            store = fg.PointStore(pts_h, w_h)
            tree = fg.build_tree(store, 25)
            cfg = fg.RunConfig(bandwidth=wl.bandwidths[0], epsilon=wl.epsilon)
            return [r.values for r in fg.sweep_run(cfg, tree, tree, wl.bandwidths, out=out_h)]

        with torch.cuda.stream(stream):
            e2e_step()
            et = []
            for _ in range(max(1, args.steps)):
                flush.zero_()
                stream.synchronize()
                e0 = torch.cuda.Event(enable_timing=True)
                e1 = torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                e2e_step()
                e1.record(stream)
                e1.synchronize()
                et.append(e0.elapsed_time(e1) * 1e-3)
        e2e = {"value": pairs_eff * len(et) / sum(et), "unit": UNIT,
               "h2d_bytes_per_step": int(wl.references.nbytes + wl.weights.nbytes),
               "d2h_bytes_per_step": int(8 * wl.m * len(wl.bandwidths)),
               "ms_per_step": 1e3 * sum(et) / len(et)}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        threads = os.cpu_count() or 1
        v, dt, mq = cpu_sample(wl, args.cpu_seconds, threads)
        cpu = {"value": v, "unit": UNIT, "cores": threads, "kind": "port",
               "sample": f"{mq} of {wl.m} queries x {len(wl.bandwidths)} bandwidths vs the full "
                         f"reference tree, oracle DFS DITO, {dt:.1f} s"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * total / args.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "f64+f32",
            "dtype_note": "FP64 traversal, bounds, series and results; leaf pairs in FP32 where "
                          "their rigorous error bound fits a reserved 10% of eps (DESIGN.md)",
            "data": "synthetic (seeded; SURVEY Appendix C)",
            "config": {"workload": describe(wl), "epsilon": wl.epsilon,
                       "bandwidths": len(wl.bandwidths), "parallelism": f"query-blocks x{world}",
                       "l2": "flushed (512 MiB write) between timed steps",
                       "engine": {"query_block": 64, "ref_leaf": "32/64/128 (D <= 4), 32/64/128/256 (D >= 5), by h / median block radius",
                                  "tree_leaf": 25}},
            "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e,
            "gpu_launches": int(lc1[0] - lc0[0]),
            "clocks": clk.summary(),
            "detail": {"kernel_ms_per_step": 1e3 * stats["kernel_s"] / args.steps,
                       "visits_per_step": stats["visits"] / args.steps,
                       "exact_pairs_per_step": stats["pairs"] / args.steps,
                       "fp32_pairs_per_step": stats["pairs32"] / args.steps},
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
