#!/usr/bin/env python
"""Benchmark: effective Gaussian pair evaluations per second (M*N*bandwidths / T)
on the largest single-GPU config of BASELINE.json, configs[4] (C5: D=3,
M=N=4e6, monochromatic, 16 bandwidths log-spaced 1e-3..1e2 x Silverman h,
eps=0.001), plus the roofline fraction of the dominant kernel.

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
    # C5 is the largest config that fits one GPU (4e6 points: 128 MB of
    # points + 16 x 32 MB of values); configs 1-4 are parity cases
    ap.add_argument("--config", type=int, default=5)
    ap.add_argument("--sample-queries", type=int, default=0,
                    help="CPU sample size M' (default: BASELINE.md section 3 per config)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    return ap.parse_args()


# seeded query subsamples for the CPU path, run
# bichromatically against the FULL reference tree (identical per-query sums)
SAMPLE_QUERIES = {1: 0, 2: 10_000, 3: 4_096, 4: 1_024, 5: 1_024}  # 0 = all queries


def workload(index):
    from paper_1206_6857_b200.configs import config

    return config(index)


def describe(wl):
    return (f"{wl.name}: D={wl.dim}, M=N={wl.n}, {wl.notes.get('mode')}, "
            f"{len(wl.bandwidths)} bandwidths, eps={wl.epsilon}, h_S={wl.h_star:.5g}")


def config_dict(wl, world):
    """The `config` object both arms print (identical keys and values)."""
    return {"workload": describe(wl), "epsilon": wl.epsilon, "bandwidths": len(wl.bandwidths),
            "parallelism": f"query shards x{world}",
            "l2": "GPU arm: 512 MiB L2 flush between timed steps (inputs 128 MB > L2 too)"}


def host_info(threads):
    model = "unknown"
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name"):
                    model = ln.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    return {"cpu_model": model, "os_cpu_count": os.cpu_count(), "threads_used": threads,
            "OMP_NUM_THREADS": os.environ.get("OMP_NUM_THREADS"),
            "OPENBLAS_NUM_THREADS": os.environ.get("OPENBLAS_NUM_THREADS")}


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
    same bench command: the whole sweep of one step).  Null when no summary is
    present."""
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
    m = re.search(r"^# launch: (.*)$", txt, re.M)
    return {"bytes_per_launch": tot, "source": os.path.basename(files[-1]),
            "launch": m.group(1) if m else "see the summary header"}


# ------------------------------------------------------------ CPU side
def cpu_step_factory(wl, mq, threads):
    """One step of the reference's algorithm on the host: the oracle port of
    its DFS DITO (oracle/fg_oracle.c: fgo_run_sharded, `threads` disjoint query
    shards).  M' seeded query rows, bichromatic against the full reference
    tree (identical per-query sums to the monochromatic problem).  Mirrors
    run_sweep's accounting (cli_harness.py:246-283): the reference tree build
    once per sweep, then per bandwidth refresh_moments + dito_run."""
    import oracle

    qp = wl.query_points()
    if mq <= 0 or mq >= qp.shape[0]:
        qs = qp
    else:
        rng = np.random.default_rng(4242)
        qs = qp[np.sort(rng.choice(qp.shape[0], mq, replace=False))]
    pl = {1: 8, 2: 8, 3: 6, 4: 4, 5: 4, 6: 2}.get(wl.dim, 1)

    def step():
        rt = oracle.Tree(wl.references, wl.weights, 25)
        for h in wl.bandwidths:
            rt.refresh_moments(h, pl)
            oracle.run_sharded("dito", qs, rt, h, wl.epsilon, threads=threads)

    return step, qs.shape[0]


def sample_desc(wl, mq, dt):
    ext = dt * wl.m / mq
    return (f"{mq} of {wl.m} seeded queries (BASELINE.md section 3) x {len(wl.bandwidths)} "
            f"bandwidths per step vs the full {wl.n}-point reference tree (bichromatic "
            f"restatement of the monochromatic sums): tree build + per-bandwidth refresh + "
            f"DFS DITO, {dt:.1f} s per step; extrapolated full-M step {ext:.4g} s")


def run_reference(args):
    """--impl reference: the reference algorithm (oracle port of its DFS DITO,
    the reference being pure Python that cannot travel to the GPU box) on all
    host cores, same metric/config, a bounded query sample per step."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import oracle

    wl = workload(args.config)
    world = int(os.environ.get("WORLD_SIZE", str(args.gpus)))
    threads = os.cpu_count() or 1
    oracle.lib()
    step, mq = cpu_step_factory(wl, args.sample_queries or SAMPLE_QUERIES[args.config], threads)
    for _ in range(args.warmup):
        step()
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        step()
        times.append(time.perf_counter() - t0)
    total = sum(times)
    pairs = mq * wl.n * len(wl.bandwidths) * args.steps
    value = pairs / total
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT,
        "n_gpus": world, "host_only": True,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * total / args.steps,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded; SURVEY Appendix C)",
        "config": config_dict(wl, world),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "port",
                         "sample": sample_desc(wl, mq, total / args.steps),
                         "host": host_info(threads)},
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

    stats = {"kernel_s": 0.0, "pairs": 0, "pairs32": 0, "visits": 0, "herm": 0,
             "herm_terms": 0}

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
                c = res.counters
                stats["kernel_s"] += res.seconds
                stats["pairs"] += c.exact_pairs
                stats["pairs32"] += c.fp32_pairs
                stats["visits"] += c.pair_visits
                stats["herm"] += c.hermite_evals
                stats["herm_terms"] += c.hermite_terms
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

    # Roofline of the dominant kernel (the fused traversal + base-case kernel;
    # DESIGN.md "Roofline").  Its algorithmic work has three legs, each at its
    # own measured peak: FP64 pairs at F(D) = 3D + 34 flops on the DFMA pipe,
    # FP32 pairs at one ex2 each on the SFU, Hermite far-field evaluations at
    # 2 K_p + 31 + 4D FP64 flops each (the dot with the moments, one exp, the
    # offsets) on the DFMA pipe.  ideal = the time an ideal kernel needs for
    # exactly this work; frac = ideal / measured kernel time.
    peak = np.zeros(1)
    _lib.call("fg_fp64_peak", _lib.ptr(peak))
    peak_tf = float(peak[0])
    ex2 = np.zeros(1)
    _lib.call("fg_ex2_peak", _lib.ptr(ex2))
    ex2_gops = float(ex2[0])
    n64, n32, ks = stats["pairs"], stats["pairs32"], stats["kernel_s"]
    herm_flops = 2.0 * stats["herm_terms"] + (31 + 4 * D) * stats["herm"]
    t64 = n64 * F_OF_D[D] / (peak_tf * 1e12)
    t32 = n32 / (ex2_gops * 1e9)
    th = herm_flops / (peak_tf * 1e12)
    ideal_s = t64 + t32 + th
    frac = ideal_s / ks if ks else None
    # achieved/peak in pair units: pairs per second of kernel time against the
    # pair rate of the ideal kernel on this step's mix
    achieved = (n64 + n32) / ks / 1e9 if ks else 0.0
    peak_mix = (n64 + n32) / ideal_s / 1e9 if ideal_s else None
    roofline = {"bound": "fp64+sfu", "achieved": achieved, "peak": peak_mix, "unit": "Gpair/s",
                "frac": frac,
                "traffic": profiled_traffic(),
                "kernel": f"traverse_kernel<{D}> (fused traversal + leaf base cases + far field)",
                "legs": {"fp64": {"pairs_per_step": n64 / args.steps,
                                  "flops_per_pair": F_OF_D[D], "peak_tflops": peak_tf,
                                  "ideal_ms_per_step": 1e3 * t64 / args.steps},
                         "fp32": {"pairs_per_step": n32 / args.steps, "ex2_per_pair": 1,
                                  "peak_ex2_gops": ex2_gops,
                                  "ideal_ms_per_step": 1e3 * t32 / args.steps},
                         "hermite": {"evals_per_step": stats["herm"] / args.steps,
                                     "flops_per_step": herm_flops / args.steps,
                                     "flops_per_eval": "2 K_p + 31 + 4D",
                                     "ideal_ms_per_step": 1e3 * th / args.steps}},
                "kernel_ms_per_step": 1e3 * ks / args.steps,
                "kernel_share_of_step": ks / total if total else None,
                "visits_per_s_in_kernel": stats["visits"] / ks if ks else None,
                "peak_source": "measured in this process: DFMA microbenchmark fg_fp64_peak and "
                               "ex2.approx microbenchmark fg_ex2_peak (burst; MEASURED_PEAKS.json "
                               "has no FP64/SFU entry); nominal DFMA 148 x 64 x 2 x 1.965 GHz = "
                               "37.2 TF/s",
                "pair_share": {"fp64": n64 / (pairs_eff * args.steps),
                               "fp32": n32 / (pairs_eff * args.steps)}}

    # end to end through the public API with host buffers: every rank builds
    # its tree from pinned host arrays (H2D inside the step); one rank runs
    # the whole sweep into a pinned host array, N ranks run their shards into
    # a device vector, all-reduce it, and rank 0 reads the result back
    e2e = None
    if not args.no_e2e:
        pts_h = torch.from_numpy(wl.references).pin_memory().numpy()
        w_h = torch.from_numpy(wl.weights).pin_memory().numpy()
        out_h = torch.empty((len(wl.bandwidths), wl.m), dtype=torch.float64,
                            pin_memory=True)

        def e2e_step():
            store = fg.PointStore(pts_h, w_h)
            tree = fg.build_tree(store, 25)
            cfg = fg.RunConfig(bandwidth=wl.bandwidths[0], epsilon=wl.epsilon)
            if world == 1:
                fg.sweep_run(cfg, tree, tree, wl.bandwidths, out=out_h.numpy())
            else:
                run_sharded_sweep(cfg, tree, tree, wl.bandwidths, vals_d, rank, world)
                if rank == 0:
                    out_h.copy_(vals_d, non_blocking=True)

        with torch.cuda.stream(stream):
            e2e_step()
            et = []
            for _ in range(max(1, args.steps)):
                flush.zero_()
                stream.synchronize()
                if world > 1:
                    dist.barrier()
                e0 = torch.cuda.Event(enable_timing=True)
                e1 = torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                e2e_step()
                e1.record(stream)
                e1.synchronize()
                et.append(e0.elapsed_time(e1) * 1e-3)
        etot = sum(et)
        if world > 1:
            t = torch.tensor([etot], dtype=torch.float64, device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            etot = float(t.item())
        e2e = {"value": pairs_eff * len(et) / etot, "unit": UNIT,
               "h2d_bytes_per_step": int(world * (wl.references.nbytes + wl.weights.nbytes)),
               "d2h_bytes_per_step": int(8 * wl.m * len(wl.bandwidths)),
               "ms_per_step": 1e3 * etot / len(et)}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        threads = os.cpu_count() or 1
        cstep, mq = cpu_step_factory(wl, args.sample_queries or SAMPLE_QUERIES[args.config],
                                     threads)
        t0 = time.perf_counter()
        cstep()
        dt = time.perf_counter() - t0
        cpu = {"value": mq * wl.n * len(wl.bandwidths) / dt, "unit": UNIT, "cores": threads,
               "kind": "port", "sample": sample_desc(wl, mq, dt), "host": host_info(threads)}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * total / args.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "f64+f32",
            "dtype_note": "FP64 traversal, bounds, series and results; leaf pairs in FP32 where "
                          "their rigorous error bound fits a reserved 10% of eps (DESIGN.md)",
            "data": "synthetic (seeded; SURVEY Appendix C)",
            "config": config_dict(wl, world),
            "engine": {"query_block": 64, "tree_leaf": 25,
                       "ref_leaf": "32/64/128 (D <= 4), 32/64/128/256 (D >= 5), by h / median "
                                   "block radius"},
            "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e,
            "gpu_launches": int(lc1[0] - lc0[0]),
            "clocks": clk.summary(),
            "detail": {"kernel_ms_per_step": 1e3 * stats["kernel_s"] / args.steps,
                       "hermite_evals_per_step": stats["herm"] / args.steps,
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
