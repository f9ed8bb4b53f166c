"""Summarise an ncu --set full report (one kernel launch) into a small text file.

  python tools/ncu_summary.py gpurun_out/x.ncu-rep > profiles/x.txt
"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units, vals = rows[0], rows[1], rows[2]
get = {h: (v, u) for h, u, v in zip(hdr, units, vals)}
keys = [
    "Kernel Name", "gpu__time_duration.sum", "launch__grid_size", "launch__block_size",
    "launch__registers_per_thread", "launch__occupancy_limit_registers",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "smsp__inst_executed.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
    "l1tex__t_sector_hit_rate.pct", "sm__cycles_elapsed.avg.per_second",
]
print(f"# ncu summary of {rep.split('/')[-1]}")
for k in keys:
    if k in get:
        v, u = get[k]
        print(f"{k:62s} {v} {u}")
tot = float(get.get("smsp__pcsamp_sample_count", ("0", ""))[0] or 0)
pre = "smsp__pcsamp_warps_issue_stalled_"
st = [(float(v.replace(",", "")), h[len(pre):]) for h, (v, u) in get.items()
      if h.startswith(pre) and not h.endswith("not_issued") and v not in ("", "n/a")]
st.sort(reverse=True)
if tot:
    print("stall reasons (share of PC samples):",
          ", ".join(f"{n} {100 * v / tot:.1f}%" for v, n in st[:8]))
