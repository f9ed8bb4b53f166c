"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv):
per-kernel totals, and the kernels of the last timed bench step.

  python tools/launch_summary.py gpurun_out/launches.csv [steps]
"""
import collections
import csv
import sys

path = sys.argv[1]
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 0
rows = [r for r in csv.reader(open(path)) if len(r) > 10]
hdr = rows[0]
ki, vi, mi = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Name")
data = [(r[ki], float(r[vi].replace(",", "")) / 1e3) for r in rows[1:]
        if r[mi] == "gpu__time_duration.sum"]
tot = collections.defaultdict(lambda: [0, 0.0])
for k, v in data:
    n = k.split("(")[0].replace("void ", "")
    n = n.split("<")[0] if "cub::" in n else n
    tot[n][0] += 1
    tot[n][1] += v
print(f"launches {len(data)}, summed kernel time {sum(v for _, v in data) / 1e3:.3f} ms")
for n, (c, v) in sorted(tot.items(), key=lambda kv: -kv[1][1]):
    per = f"  per step {v / steps:8.1f} us" if steps else ""
    print(f"{n[:64]:64s} n={c:5d} us={v:10.1f}{per}")
