"""Group an ncu report's per-line instruction counts and stall samples by
file and by line range of fg_traverse_kernel.cuh (ranges given as name=a-b).

  python tools/ncu_regions.py gpurun_out/x.ncu-rep step=430-540 base=540-610
"""
import csv
import io
import subprocess
import sys
from collections import defaultdict

rep = sys.argv[1]
ranges = []
for arg in sys.argv[2:]:
    name, span = arg.split("=")
    a, b = span.split("-")
    ranges.append((name, int(a), int(b)))
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
fname, hdr = "?", None
agg = defaultdict(lambda: [0, 0])
for r in csv.reader(io.StringIO(out)):
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or r[0] in ("", "Function Name"):
        continue
    d = dict(zip(hdr, r))
    try:
        s = int(d.get("Warp Stall Sampling (All Samples)", "0") or 0)
        i = int(d.get("Instructions Executed", "0") or 0)
        ln = int(r[0])
    except ValueError:
        continue
    key = fname
    if fname == "fg_traverse_kernel.cuh":
        for name, a, b in ranges:
            if a <= ln <= b:
                key = f"{fname}:{name}"
                break
    agg[key][0] += s
    agg[key][1] += i
ts = sum(v[0] for v in agg.values()) or 1
ti = sum(v[1] for v in agg.values()) or 1
print(f"total samples {ts}, warp instructions {ti:.3e}")
for k, (s, i) in sorted(agg.items(), key=lambda kv: -kv[1][0]):
    print(f"{100*s/ts:5.1f}% samp {100*i/ti:5.1f}% inst ({i:.2e})  {k}")
