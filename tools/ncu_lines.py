"""Per-source-line hot spots of an ncu report (cuda,sass view): instructions
executed and stall samples, top N lines.

  python tools/ncu_lines.py gpurun_out/x.ncu-rep [N]
"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = []
fname = "?"
hdr = None
for r in csv.reader(io.StringIO(out)):
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or r[0] == "" or r[0] == "Function Name":
        continue
    d = dict(zip(hdr, r))
    try:
        samp = int(d.get("Warp Stall Sampling (All Samples)", "0") or 0)
        inst = int(d.get("Instructions Executed", "0") or 0)
    except ValueError:
        continue
    st = sorted(((int(d[k] or 0), k[6:]) for k in hdr
                 if k.startswith("stall_") and "Not Issued" not in k and (d.get(k) or "0").isdigit()),
                reverse=True)[:2]
    why = ",".join(f"{k}:{100*v/max(samp,1):.0f}%" for v, k in st if v)
    rows.append((samp, inst, fname, r[0], r[1][:70] + "  [" + why + "]"))
tot_s = sum(r[0] for r in rows) or 1
tot_i = sum(r[1] for r in rows) or 1
print(f"total samples {tot_s}, warp instructions {tot_i:.3e}")
for s, i, f, ln, src in sorted(rows, reverse=True)[:top]:
    print(f"{100*s/tot_s:5.1f}% samp {100*i/tot_i:5.1f}% inst  {f}:{ln}  {src}")
