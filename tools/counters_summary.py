"""Tabulate tools/counters_report.py's JSONL (one row per config, bandwidth and
algorithm) and the SPEC.md:571 dominance counts.

  python tools/counters_summary.py profiles/r02_counters.jsonl > profiles/r02_counters_summary.txt
"""
import json
import sys

rows = [json.loads(l) for l in open(sys.argv[1]) if l.startswith("{")]
N = ["pair_visits", "base_cases", "fd_prunes", "hermite_prunes", "local_prunes", "h2l_prunes"]
print("# Counters parity (SURVEY 8(f)3): tools/counters_report.py on GPU + the oracle's DFS (pinned to the")
print(f"# reference's counters by tests/test_oracle_pins.py), {len(rows)} (config, bandwidth) rows, configs at the sub_C* scales.")
print("# Engine units: (query block <= 64 pts, reference node) events; reference units: (query node, reference node) pairs.")
print("# The engine's DITO rows run at its own series order cap (12 at D = 3); the reference's at default_plimit.")
print("config  scale  h          alg   | engine visits  base  fd  dh  dl  h2l  err   | reference visits  base  fd  dh  dl  h2l  err")
dom = {k: [0, 0] for k in ("visits", "base", "pairs")}
lit = [0, 0]
worst = [0.0, 0.0]
for r in rows:
    for alg in ("dfd", "dfdo", "dito"):
        e, f = r[alg]["engine"], r[alg]["reference_dfs"]
        print(f"{r['config']:4s} {r['scale']:6.3f} {r['h']:10.4g} {alg:5s} | " +
              " ".join(f"{e[k]:8d}" for k in N[:3]) + " " + " ".join(f"{e[k]:7d}" for k in N[3:4]) +
              " " + " ".join(f"{e[k]:4d}" for k in N[4:]) + f" {e['err']:.1e} | " +
              " ".join(f"{f[k]:9d}" for k in N[:3]) + " " + " ".join(f"{f[k]:7d}" for k in N[3:5]) +
              f" {f[N[5]]:4d} {f['err']:.1e}")
        worst[0] = max(worst[0], e["err"] / r["eps"])
        worst[1] = max(worst[1], f["err"] / r["eps"])
    a, b = r["dfd"], r["dfdo"]
    dom["visits"][0] += b["engine"]["pair_visits"] <= a["engine"]["pair_visits"]
    dom["visits"][1] += b["reference_dfs"]["pair_visits"] <= a["reference_dfs"]["pair_visits"]
    dom["base"][0] += b["engine"]["base_cases"] <= a["engine"]["base_cases"]
    dom["base"][1] += b["reference_dfs"]["base_cases"] <= a["reference_dfs"]["base_cases"]
    dom["pairs"][0] += (b["engine"]["exact_pairs"] + b["engine"]["fp32_pairs"]
                        <= a["engine"]["exact_pairs"] + a["engine"]["fp32_pairs"])
    lit[0] += b["engine"]["fd_prunes"] >= a["engine"]["fd_prunes"]
    lit[1] += b["reference_dfs"]["fd_prunes"] >= a["reference_dfs"]["fd_prunes"]
n = len(rows)
print(f"# DFDO <= DFD: visits engine {dom['visits'][0]}/{n} reference {dom['visits'][1]}/{n}; base cases engine "
      f"{dom['base'][0]}/{n} reference {dom['base'][1]}/{n}; exact+fp32 pairs engine {dom['pairs'][0]}/{n}")
print(f"# DFDO fd prunes >= DFD (SPEC.md:571 literal): engine {lit[0]}/{n}, reference {lit[1]}/{n}")
print(f"# max err/eps: engine {worst[0]:.3f}, reference {worst[1]:.3f}")
