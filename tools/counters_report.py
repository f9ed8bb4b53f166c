"""Counters parity report: the engine's traversal counters next
to the reference DFS's (oracle port of summation_engine.py:291-428, whose
counters are pinned to the reference's own by tests/test_oracle_pins.py), per
config, bandwidth and algorithm, plus the max relative error of both against
the exhaustive sums.

  python tools/counters_report.py [--configs 1,2,3,4,5] > profiles/r02_counters.jsonl

Configs run at the scales of the sub_C* goldens (the DFS oracle must finish):
C1 full, C2 0.1, C3 0.05, C4 0.02, C5 0.005.  The engine counts (query block,
reference node) events: a visit is one frontier entry examined for one block
of <= 64 queries, a base case one (block, leaf item) evaluation -- the
reference counts node pairs of its own query tree.  exact_pairs / fp32_pairs
(engine) and the SPEC.md:571 token dominance (DFDO settles more by pruning
than DFD: fewer exactly evaluated pairs) are reported per row.
"""
import argparse
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

SCALES = {1: 1.0, 2: 0.1, 3: 0.05, 4: 0.02, 5: 0.005}
NAMES = ["pair_visits", "base_cases", "fd_prunes", "hermite_prunes", "local_prunes",
         "h2l_prunes"]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="1,2,3,4,5")
    args = ap.parse_args()
    import oracle
    import paper_1206_6857_b200 as fg
    from paper_1206_6857_b200.configs import config

    for k in [int(v) for v in args.configs.split(",")]:
        wl = config(k, scale=SCALES[k])
        qp = wl.query_points()
        rt = fg.build_tree(fg.PointStore(wl.references, wl.weights), 25)
        qt = rt if wl.monochromatic else fg.build_tree(fg.PointStore(wl.queries), 25)
        ort = oracle.Tree(wl.references, wl.weights, 25)
        oqt = ort if wl.monochromatic else oracle.Tree(wl.queries, None, 25)
        pl = fg.default_plimit(wl.dim)
        for h in wl.bandwidths:
            exact = fg.naive_sum(qp, wl.references, wl.weights, h).values
            rt.refresh_moments(h, pl)
            ort.refresh_moments(h, pl)
            row = {"config": wl.name, "scale": SCALES[k], "n": wl.n, "dim": wl.dim,
                   "h": h, "eps": wl.epsilon}
            for alg in ("dfd", "dfdo", "dito"):
                res = getattr(fg, f"{alg}_run")(fg.RunConfig(bandwidth=h, epsilon=wl.epsilon),
                                                qt, rt)
                t0 = time.perf_counter()
                ov, oc = oracle.run(alg, oqt, ort, h, wl.epsilon)
                ot = time.perf_counter() - t0
                c = res.counters
                row[alg] = {
                    "engine": {**c.as_dict(), "exact_pairs": c.exact_pairs,
                               "fp32_pairs": c.fp32_pairs, "hermite_evals": c.hermite_evals,
                               "err": float(oracle.max_rel_error(res.values, exact)),
                               "kernel_ms": 1e3 * res.seconds},
                    "reference_dfs": {**dict(zip(NAMES, (int(v) for v in oc))),
                                      "err": float(oracle.max_rel_error(ov, exact)),
                                      "cpu_ms_1thread": 1e3 * ot},
                }
            e = {a: row[a]["engine"]["exact_pairs"] + row[a]["engine"]["fp32_pairs"]
                 for a in ("dfd", "dfdo")}
            row["dfdo_le_dfd_exact_pairs"] = e["dfdo"] <= e["dfd"]
            row["reference_dfdo_ge_dfd_prunes"] = (row["dfdo"]["reference_dfs"]["fd_prunes"] >=
                                                  row["dfd"]["reference_dfs"]["fd_prunes"])
            print(json.dumps(row), flush=True)


if __name__ == "__main__":
    main()
