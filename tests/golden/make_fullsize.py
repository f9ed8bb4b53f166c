"""Full-size parity fixtures for BASELINE.json configs 2-5 (SURVEY 8(c),
BASELINE.md section 3), made by the CPU oracle (oracle/fg_oracle.c, pinned to
the unmodified reference by tests/test_oracle_pins.py):

  * ``naive``: exact FP64 sums (naive_sum, summation_engine.py:122-154) of a
    seeded query subsample of M' rows against ALL N reference points, at every
    bandwidth of the config, accumulated with Neumaier compensation (a plain
    sequential sum of 4e6 terms carries ~1e-12 of its own rounding, the size
    of the tolerance being tested);
  * ``dito``: the reference's depth-first DITO (summation_engine.py:431-480)
    on the same subsample, bichromatic against the full reference tree (the
    per-query sums equal the monochromatic problem's).

M' = 1024 for every config (the naive leg at C5 is 1024 x 4e6 x 16 pairs).
Run in the build container (minutes, all host threads):

    python tests/golden/make_fullsize.py [--configs 2,3,4,5]

Writes tests/golden/full_C{k}.npz: idx (M'), hs, naive (nh x M'), dito
(nh x M').  No GPU test reads /root/reference or runs the oracle at this size.
"""

import argparse
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(HERE, "..", ".."))

import oracle  # noqa: E402
from paper_1206_6857_b200.configs import config  # noqa: E402

SAMPLE = 1024
SEED = 4242  # the same subsample rule as bench.py's CPU leg
PLIMIT = {1: 8, 2: 8, 3: 6, 4: 4, 5: 4, 6: 2}


def subsample(m, k, seed=SEED):
    return np.sort(np.random.default_rng(seed).choice(m, min(k, m), replace=False))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="2,3,4,5")
    ap.add_argument("--threads", type=int, default=os.cpu_count() or 1)
    args = ap.parse_args()
    for k in [int(v) for v in args.configs.split(",")]:
        t0 = time.time()
        wl = config(k)
        idx = subsample(wl.m, SAMPLE)
        qs = np.ascontiguousarray(wl.query_points()[idx])
        hs = np.array(wl.bandwidths)
        naive = np.stack([oracle.naive_sum(qs, wl.references, wl.weights, h,
                                           threads=args.threads, compensated=True) for h in hs])
        t1 = time.time()
        rt = oracle.Tree(wl.references, wl.weights, 25)
        dito = []
        for h in hs:
            rt.refresh_moments(h, PLIMIT.get(wl.dim, 1))
            v, _ = oracle.run_sharded("dito", qs, rt, h, wl.epsilon, threads=args.threads)
            dito.append(v)
        dito = np.stack(dito)
        err = np.max(np.abs(dito - naive) / naive)
        np.savez_compressed(os.path.join(HERE, f"full_C{k}.npz"), idx=idx, hs=hs, naive=naive,
                            dito=dito, epsilon=wl.epsilon)
        print(f"C{k}: naive {t1 - t0:.1f} s, dito {time.time() - t1:.1f} s, "
              f"oracle dito max rel err {err:.3e} (eps {wl.epsilon})", flush=True)


if __name__ == "__main__":
    main()
