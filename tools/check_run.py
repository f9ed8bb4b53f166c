"""Run the engine's workloads under a -DFG_CHECKS=1 build and report device
bounds-check violations (compute-sanitizer is not available on the GPU pool).

  tools/build_variant.sh HEAD checks EXTRA=-DFG_CHECKS=1
  FG_LIB=variants/checks.so python tools/check_run.py
Exits 1 if any check failed or any run broke its eps contract.
"""
import os
import sys
import threading

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import paper_1206_6857_b200 as fg
    from paper_1206_6857_b200 import _lib
    from paper_1206_6857_b200.configs import config
    import ctypes

    def failures():
        c = ctypes.c_int64()
        _lib.call("fg_check_failures", ctypes.byref(c))
        return c.value

    if failures() < 0:
        print("library built without FG_CHECKS")
        sys.exit(2)
    bad = 0

    def run_case(name, pts, w, hs, eps, algos=("dfd", "dfdo", "dito")):
        nonlocal bad
        tree = fg.build_tree(fg.PointStore(pts, w), 25)
        ex = fg.naive_sum(pts[:300], pts, w if w is not None else np.ones(len(pts)), hs).values
        worst = 0.0
        for alg in algos:
            res = fg.sweep_run(fg.RunConfig(bandwidth=hs[0], epsilon=eps, algorithm=alg), tree,
                               tree, hs)
            for j in range(len(hs)):
                worst = max(worst, float(np.max(np.abs(res[j].values[:300] - ex[j]) / ex[j])))
        f = failures()
        ok = f == 0 and worst <= eps
        bad += not ok
        print(f"{name}: check failures {f}, max rel err {worst:.3e} (eps {eps}) {'ok' if ok else 'FAIL'}",
              flush=True)

    rng = np.random.default_rng(9)
    for D in range(1, 9):
        pts = np.concatenate([rng.normal(0.5, 0.05, (3000, D)), rng.random((3000, D))])
        w = rng.uniform(0.5, 1.5, 6000)
        for fp32 in (1, 0):
            _lib.call("fg_set_engine_params", 0, 0, fp32)
            run_case(f"D={D} fp32={fp32}", pts, w, [0.01, 0.05, 0.3, 2.0], 0.01)
        _lib.call("fg_set_engine_params", 0, 0, 1)
        run_case(f"D={D} eps=1e-3", pts, w, [0.02, 0.2], 0.001)
    for k, sc in ((1, 1.0), (2, 0.3), (3, 0.1), (4, 0.02), (5, 0.05)):
        wl = config(k, scale=sc)
        if wl.monochromatic:
            run_case(f"C{k} x{sc}", wl.references, wl.weights, list(wl.bandwidths), wl.epsilon,
                     algos=("dito",))
    os.environ["FG_FAR"] = "1"
    wl = config(5, scale=0.05)
    run_case("C5 x0.05 far pass", wl.references, wl.weights, list(wl.bandwidths), wl.epsilon,
             algos=("dfdo", "dito"))
    del os.environ["FG_FAR"]
    # duplicates, a single point, identical points
    run_case("duplicates", np.repeat(rng.random((50, 3)), 40, axis=0), None, [0.01, 0.1], 0.01)
    run_case("identical", np.tile([0.2, 0.4, 0.6], (500, 1)), None, [0.1], 0.01)
    # two host threads on distinct trees
    outs = []

    def worker(seed):
        r = np.random.default_rng(seed)
        p = r.random((20000, 3))
        t = fg.build_tree(fg.PointStore(p), 25)
        outs.append(fg.sweep_run(fg.RunConfig(bandwidth=0.05), t, t, [0.02, 0.05, 0.2]))

    ths = [threading.Thread(target=worker, args=(s,)) for s in (1, 2)]
    [t.start() for t in ths]
    [t.join() for t in ths]
    f = failures()
    bad += f != 0
    print(f"two threads: check failures {f}")
    print("ALL OK" if not bad else f"{bad} FAILED")
    sys.exit(1 if bad else 0)


if __name__ == "__main__":
    main()
