"""The reference's own CPU path, timed in the build container (it cannot run on
the GPU box: /root/reference is not shipped there).  refmath.boys_downward(n, x,
Precision(64)) over a seeded sample of a BASELINE config, one process per
core (the mpmath context is process-global), values/s = sum(n+1) / wall time.

Usage: python tools/ref_mpmath_rate.py [cfg3] [seconds]  -> one JSON line."""
import json
import multiprocessing as mp
import os
import platform
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = "/root/reference/pkg/src"


def _work(args):
    n, xs, deadline = args
    sys.path.insert(0, REF)
    from boysfn import refmath as R
    done = 0
    for x in xs:
        R.boys_downward(n, float(x), R.Precision(64))
        done += 1
        if time.time() > deadline:
            break
    return done


def main():
    cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg3"
    secs = float(sys.argv[2]) if len(sys.argv) > 2 else 20.0
    sys.path.insert(0, ROOT)
    from paper_2504_07637_b200 import workloads as W
    c = W.CONFIGS[cfg]
    x = W.config_x(cfg, n=1 << 18).numpy()
    procs = os.cpu_count()
    parts = [x[k::procs] for k in range(procs)]
    t0 = time.time()
    with mp.Pool(procs) as pool:
        done = sum(pool.map(_work, [(c.n_max, p, t0 + secs) for p in parts]))
    el = time.time() - t0
    print(json.dumps({"impl": "reference (refmath.boys_downward, mpmath, Precision(64))",
                      "config": cfg, "points": done, "seconds": round(el, 2),
                      "points_per_s": done / el, "values_per_s": done * (c.n_max + 1) / el,
                      "processes": procs, "host": platform.processor() or platform.machine(),
                      "where": "build container (no GPU); the GPU box cannot run the reference"}))


if __name__ == "__main__":
    main()
