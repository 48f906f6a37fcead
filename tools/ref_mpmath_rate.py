"""The reference's own CPU path, timed in the build container (it cannot run on
the GPU box: /root/reference is not shipped there).  refmath.boys_downward(n, x,
Precision(64)) over a seeded sample of a BASELINE config, one process per
core (the mpmath context is process-global), values/s = sum(n+1) / wall time.

Usage: python tools/ref_mpmath_rate.py [cfg3] [seconds] [points]  -> one JSON line."""
import json
import multiprocessing as mp
import os
import platform
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = "/root/reference/pkg/src"


def _work(args):
    ns, xs, deadline = args
    sys.path.insert(0, REF)
    from boysfn import refmath as R
    done = vals = 0
    for n, x in zip(ns, xs):
        R.boys_downward(int(n), float(x), R.Precision(64))
        done += 1
        vals += int(n) + 1
        if time.time() > deadline:
            break
    return done, vals


def main():
    cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg3"
    secs = float(sys.argv[2]) if len(sys.argv) > 2 else 20.0
    sys.path.insert(0, ROOT)
    from paper_2504_07637_b200 import workloads as W
    c = W.CONFIGS[cfg]
    npts = int(sys.argv[3]) if len(sys.argv) > 3 else 1 << 18
    if c.layout == "ragged":
        x, nm = W.cfg4_batch(npts, chunk=0)
        x, nm = x.numpy(), nm.numpy()
    else:
        x = W.config_x(cfg, n=npts).numpy()
        nm = np.full(x.size, c.n_max)
    procs = os.cpu_count()
    parts = [(nm[k::procs], x[k::procs]) for k in range(procs)]
    t0 = time.time()
    with mp.Pool(procs) as pool:
        res = pool.map(_work, [(a, b, t0 + secs) for a, b in parts])
    el = time.time() - t0
    done = sum(r[0] for r in res)
    vals = sum(r[1] for r in res)
    print(json.dumps({"impl": "reference (refmath.boys_downward, mpmath, Precision(64))",
                      "config": cfg, "points": done, "seconds": round(el, 2),
                      "points_per_s": done / el, "values_per_s": vals / el,
                      "processes": procs, "host": platform.processor() or platform.machine(),
                      "where": "build container (no GPU); the GPU box cannot run the reference"}))


if __name__ == "__main__":
    main()
