"""Generate golden F_0..F_n vectors from the REFERENCE oracle.

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py [--procs 8]

Runs only in the build container (it imports boysfn.refmath from
/root/reference); the resulting .npz fixtures are committed and travel to the
GPU box.  Each value is refmath.boys_downward(n, x, Precision(96))
(refmath.py:330-341: an exact F_n seed plus the downward recursion at
96 + 24 bits), stored as a double-double (hi, lo) so the fixture itself adds
no rounding error at the 2^-53 level.

Fixtures
  scan_f64.npz / scan_f32.npz : Table-I style scans: an
        equally spaced grid on [0, z_nb) per order (z_{n,53} / z_{n,24}).
  configs.npz : stratified samples of the five BASELINE configurations,
        including their edge strata (zeros, cut-off neighbourhood), plus
        the ragged ERI-like batch (own order per element).
  edges.npz   : every order with the edge points (0, denormals, z +- 1 ulp,
        z (1 +- 1e-3), 708/86 and neighbours, x_up, very large x).
"""

from __future__ import annotations

import argparse
import math
import multiprocessing as mp_
import os
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
ROOT = HERE.parents[1]
REF = os.environ.get("BOYS_REFERENCE_SRC", "/root/reference/pkg/src")
sys.path.insert(0, REF)
sys.path.insert(0, str(ROOT))

PREC_BITS = 96


def _dd(v):
    from mpmath import mp
    hi = float(v)
    with mp.workprec(300):
        lo = float(v - mp.mpf(hi))
    return hi, lo


def _job(args):
    n, xs = args
    from boysfn import refmath as R
    out = np.empty((len(xs), n + 1, 2))
    for i, x in enumerate(xs):
        vals = R.boys_downward(n, float(x), R.Precision(PREC_BITS))
        for m, v in enumerate(vals):
            out[i, m] = _dd(v)
    return out


def run(pool, n, xs, chunk=64):
    xs = np.asarray(xs, dtype=np.float64)
    parts = [(n, xs[i:i + chunk]) for i in range(0, len(xs), chunk)]
    res = pool.map(_job, parts)
    return np.concatenate(res) if res else np.empty((0, n + 1, 2))


def load_ds(profile):
    from paper_2504_07637_b200 import coeffs as C
    return C.load_default(profile)


def edge_points(rec, dtype):
    fi = np.finfo(dtype)
    xexp = 86.0 if dtype == np.float32 else 708.0
    base = [0.0, fi.smallest_subnormal, fi.tiny, 1e-30, 1e-12, 1e-6, 1e-3, 0.5, 1.0, 2.0,
            rec.z, rec.x_up, xexp, 10.0, 20.0, 30.0, 50.0, 100.0, 1e3, 1e4, 1e6, 1e9, 1e15]
    out = []
    for v in base:
        v = dtype(v)
        out += [v, np.nextafter(v, dtype(np.inf)), np.nextafter(v, dtype(0))]
    for f in (1 - 1e-3, 1 - 1e-6, 1 + 1e-6, 1 + 1e-3):
        out.append(dtype(rec.z * f))
    return np.unique(np.array([v for v in out if v >= 0 and np.isfinite(v)], dtype=dtype))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--procs", type=int, default=os.cpu_count())
    ap.add_argument("--scan-points", type=int, default=2048)
    ap.add_argument("--config-points", type=int, default=2048)
    a = ap.parse_args()
    rng = np.random.default_rng(20250410)
    d64, d32 = load_ds("double53"), load_ds("single24")
    with mp_.Pool(a.procs) as pool:
        # ---- Table-I scans --------------------------------------------------
        for tag, ds, orders, dtype in (("f64", d64, (0, 2, 5, 8, 12, 16, 24, 36), np.float64),
                                       ("f32", d32, (0, 5, 8, 16), np.float32)):
            blob = {}
            for n in orders:
                z = ds.records[n].z
                xs = (np.arange(a.scan_points) * (z / a.scan_points)).astype(dtype)
                blob[f"x{n}"] = xs
                blob[f"F{n}"] = run(pool, n, xs)
                print(f"scan {tag} n={n} done", flush=True)
            np.savez_compressed(HERE / f"scan_{tag}.npz", **blob)
        # ---- configuration samples -----------------------------------------
        M = a.config_points
        q = M // 4

        def logu(k, lo, hi):
            return np.exp(rng.uniform(math.log(lo), math.log(hi), k))

        z16 = d64.records[16].z
        cfg = {
            "cfg1": (0, np.concatenate([np.zeros(q), rng.uniform(0, 1, q), rng.uniform(1, 40, q),
                                        logu(M - 3 * q, 1e-10, 1e4)])),
            "cfg2": (8, np.concatenate([rng.uniform(0, 30, M // 2), logu(M - M // 2, 1e-8, 1e4)])),
            "cfg3": (16, np.concatenate([logu(M - M // 5, 1e-12, 1e5),
                                         z16 * (1 + rng.uniform(-1e-3, 1e-3, M // 5))])),
            "cfg5": (12, logu(M, 1e-10, 1e4)),
        }
        blob = {}
        for name, (n, xs) in cfg.items():
            blob[f"{name}_x"] = xs
            blob[f"{name}_F"] = run(pool, n, xs)
            print(f"config {name} done", flush=True)
        # ragged ERI-like (cfg4): x = rho |P-Q|^2, n ~ 1/(n+1)
        K = M
        e = logu(4 * K, 0.05, 1e4).reshape(4, K)
        c = rng.uniform(0, 20, (4, 3, K))
        P = (e[0] * c[0] + e[1] * c[1]) / (e[0] + e[1])
        Qc = (e[2] * c[2] + e[3] * c[3]) / (e[2] + e[3])
        rho = (e[0] + e[1]) * (e[2] + e[3]) / e.sum(0)
        x4 = rho * ((P - Qc) ** 2).sum(0)
        w = np.array([1.0 / (k + 1) for k in range(13)])
        n4 = rng.choice(13, size=K, p=w / w.sum()).astype(np.uint8)
        vals = []
        for n in range(13):
            sel = np.nonzero(n4 == n)[0]
            r = run(pool, n, x4[sel])
            vals.append((sel, r))
        off = np.zeros(K + 1, dtype=np.int64)
        np.cumsum(n4.astype(np.int64) + 1, out=off[1:])
        flat = np.empty((off[-1], 2))
        for sel, r in vals:
            for j, i in enumerate(sel):
                flat[off[i]:off[i + 1]] = r[j]
        blob.update(cfg4_x=x4, cfg4_n=n4, cfg4_F=flat)
        # fp32 ragged subset (n <= 8), x rounded to fp32 first
        keep = np.nonzero(n4 <= 8)[0][: M // 2]
        x4f = x4[keep].astype(np.float32)
        n4f = n4[keep]
        offf = np.zeros(keep.size + 1, dtype=np.int64)
        np.cumsum(n4f.astype(np.int64) + 1, out=offf[1:])
        flatf = np.empty((offf[-1], 2))
        for n in range(9):
            sel = np.nonzero(n4f == n)[0]
            r = run(pool, n, x4f[sel].astype(np.float64))
            for j, i in enumerate(sel):
                flatf[offf[i]:offf[i + 1]] = r[j]
        blob.update(cfg4f32_x=x4f, cfg4f32_n=n4f, cfg4f32_F=flatf)
        print("config cfg4 done", flush=True)
        np.savez_compressed(HERE / "configs.npz", **blob)
        # ---- edges: every order ---------------------------------------------
        blob = {}
        for tag, ds, dtype in (("f64", d64, np.float64), ("f32", d32, np.float32)):
            for n in ds.orders():
                xs = edge_points(ds.records[n], dtype)
                blob[f"{tag}_x{n}"] = xs
                blob[f"{tag}_F{n}"] = run(pool, n, xs.astype(np.float64))
        np.savez_compressed(HERE / "edges.npz", **blob)
        print("edges done", flush=True)


if __name__ == "__main__":
    main()
