"""Fit every order the kernels need and write the coefficient datasets.

    python tablegen/run_fits.py [--procs 8] [--double 0-16] [--single 0-8]

Build-time only (needs /root/reference for the oracle).  Outputs:

* ``tablegen/solutions_hp.json``  -- fit-precision values (60 significant digits)
* ``paper_2504_07637_b200/data/boys_{double53,single24}.dat`` -- rounded once
* ``paper_2504_07637_b200/csrc/boys_tables.inc``             -- generated header

N per order follows Table I.
"""

from __future__ import annotations

import argparse
import json
import math
import multiprocessing as mp_
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tablegen"))

# Table I denominator degrees N (blank cells repeat the row above)
N_DOUBLE = {0: 10, 1: 10, 2: 11, 3: 11, 4: 11, 5: 11, 6: 11, 7: 12, 8: 12, 9: 12, 10: 12}
N_DOUBLE.update({n: 13 for n in range(11, 18)})
N_DOUBLE.update({n: 14 for n in range(18, 37)})
N_SINGLE = {0: 4, 1: 4}
N_SINGLE.update({n: 5 for n in range(2, 10)})
N_SINGLE.update({n: 6 for n in range(10, 37)})

HP_JSON = ROOT / "tablegen" / "solutions_hp.json"
UNDERFLOW_BITS = {53: 1000, 24: 120}


def _job(args):
    n, N, b = args
    import fit as F
    from mpmath import mp
    t0 = time.time()
    r = F.fit(n, N, b)
    bad = F.validate(r)
    s = lambda v: mp.nstr(v, 60, strip_zeros=False)
    return dict(
        n=n, N=N, bits=b, exact_bits=r.exact_bits, argmax=r.argmax, violations=bad,
        seconds=time.time() - t0,
        c=s(r.consts.c), q0=s(r.consts.q0), q1=s(r.consts.q1),
        q2=s(r.consts.alpha - r.consts.q1), alpha=s(r.consts.alpha), beta=s(r.consts.beta),
        z=s(r.z),
        u_quads=[[s(y), s(a)] for y, a in r.u_quads], u_lins=[s(y) for y in r.u_lins],
        v_quads=[[s(y), s(a)] for y, a in r.v_quads], v_lins=[s(y) for y in r.v_lins],
    )


def _round(dec: str, bits: int) -> float:
    """Round a decimal string ONCE to binary64 / binary32 (round-to-nearest-even)."""
    from mpmath import mp, mpf
    with mp.workprec(400):
        v = mpf(dec)
    if bits == 53:
        with mp.workprec(53):
            return float(+v)
    with mp.workprec(24):
        f = float(+v)          # exact: a 24-bit value is representable in binary64
    from paper_2504_07637_b200.coeffs import to_f32
    return to_f32(f)


def build_dataset(sols, profile):
    from paper_2504_07637_b200.coeffs import Dataset, Record
    bits = 53 if profile == "double53" else 24
    ds = Dataset(profile=profile)
    for s in sols:
        if s["bits"] != bits:
            continue
        n = s["n"]
        R = lambda v: _round(v, bits)
        x_up = 2.0 ** min(60, math.floor(UNDERFLOW_BITS[bits] / (n + 0.5)))
        ds.records[n] = Record(
            n=n, N=s["N"], c=R(s["c"]), q0=R(s["q0"]), q1=R(s["q1"]), q2=R(s["q2"]),
            alpha=R(s["alpha"]), beta=R(s["beta"]), z=R(s["z"]), x_up=x_up,
            u_quads=[(R(y), R(a)) for y, a in s["u_quads"]], u_lins=[R(y) for y in s["u_lins"]],
            v_quads=[(R(y), R(a)) for y, a in s["v_quads"]], v_lins=[R(y) for y in s["v_lins"]],
            exact_bits=round(s["exact_bits"], 3))
    return ds


def _parse_range(s):
    if not s:
        return []
    a, _, b = s.partition("-")
    return list(range(int(a), int(b or a) + 1))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--procs", type=int, default=8)
    ap.add_argument("--double", default="0-16")
    ap.add_argument("--single", default="0-8")
    ap.add_argument("--regen-only", action="store_true",
                    help="skip fitting; rebuild datasets/header from solutions_hp.json")
    a = ap.parse_args()
    old = json.loads(HP_JSON.read_text()) if HP_JSON.exists() else []
    if not a.regen_only:
        jobs = [(n, N_DOUBLE[n], 53) for n in _parse_range(a.double)]
        jobs += [(n, N_SINGLE[n], 24) for n in _parse_range(a.single)]
        jobs.sort(key=lambda j: -j[1] * (1 + j[0] / 8))   # longest first
        with mp_.Pool(a.procs) as pool:
            new = []
            for r in pool.imap_unordered(_job, jobs):
                print(f"n={r['n']:2d} N={r['N']:2d} b={r['bits']}: {r['exact_bits']:.2f} bits "
                      f"({r['seconds']:.0f}s) {r['violations'] or 'ok'}", flush=True)
                new.append(r)
        keep = {(s["n"], s["bits"]): s for s in old}
        for s in new:
            keep[(s["n"], s["bits"])] = s
        sols = sorted(keep.values(), key=lambda s: (s["bits"], s["n"]))
        HP_JSON.write_text(json.dumps(sols, indent=1) + "\n")
    else:
        sols = old
    bad = [s for s in sols if s["violations"]]
    if bad:
        raise SystemExit(f"rejected fits: {[(s['n'], s['bits'], s['violations']) for s in bad]}")
    from paper_2504_07637_b200 import coeffs as C
    tables = []
    for prof in ("double53", "single24"):
        ds = build_dataset(sols, prof)
        C.save(ds, C.default_path(prof))
        assert C.load(C.default_path(prof)) == ds
        tables.append(C.build_kernel_table(ds))
    hdr = ROOT / "paper_2504_07637_b200" / "csrc" / "boys_tables.inc"
    hdr.write_text(C.gen_header(tables))
    print("wrote", [str(C.default_path(p)) for p in ("double53", "single24")], hdr)


if __name__ == "__main__":
    main()
