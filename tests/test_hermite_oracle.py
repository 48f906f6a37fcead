"""The fused consumer's CPU restatement (oracle boys_oracle_hermite, the
checker of tests/test_gpu_hermite.py) against an independent high-precision
evaluation: the same McMurchie-Davidson recurrences in 160-bit arithmetic with
F_n(x) from the reference oracle (refmath.boys_ref).  Needs /root/reference."""

import os
import sys
from pathlib import Path

import numpy as np
import pytest

REF = Path(os.environ.get("BOYS_REFERENCE_SRC", "/root/reference/pkg/src"))
pytestmark = pytest.mark.skipif(not (REF / "boysfn").exists(), reason="reference not present")


def _exact(L, b, k):
    if str(REF) not in sys.path:
        sys.path.insert(0, str(REF))
    from boysfn import refmath as R
    from mpmath import mp, mpf, pi, sqrt
    with mp.workprec(160):
        p, q = mpf(b[0]), mpf(k[0])
        X, Y, Z = (mpf(b[i]) - mpf(k[i]) for i in (1, 2, 3))
        a = p * q / (p + q)
        x = a * (X * X + Y * Y + Z * Z)
        F = [R.boys_ref(n, x, R.Precision(160)) for n in range(L + 1)]
        Rn = {}
        for n in range(L + 1):
            Rn[(n, 0, 0, 0)] = (-2 * a) ** n * F[n]

        def r(n, t, u, v):
            if min(t, u, v) < 0:
                return mpf(0)
            key = (n, t, u, v)
            if key not in Rn:
                if t > 0:
                    Rn[key] = (t - 1) * r(n + 1, t - 2, u, v) + X * r(n + 1, t - 1, u, v)
                elif u > 0:
                    Rn[key] = (u - 1) * r(n + 1, t, u - 2, v) + Y * r(n + 1, t, u - 1, v)
                else:
                    Rn[key] = (v - 1) * r(n + 1, t, u, v - 2) + Z * r(n + 1, t, u, v - 1)
            return Rn[key]

        pref = 2 * pi ** mpf(2.5) / (p * q * sqrt(p + q)) * mpf(b[4]) * mpf(k[4])
        out = []
        for s in range(L + 1):
            for t in range(s, -1, -1):
                for u in range(s - t, -1, -1):
                    out.append(pref * r(0, t, u, s - t - u))
        return [float(v) for v in out]


@pytest.mark.parametrize("L", [0, 2, 4])
def test_oracle_hermite_matches_high_precision(L):
    sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
    from oracle import oracle as O
    from paper_2504_07637_b200 import workloads as W
    bra, ket = W.shell_pairs(6, seed=11).numpy(), W.shell_pairs(5, seed=12).numpy()
    got, bad = O.hermite(L, bra, ket)
    assert bad == -1
    for i in range(bra.shape[0]):
        for j in range(ket.shape[0]):
            ex = np.array(_exact(L, bra[i], ket[j]))
            scale = np.abs(ex).max()
            # Table I bound on F (~2^-44 relative at these orders) carried through
            # the recurrences, relative to the quartet's largest integral
            assert np.abs(got[i, j] - ex).max() <= 2.0 ** -40 * scale, (L, i, j)
