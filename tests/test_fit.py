"""The offline fitter (tablegen/fit.py) and SPEC acceptance
criteria 4, 8 and 9.

The fitter samples Q_n from the reference oracle (refmath), so these tests
need /root/reference and are skipped without it (the GPU box has no copy;
they are CPU tests, run in the build container).  The fits here are small
(n = 0, N = 4, single profile, short grids) to keep the CPU suite fast; the
shipped tables come from tablegen/run_fits.py at full settings.
"""

import copy
import math
import os
import sys
from pathlib import Path

import numpy as np
import pytest

REF = Path(os.environ.get("BOYS_REFERENCE_SRC", "/root/reference/pkg/src"))
pytestmark = pytest.mark.skipif(not (REF / "boysfn").exists(), reason="reference not present")

ROOT = Path(__file__).resolve().parents[1]


@pytest.fixture(scope="module")
def F():
    sys.path.insert(0, str(ROOT / "tablegen"))
    import fit
    return fit


@pytest.fixture(scope="module")
def R():
    if str(REF) not in sys.path:
        sys.path.insert(0, str(REF))
    from boysfn import refmath
    return refmath


def _small_fit(F):
    # SPEC.md:162 example (n=0, N=4): exact_error_bits >= 25 (paper 27.3)
    return F.fit(0, 4, 24, m_nodes=60, lawson_iters=25, exchange_rounds=1, grid=240)


@pytest.fixture(scope="module")
def small(F):
    return _small_fit(F)


def test_fit_quality_single_profile_n0(small):
    """Acceptance 4 (n=0, N=4): >= 25 bits, paper 27.3 (Table I)."""
    assert small.exact_bits >= 25.0
    assert small.v[0] > 0                                # B_N > 0
    assert 2 * len(small.u_quads) + len(small.u_lins) == 3
    assert 2 * len(small.v_quads) + len(small.v_lins) == 4


def test_fit_is_deterministic(F, small):
    """same inputs, same precision -> bit-identical solution."""
    again = _small_fit(F)
    assert again.u == small.u and again.v == small.v     # mpf equality, every coefficient
    assert again.u_quads == small.u_quads and again.v_quads == small.v_quads
    assert again.u_lins == small.u_lins and again.v_lins == small.v_lins
    assert again.exact_bits == small.exact_bits


def test_validate_accepts_the_fit(F, small):
    assert F.validate(copy.deepcopy(small), rescan=0) == []


def test_validate_rejects_corrupted_B_N(F, small):
    """a hand-corrupted B_N sign is rejected, naming the
    section III rule."""
    bad = copy.deepcopy(small)
    bad.v = list(bad.v)
    bad.v[0] = -bad.v[0]
    msgs = F.validate(bad, rescan=0)
    assert any("B_N" in m and "PAPER.md:163-164" in m for m in msgs), msgs


def test_validate_rejects_poles_and_bad_factors(F, small):
    from mpmath import mp
    pole = copy.deepcopy(small)
    pole.v_lins = [mp.mpf("1.5")] + list(pole.v_lins)        # a real root of v at x = 1.5
    assert any("pole" in m for m in F.validate(pole, rescan=0))
    neg = copy.deepcopy(small)
    y, a = neg.u_quads[0]
    neg.u_quads = [(y, -a)] + list(neg.u_quads[1:])
    assert any("a <= 0" in m for m in F.validate(neg, rescan=0))
    deg = copy.deepcopy(small)
    deg.v_quads = list(deg.v_quads) + [(mp.mpf(-3), mp.mpf(2))]
    assert any("degree(v)" in m for m in F.validate(deg, rescan=0))


def test_validate_rescan_and_grid_drift(F, small):
    """exact bits re-derived on a fresh denser grid; a
    recorded value more than 0.5 bit above it is flagged as under-resolved."""
    ok = copy.deepcopy(small)
    assert F.validate(ok, rescan=2) == []
    assert abs(ok.rescan_bits - ok.exact_bits) <= 0.5
    drift = copy.deepcopy(small)
    drift.exact_bits += 3.0
    assert any("grid-refinement drift" in m for m in F.validate(drift, rescan=2))


def test_factorize_round_trip(F, small):
    """factored vs coefficient form agree far beyond double."""
    from mpmath import mp
    with mp.workprec(F.FIT_BITS):
        for poly, (quads, lins) in ((small.u, (small.u_quads, small.u_lins)),
                                    (small.v, (small.v_quads, small.v_lins))):
            back = F.expand(quads, lins)
            for x in (mp.mpf(0), mp.mpf("0.5"), small.z / 3, small.z):
                a, b = F._polyval(back, x), F._polyval(poly, x)
                assert abs(a - b) <= abs(b) * mp.mpf(2) ** -200


def _factored_q(r, x):
    """Q~ from the stored root-factored form in IEEE double (Eqs. 12-14)."""
    u = np.ones_like(x)
    for y, a in r.u_quads:
        d = x - y
        u = u * (d * d + a)
    for y in r.u_lins:
        u = u * (x - y)
    v = np.ones_like(x)
    for y, b in r.v_quads:
        d = x - y
        v = v * (d * d + b)
    for y in r.v_lins:
        v = v * (x - y)
    return r.q0 + x * (r.q1 + x * (r.q2 * (u / v)))


def _raw_q(r, x):
    """Q~ from expanded (raw) polynomial coefficients, Horner in IEEE double
    (the coefficient form of Eq. 11 the factored form replaces)."""
    from mpmath import mp
    sys.path.insert(0, str(ROOT / "tablegen"))
    import fit
    with mp.workprec(256):
        uq = [(mp.mpf(y), mp.mpf(a)) for y, a in r.u_quads]
        vq = [(mp.mpf(y), mp.mpf(b)) for y, b in r.v_quads]
        uc = [float(c) for c in fit.expand(uq, [mp.mpf(y) for y in r.u_lins])]
        vc = [float(c) for c in fit.expand(vq, [mp.mpf(y) for y in r.v_lins])]
    u = np.zeros_like(x)
    for c in reversed(uc):
        u = u * x + c
    v = np.zeros_like(x)
    for c in reversed(vc):
        v = v * x + c
    return r.q0 + x * (r.q1 + x * (r.q2 * (u / v)))


def _exact_q(r, x):
    """The same stored rational evaluated in 256-bit arithmetic."""
    from mpmath import mp
    out = []
    with mp.workprec(256):
        for xi in x:
            X = mp.mpf(float(xi))
            u = mp.mpf(1)
            for y, a in r.u_quads:
                u *= (X - y) ** 2 + a
            for y in r.u_lins:
                u *= X - y
            v = mp.mpf(1)
            for y, b in r.v_quads:
                v *= (X - y) ** 2 + b
            for y in r.v_lins:
                v *= X - y
            out.append(r.q0 + X * (r.q1 + X * (r.q2 * (u / v))))
    return out


def test_root_factored_necessity():
    """Acceptance 8: for the largest fitted n (36 here), double
    evaluation through raw coefficients loses >= 4 more bits than the
    factored form on the same grid, measured on the half-integer power
    F ~ Q^-(n+1/2) (the quantity the tables feed; section III)."""
    from mpmath import mp
    from paper_2504_07637_b200 import coeffs as C
    ds = C.load_default("double53")
    n = max(ds.orders())
    assert n >= 8
    r = ds.records[n]
    x = np.linspace(0.0, r.z, 401)[1:-1]
    ex = _exact_q(r, x)
    p = n + 0.5

    def bits(q):
        with mp.workprec(256):
            worst = max(abs(mp.power(mp.mpf(float(a)) / e, p) - 1) for a, e in zip(q, ex))
        return float(-mp.log(worst, 2))

    fac, raw = bits(_factored_q(r, x)), bits(_raw_q(r, x))
    assert fac >= raw + 4.0, (n, fac, raw)


def test_cutoff_correctness(R):
    """Acceptance 9: for every tabulated (n, b), the asymptote
    c_n x^-(n+1/2) is within 2^-b of F_n just above z_nb and not just below."""
    from mpmath import mp
    from paper_2504_07637_b200 import coeffs as C
    prec = R.Precision(128)
    for profile in ("double53", "single24"):
        ds = C.load_default(profile)
        b = ds.bits
        for n, r in ds.records.items():
            cn = R.c_n(n, prec)

            def rel(x):
                with mp.workprec(160):
                    X = mp.mpf(x)
                    return abs(cn * X ** -(mp.mpf(2 * n + 1) / 2) / R.boys_ref(n, X, prec) - 1)

            above, below = rel(r.z * (1 + 1e-6)), rel(r.z * (1 - 1e-3))
            assert above <= mp.mpf(2) ** -b, (profile, n, float(above))
            assert below > mp.mpf(2) ** -b, (profile, n, float(below))
