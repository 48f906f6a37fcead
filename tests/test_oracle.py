"""Pin the CPU oracle (oracle/boys_oracle.c) before trusting it.

1. Against golden vectors from the reference oracle refmath.boys_downward at
   Precision(96) (tests/golden/make_golden.py): per-(n, m) accuracy >= the
   paper's Table I finite-precision figure minus 2 bits.
2. Against the SPEC's known-answer examples.
3. Properties: positivity/ordering, recursion consistency, recursion
   improvement (acceptance 7).
"""

import math

import numpy as np
import pytest

import accuracy as A

C0 = math.sqrt(math.pi) / 2


def _cn(n):
    return math.factorial(2 * n) * math.sqrt(math.pi) / (math.factorial(n) * 2 ** (2 * n + 1))


@pytest.mark.parametrize("tag,dtype", [("f64", np.float64), ("f32", np.float32)])
def test_table1_scans(oracle, tag, dtype):
    d = A.load(f"scan_{tag}.npz")
    orders = sorted(int(k[1:]) for k in d.files if k.startswith("x"))
    for n in orders:
        x = d[f"x{n}"].astype(dtype)
        gold = d[f"F{n}"]                       # [M, n+1, 2]
        got, bad = oracle.dense(n, x, "aos")
        assert bad == -1
        per_m = [A.bits(A.rel_err(got[:, m], gold[:, m], dtype)) for m in range(n + 1)]
        for m, b in enumerate(per_m):
            assert b >= A.bar(n, m, dtype), f"{tag} n={n} m={m}: {b:.2f} bits < {A.bar(n, m, dtype)}"
        # acceptance 7: the recursion recovers accuracy (eps_0 >= eps_n - 1)
        assert per_m[0] >= per_m[n] - 1


@pytest.mark.parametrize("name,n", [("cfg1", 0), ("cfg2", 8), ("cfg3", 16), ("cfg5", 12)])
def test_config_samples(oracle, name, n):
    d = A.load("configs.npz")
    x, gold = d[f"{name}_x"], d[f"{name}_F"]
    got, bad = oracle.dense(n, x, "aos")
    assert bad == -1
    ok = A.representable(gold, np.float64)
    for m in range(n + 1):
        r = A.rel_err(got[:, m], gold[:, m])[ok[:, m]]
        assert A.bits(r) >= A.bar(n, m, np.float64), f"{name} F_{m}"


@pytest.mark.parametrize("tag,dtype", [("cfg4", np.float64), ("cfg4f32", np.float32)])
def test_ragged_sample(oracle, tag, dtype):
    d = A.load("configs.npz")
    x, nm, gold = d[f"{tag}_x"].astype(dtype), d[f"{tag}_n"], d[f"{tag}_F"]
    got, off, bad = oracle.ragged(x, nm)
    assert bad == -1 and off[-1] == gold.shape[0]
    r = A.rel_err(got, gold, dtype)
    for i in range(x.size):
        n = int(nm[i])
        for m in range(n + 1):
            k = off[i] + m
            if dtype == np.float64 and abs(gold[k, 0]) < np.finfo(np.float64).tiny:
                continue
            b = A.bits(r[k:k + 1])
            assert b >= A.bar(n, m, dtype), f"elem {i} n={n} m={m} x={x[i]}: {b:.2f}"


@pytest.mark.parametrize("tag,dtype", [("f64", np.float64), ("f32", np.float32)])
def test_edges_every_order(oracle, tag, dtype):
    d = A.load("edges.npz")
    n = 0
    while f"{tag}_x{n}" in d.files:
        x, gold = d[f"{tag}_x{n}"].astype(dtype), d[f"{tag}_F{n}"]
        got, bad = oracle.dense(n, x, "aos")
        assert bad == -1
        r = A.rel_err(got, gold, dtype)
        if dtype == np.float64:
            r = np.where(A.representable(gold, np.float64), r, 0.0)
        for m in range(n + 1):
            b = A.bits(r[:, m])
            assert b >= A.bar(n, m, dtype), f"{tag} n={n} m={m}: {b:.2f} worst x={x[np.argmax(r[:, m])]}"
        n += 1


# ---------------------------------------------------------------- KATs -------

def test_kat_x0_ladder(oracle):
    # x=0 -> [1, 1/3, ..., 1/(2n+1)] within 1 ulp each
    for n in range(17):
        F, _ = oracle.dense(n, np.zeros(1), "aos")
        exact = np.array([1.0 / (2 * m + 1) for m in range(n + 1)])
        ulps = np.abs(F[0] - exact) / np.spacing(exact)
        assert ulps[:n].max(initial=0) == 0          # m < n: exact via the recursion
        if n == 0:
            assert ulps[0] <= 1
        assert ulps[n] <= 2 ** (53 - A.bar(n, n, np.float64))
    for n in range(9):
        F, _ = oracle.dense(n, np.zeros(1, np.float32), "aos")
        exact = np.array([1.0 / (2 * m + 1) for m in range(n + 1)], dtype=np.float32)
        assert np.array_equal(F[0, :n], exact[:n])


def test_kat_f0_25_and_asymptote(oracle):
    # F_0(25) ~ c_0 25^-1/2 within 2^-30
    F, _ = oracle.dense(0, np.array([25.0]), "soa")
    assert abs(F[0, 0] / (C0 / 5.0) - 1) < 2 ** -30
    # (n=2, x=1e9) -> asymptotic branch, equals c_2 x^-5/2 to 1 ulp
    x = 1e9
    F, _ = oracle.dense(2, np.array([x]), "soa")
    ref = _cn(2) * x ** -2.5
    assert abs(F[2, 0] - ref) <= np.spacing(ref)


def test_kat_qtilde(oracle):
    from paper_2504_07637_b200 import coeffs as C
    ds = C.load_default("double53")
    for n in range(17):
        r = ds.records[n]
        q = oracle.qtilde(n, np.array([0.0, 1e6]))
        assert q[0] == r.q0                          # Q~(0) = q0
        lin = r.alpha * 1e6 + r.beta
        assert abs(q[1] / lin - 1) < 1e-4


def test_domain_reported(oracle):
    x = np.array([1.0, -2.0, np.nan, 3.0])
    F, bad = oracle.dense(3, x, "soa")
    assert bad == 1 and np.isnan(F[:, 1]).all() and np.isnan(F[:, 2]).all()
    assert np.isfinite(F[:, [0, 3]]).all()


# ----------------------------------------------------------- properties ------

def test_positivity_ordering_and_recursion_consistency(oracle):
    rng = np.random.default_rng(11)
    x = np.concatenate([np.exp(rng.uniform(np.log(1e-8), np.log(1e4), 20000)),
                        rng.uniform(0, 80, 20000)])
    for n in (4, 11, 16):
        F, _, t = oracle.dense(n, x, "soa", expx=True)
        m = np.arange(n + 1)[:, None]
        assert (F > 0).all() and (F <= 1.0 / (2 * m + 1)).all()
        assert (F[1:] < F[:-1]).all()
        # |(2x F_m + e^-x)/(2m+1) - F_{m-1}| <= 4 ulp (index per refmath.py:340)
        xl, Fl, tl = (np.longdouble(x), F.astype(np.longdouble), np.longdouble(t))
        for mm in range(1, n + 1):
            pred = (2 * xl * Fl[mm] + tl) / (2 * mm - 1)
            ulps = np.abs(pred - Fl[mm - 1]) / np.spacing(F[mm - 1]).astype(np.longdouble)
            assert float(ulps.max()) <= 4, f"n={n} m={mm}"


def test_batch_equals_scalar_and_shuffle(oracle):
    rng = np.random.default_rng(5)
    x = rng.uniform(0, 90, 1000)
    F, _ = oracle.dense(9, x, "aos")
    for i in (0, 17, 999):
        F1, _ = oracle.dense(9, x[i:i + 1], "aos")
        assert np.array_equal(F1[0], F[i])
    p = rng.permutation(x.size)
    Fp, _ = oracle.dense(9, x[p], "aos")
    assert np.array_equal(Fp, F[p])


def test_exp_accuracy(oracle):
    x = np.linspace(0, 708, 200001)
    e = oracle.expneg(x)
    ref = np.exp(-np.longdouble(x))
    ulps = np.abs(e.astype(np.longdouble) - ref) / np.spacing(e).astype(np.longdouble)
    assert float(ulps.max()) <= 1.0
    xf = np.linspace(0, 86, 100001).astype(np.float32)
    ef = oracle.expneg(xf)
    reff = np.exp(-np.float64(xf))
    assert (np.abs(ef - reff) / np.spacing(ef.astype(np.float32)).astype(np.float64)).max() <= 1.0
    assert oracle.expneg(np.array([709.0, 1e300]))[0] == 0.0


def test_split_matches_two_dense(oracle):
    x = np.random.default_rng(2).uniform(0, 80, 500)
    S, _ = oracle.split(16, 7, x, "soa")
    lo, _ = oracle.dense(7, x, "soa")
    hi, _ = oracle.dense(16, x, "soa")
    assert np.array_equal(S[:8], lo) and np.array_equal(S[8:], hi[8:])


def test_split_improves_low_orders(oracle):
    # accuracy of F_0..F_nbar >= single-seed eval at the same n
    d = A.load("scan_f64.npz")
    x, gold = d["x16"], d["F16"]
    S, _ = oracle.split(16, 8, x, "aos")
    D, _ = oracle.dense(16, x, "aos")
    for m in range(9):
        assert A.bits(A.rel_err(S[:, m], gold[:, m])) >= A.bits(A.rel_err(D[:, m], gold[:, m])) - 1.0
