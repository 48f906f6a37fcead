"""Coefficient dataset: format round trips, fault injection, table invariants
(SPEC.md:126-272), generated header, and -- where the reference is present --
constants re-derived from refmath."""

import math
import os
import struct
import sys
from pathlib import Path

import numpy as np
import pytest
from hypothesis import given, settings, strategies as st

from paper_2504_07637_b200 import coeffs as C

import accuracy as A

REF = Path(os.environ.get("BOYS_REFERENCE_SRC", "/root/reference/pkg/src"))
needs_ref = pytest.mark.skipif(not (REF / "boysfn").exists(), reason="reference not present")


@pytest.fixture(scope="module", params=["double53", "single24"])
def ds(request):
    return C.load_default(request.param)


def test_orders_and_degrees(ds):
    mx = max(ds.orders())
    assert mx >= (16 if ds.profile == "double53" else 8)     # the configs' orders
    assert ds.orders() == list(range(mx + 1))
    for n, r in ds.records.items():
        Lu, lu, Lv, lv = r.counts()
        assert 2 * Lu + lu == r.N - 1 and 2 * Lv + lv == r.N
        assert all(a > 0 for _, a in r.u_quads) and all(b > 0 for _, b in r.v_quads)
        assert all(z < 0 for z in r.v_lins)                      # no pole on [0, inf)
        v0 = np.prod([y * y + b for y, b in r.v_quads]) * np.prod([-z for z in r.v_lins])
        assert v0 > 0                                            # B_N > 0
        eps = 2.0 ** (-52 if ds.profile == "double53" else -23)
        assert r.q2 == pytest.approx(r.alpha - r.q1, rel=4 * eps)
        assert r.z > 0 and r.x_up > r.z
        ys = [y for y, _ in r.u_quads]
        assert ys == sorted(ys)                                  # SPEC.md:176 order


def test_n_matches_table1(ds):
    table = {"double53": {0: 10, 1: 10, 2: 11, 7: 12, 11: 13, 18: 14},
             "single24": {0: 4, 1: 4, 2: 5, 10: 6}}[ds.profile]
    cur = None
    for n in ds.orders():
        cur = table.get(n, cur)
        assert ds.records[n].N == cur


def test_exact_bits_vs_paper(ds):
    # SPEC acceptance 3/4: refit reaches the paper's exact-arithmetic eps within 2 bits
    t = A.TABLE1_F64 if ds.profile == "double53" else A.TABLE1_F32
    for n, r in ds.records.items():
        assert r.exact_bits >= t[n][3] - 2.0, f"n={n}: {r.exact_bits} vs {t[n][3]}"


def test_roundtrip_and_literal(ds, tmp_path):
    p = tmp_path / "d.dat"
    C.save(ds, p)
    assert C.load(p) == ds
    assert C.dumps(ds) == p.read_text()
    assert (1.0).hex() == "0x1.0000000000000p+0"


def test_fault_injection(ds, tmp_path):
    text = C.dumps(ds)
    with pytest.raises(C.DatasetError, match="truncated"):
        C.loads(text[: len(text) // 2])
    with pytest.raises(C.DatasetError, match="checksum"):
        C.loads(text.replace("record 0", "record  0", 1))
    lines = text.split("\n")
    bad = "\n".join(lines[:-2]).replace(" c 0x", " c 1x", 1) + "\n"
    import hashlib
    bad += f"checksum sha256 {hashlib.sha256(bad.encode()).hexdigest()}\n"
    with pytest.raises(C.DatasetError, match=r"line \d+: malformed"):
        C.loads(bad)
    v2 = text.replace("version 1", "version 2", 1)
    body = v2[: v2.rindex("checksum")]
    v2 = body + f"checksum sha256 {hashlib.sha256(body.encode()).hexdigest()}\n"
    with pytest.raises(C.DatasetError, match="version"):
        C.loads(v2)


@settings(max_examples=300, deadline=None)
@given(st.integers(min_value=0, max_value=2 ** 64 - 1))
def test_serialization_lossless_for_any_double(bits):
    v = struct.unpack("<d", struct.pack("<Q", bits))[0]
    if not math.isfinite(v):
        return
    r = C.Record(n=0, N=2, c=v, q0=v, q1=v, q2=v, alpha=v, beta=v, z=v, x_up=v,
                 u_quads=[], u_lins=[v], v_quads=[(v, v)], v_lins=[])
    ds = C.Dataset(profile="double53", records={0: r})
    back = C.loads(C.dumps(ds))
    assert struct.pack("<d", back.records[0].c) == struct.pack("<d", v)


def test_generated_header_is_current():
    tables = [C.build_kernel_table(C.load_default(p)) for p in ("double53", "single24")]
    hdr = Path(C.__file__).parent / "csrc" / "boys_tables.inc"
    assert C.gen_header(tables) == hdr.read_text()
    # deterministic and idempotent
    assert C.gen_header(tables) == C.gen_header(
        [C.build_kernel_table(C.load_default(p)) for p in ("double53", "single24")])


def test_kernel_table_missing_order():
    ds = C.load_default("double53")
    ds.records.pop(3)
    with pytest.raises(C.DatasetError, match="contiguous"):
        C.build_kernel_table(ds)


@needs_ref
def test_constants_rederived_from_reference():
    """c_n, alpha, beta, q0, q1, z_{n,b} equal the reference oracle's values
    rounded once (refmath.py:344-363, 417-477)."""
    sys.path.insert(0, str(REF))
    from boysfn import refmath as R
    from mpmath import mp
    for prof, bits in (("double53", 53), ("single24", 24)):
        ds = C.load_default(prof)
        for n in (0, 1, 5, 8) + ((12, 16) if bits == 53 else ()):
            k = R.constants(n, R.Precision(128))
            r = ds.records[n]

            def rnd(v):
                with mp.workprec(bits):
                    return float(+v)
            assert r.c == rnd(k.c) and r.q0 == rnd(k.q0) and r.q1 == rnd(k.q1)
            assert r.alpha == rnd(k.alpha) and r.beta == rnd(k.beta)
            with mp.workprec(200):
                q2 = k.alpha - k.q1
            assert r.q2 == rnd(q2)
            z = R.cutoff_solve(n, bits, R.Precision(128))
            assert r.z == rnd(z)


def test_survey_appendix_a_constants():
    """Pin against the reference values transcribed in SURVEY.md Appendix A."""
    ds = C.load_default("double53")
    appx = {0: (0.88622692545275805, 0.61685027506808487, 0.48537125676538645, 34.381626105834208),
            8: (7017.2036467417065, 1.1756134329362744, 0.1179040820267815, 57.743962522346173),
            16: (2594999226520.0625, 1.1250606770019416, 0.06232542527975888, 74.506825355932591)}
    for n, (c, q0, q1, z) in appx.items():
        r = ds.records[n]
        assert (r.c, r.q0, r.q1, r.z) == (c, q0, q1, z)
