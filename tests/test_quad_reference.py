"""Pin the extended-precision oracle restatements (oracle/boys_quad.c) to the
reference's own outputs: refmath.boys_downward at Precision(96) goldens."""

import numpy as np
import pytest

import accuracy as A


def _agree_bits(ref, gold):
    ok = np.abs(gold[..., 0]) > 1e-300
    d = np.abs((ref[..., 0] - gold[..., 0]) + (ref[..., 1] - gold[..., 1]))
    r = np.where(ok, d / np.where(ok, np.abs(gold[..., 0]), 1.0), 0.0)
    return -np.log2(r.max()) if r.max() > 0 else np.inf


@pytest.mark.parametrize("precision,bits", [("ld", 57.0), ("quad", 100.0)])
def test_reference_matches_mpmath_goldens(oracle, precision, bits):
    d = A.load("scan_f64.npz")
    for n in (0, 8, 16):
        x = d[f"x{n}"] if precision == "ld" else d[f"x{n}"][::8]
        g = d[f"F{n}"] if precision == "ld" else d[f"F{n}"][::8]
        assert _agree_bits(oracle.reference(n, x, precision), g) >= bits, (precision, n)
    c = A.load("configs.npz")
    for name, n in (("cfg1", 0), ("cfg2", 8), ("cfg3", 16), ("cfg5", 12)):
        x, g = c[f"{name}_x"][::4], c[f"{name}_F"][::4]
        assert _agree_bits(oracle.reference(n, x, precision), g) >= bits, (precision, name)
