"""Accuracy bars from the paper's Table I and the
relative-error measurement against double-double golden vectors."""

from __future__ import annotations

from pathlib import Path

import numpy as np

GOLDEN = Path(__file__).resolve().parent / "golden"

# n: (eps_bar_0, eps_bar_{n-1}, eps_bar_n, eps_n) -- PAPER.md:186-202 (53-bit double)
TABLE1_F64 = {
    0: (52.0, None, 52.0, 58.0), 1: (50.2, None, 49.6, 52.7), 2: (49.9, 50.0, 49.0, 53.8),
    3: (49.0, 49.1, 48.4, 51.5), 4: (48.7, 48.8, 47.7, 51.1), 5: (48.7, 48.9, 46.9, 50.7),
    6: (48.3, 48.3, 47.0, 51.1), 7: (48.1, 48.3, 46.6, 51.3), 8: (48.2, 48.2, 46.2, 51.0),
    9: (47.8, 47.9, 45.5, 50.1), 10: (47.6, 47.5, 45.4, 49.3), 11: (47.8, 47.4, 45.0, 51.0),
    12: (47.6, 47.4, 44.6, 50.7), 13: (47.4, 47.2, 44.8, 50.3), 14: (47.3, 47.0, 44.5, 49.9),
    15: (47.1, 46.5, 43.9, 49.6), 16: (47.0, 46.6, 44.1, 49.2), 17: (47.0, 46.4, 43.8, 48.8),
    18: (47.4, 46.2, 43.4, 51.6), 19: (47.2, 46.1, 43.2, 51.3), 20: (47.1, 46.0, 43.3, 51.1),
    21: (47.1, 45.7, 43.1, 50.8), 22: (47.0, 45.8, 43.2, 50.5), 23: (46.8, 45.6, 42.8, 50.3),
    24: (46.7, 45.6, 42.9, 50.1), 25: (46.5, 45.6, 43.0, 49.9), 26: (46.7, 45.0, 42.4, 49.7),
    27: (46.6, 45.5, 42.7, 49.5), 28: (46.4, 45.1, 42.3, 49.3), 29: (46.4, 45.1, 42.3, 49.1),
    30: (46.4, 45.1, 42.2, 48.9), 31: (46.3, 44.5, 41.8, 48.8), 32: (46.3, 44.9, 42.2, 48.6),
    33: (46.3, 44.4, 41.8, 48.4), 34: (46.3, 44.6, 41.8, 48.3), 35: (46.1, 44.3, 41.5, 48.2),
    36: (46.0, 44.3, 41.8, 48.0),
}
# 24-bit single half of Table I
TABLE1_F32 = {
    0: (22.9, None, 22.9, 27.3), 1: (21.4, None, 21.1, 23.7), 2: (21.0, 21.1, 19.8, 27.3),
    3: (20.4, 20.4, 19.0, 25.5), 4: (20.1, 20.2, 18.5, 24.2), 5: (19.8, 20.0, 18.3, 23.3),
    6: (19.4, 19.5, 17.7, 22.5), 7: (19.2, 19.4, 17.5, 21.9), 8: (19.0, 19.0, 17.0, 21.3),
    9: (18.9, 18.8, 16.7, 20.9), 10: (18.9, 18.7, 16.4, 24.9), 11: (19.2, 18.6, 16.1, 24.5),
    12: (18.6, 18.4, 16.1, 24.2), 13: (18.5, 18.3, 15.9, 23.8), 14: (18.4, 18.1, 15.7, 23.5),
    15: (18.5, 17.8, 15.1, 23.3), 16: (18.4, 17.7, 15.3, 23.0),
}
SLACK = 2.0   # SPEC.md:424-426 ("within 2 bits")


def bar(n: int, m: int, dtype) -> float:
    """Minimum -log2(rel err) for F_m at order n: eps_bar - 2."""
    t = (TABLE1_F32 if np.dtype(dtype) == np.float32 else TABLE1_F64)[n]
    e0, enm1, en, _ = t
    if m == n:
        return en - SLACK
    lo = e0 if enm1 is None else min(e0, enm1)
    return lo - SLACK


def rel_err(got: np.ndarray, gold: np.ndarray, dtype=np.float64) -> np.ndarray:
    """|got - F| / F with F given as double-double gold[..., 0] + gold[..., 1].
    For fp32, values whose true magnitude is below FLT_MIN are measured in
    absolute terms relative to FLT_MIN."""
    g = got.astype(np.float64)
    hi, lo = gold[..., 0], gold[..., 1]
    err = np.abs((g - hi) - lo)
    if np.dtype(dtype) == np.float32:
        tiny = np.finfo(np.float32).tiny
        den = np.maximum(np.abs(hi), tiny)
    else:
        den = np.abs(hi)
    with np.errstate(divide="ignore", invalid="ignore"):
        r = np.where(den > 0, err / den, np.where(err == 0, 0.0, np.inf))
    return r


def bits(r: np.ndarray) -> float:
    m = float(np.max(r)) if r.size else 0.0
    return float("inf") if m == 0 else -np.log2(m)


def load(name):
    return np.load(GOLDEN / name)


def representable(gold, dtype) -> np.ndarray:
    """True magnitude is a normal number of `dtype` (denormal/underflowed
    references are excluded from relative checks; fp64 only)."""
    return np.abs(gold[..., 0]) >= np.finfo(dtype).tiny
