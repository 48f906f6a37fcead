"""Algorithmic bytes and FP64/FP32 operation counts per point (the roofline
model of DESIGN.md / SURVEY.md 8(d)).

Bytes are compulsory traffic: read x (and n_i + offsets for ragged), write
every output value once.  Operations count each DADD/DMUL/DFMA (FADD/FMUL/
FFMA) as one pipe op; correctly rounded division, reciprocal and square root
are weighted by their sm_100a fast-path instruction counts measured with
cuobjdump in the survey (div/rcp 8, sqrt 7 for f64; 5/5/4 for f32).  Factor
counts come from the frozen coefficient tables.
"""

from __future__ import annotations

from functools import lru_cache

from . import coeffs as C

DIV = {8: 8, 4: 5}
SQRT = {8: 7, 4: 4}
EXP = {8: 18, 4: 12}   # 2 (k) + 2 (r) + Taylor Horner (13 / 7 fma) + scale


def pw(n: int) -> int:
    """Multiplies in LSB-first binary exponentiation of b^n (n >= 1)."""
    return n.bit_length() - 1 + bin(n).count("1") - 1 if n > 0 else 0


@lru_cache(maxsize=None)
def _shape(profile: str, n: int):
    return C.load_default(profile).records[n].counts()


def ops_per_point(n: int, elem_bytes: int = 8, below_cut: bool = True) -> int:
    """Pipe ops for F_0..F_n of one x (below the cut-off unless told otherwise)."""
    prof = "double53" if elem_bytes == 8 else "single24"
    Lu, lu, Lv, lv = _shape(prof, n)

    def prod(L, l):
        k = 3 * L + 2 * l
        return k - 1 if k else 0     # first factor needs no multiply

    ops = EXP[elem_bytes]
    if below_cut:
        ops += prod(Lu, lu) + prod(Lv, lv) + DIV[elem_bytes] + 3   # u, v, u/v, Q
        ops += SQRT[elem_bytes] + (pw(n) + 1 if n else 0) + 1         # s, y
    ops += DIV[elem_bytes] + SQRT[elem_bytes] + (pw(n) + 1 if n else 0) + 1   # F_n
    if n:
        ops += 1 + 2 * n                                              # recursion
    return ops


def dense_bytes_per_point(n: int, elem_bytes: int = 8) -> int:
    return elem_bytes * (1 + n + 1)


def ragged_bytes(N: int, total_values: int, elem_bytes: int = 8) -> int:
    """x + n_i (u8) + offsets (int64, N+1) + values."""
    return N * elem_bytes + N + (N + 1) * 8 + total_values * elem_bytes
