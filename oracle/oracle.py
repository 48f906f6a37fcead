"""ctypes wrapper of the CPU oracle (liboracle.so) -- TEST INFRASTRUCTURE.

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline / reference
arm may import this module, and only as the checker.  The product path
(paper_2504_07637_b200) never imports it.

The oracle restates the SPEC'd kernel in C; see
boys_oracle.c for the line-by-line citations and the pinning strategy.
"""

from __future__ import annotations

import ctypes as C
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
ROOT = HERE.parent
LIB = HERE / "liboracle.so"
QLIB = HERE / "libquad.so"
DATA = ROOT / "paper_2504_07637_b200" / "data"

_lib = None
_tables = {}


def build(force: bool = False) -> Path:
    srcs = ("boys_oracle.c", "boys_oracle_impl.h", "boys_quad.c")
    newest = max((HERE / f).stat().st_mtime for f in srcs)
    if force or not LIB.exists() or not QLIB.exists() or min(
            LIB.stat().st_mtime, QLIB.stat().st_mtime) < newest:
        subprocess.run(["make", "-s", "-C", str(HERE)], check=True)
    return LIB


_qlib = None


def _quad():
    global _qlib
    if _qlib is None:
        build()
        Q = C.CDLL(str(QLIB))
        for f in (Q.boys_quad_downward, Q.boys_ld_downward):
            f.argtypes = [C.c_int, C.c_void_p, C.c_int64, C.c_void_p]
        _qlib = Q
    return _qlib


def reference(n: int, x, precision: str = "ld"):
    """Extended-precision restatement of refmath.boys_downward (oracle/boys_quad.c):
    F_0..F_n(x) as double-double [N, n+1, 2].  precision 'ld' (x87, ~2^-59,
    fast) or 'quad' (binary128, ~2^-106)."""
    xd = np.ascontiguousarray(x, dtype=np.float64).reshape(-1)
    out = np.empty((xd.size, n + 1, 2))
    f = _quad().boys_ld_downward if precision == "ld" else _quad().boys_quad_downward
    f(n, _ptr(xd), xd.size, _ptr(out))
    return out


def lib():
    global _lib
    if _lib is None:
        build()
        L = C.CDLL(str(LIB))
        L.boys_oracle_load.restype = C.c_void_p
        L.boys_oracle_load.argtypes = [C.c_char_p]
        L.boys_oracle_max_order.argtypes = [C.c_void_p]
        L.boys_oracle_dense.restype = C.c_int64
        L.boys_oracle_dense.argtypes = [C.c_void_p, C.c_int, C.c_void_p, C.c_int64, C.c_void_p,
                                        C.c_int, C.c_void_p]
        L.boys_oracle_ragged.restype = C.c_int64
        L.boys_oracle_ragged.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                         C.c_int64, C.c_void_p]
        L.boys_oracle_split.restype = C.c_int64
        L.boys_oracle_split.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_void_p, C.c_int64,
                                        C.c_void_p, C.c_int]
        L.boys_oracle_qtilde.argtypes = [C.c_void_p, C.c_int, C.c_void_p, C.c_int64, C.c_void_p]
        L.boys_oracle_expneg.argtypes = [C.c_int, C.c_void_p, C.c_int64, C.c_void_p]
        L.boys_oracle_threads.restype = C.c_int
        L.boys_oracle_hermite.restype = C.c_int64
        L.boys_oracle_hermite.argtypes = [C.c_void_p, C.c_int, C.c_void_p, C.c_int64,
                                          C.c_void_p, C.c_int64, C.c_void_p]
        _lib = L
    return _lib


def table(dtype, path=None):
    """Oracle table for dtype: the shipped dataset, or the dataset file `path`
    (the oracle's own parser; used to check the uploaded-table path)."""
    dtype = np.dtype(dtype)
    key = (dtype, str(path) if path else None)
    if key not in _tables:
        prof = "single24" if dtype == np.float32 else "double53"
        src = str(path) if path else str(DATA / f"boys_{prof}.dat")
        t = lib().boys_oracle_load(src.encode())
        if not t:
            raise RuntimeError(f"oracle could not parse the dataset {src}")
        _tables[key] = t
    return _tables[key]


def max_order(dtype) -> int:
    return lib().boys_oracle_max_order(table(dtype))


def _ptr(a):
    return a.ctypes.data_as(C.c_void_p)


def dense(n: int, x, layout: str = "soa", expx: bool = False, table_path=None):
    """F_0..F_n for every x (dtype float64 or float32).  Returns
    (values, first_bad[, expx]); values [n+1][N] (soa) or [N][n+1] (aos).
    table_path: evaluate with that dataset file instead of the shipped one."""
    x = np.ascontiguousarray(x)
    assert x.dtype in (np.float64, np.float32)
    N = x.size
    shape = (n + 1, N) if layout == "soa" else (N, n + 1)
    out = np.empty(shape, dtype=x.dtype)
    ex = np.empty(N, dtype=x.dtype) if expx else None
    bad = lib().boys_oracle_dense(table(x.dtype, table_path), n, _ptr(x), N, _ptr(out),
                                  0 if layout == "soa" else 1, _ptr(ex) if expx else None)
    return (out, bad, ex) if expx else (out, bad)


def offsets(nmax):
    nmax = np.asarray(nmax, dtype=np.uint8)
    off = np.zeros(nmax.size + 1, dtype=np.int64)
    np.cumsum(nmax.astype(np.int64) + 1, out=off[1:])
    return off


def ragged(x, nmax):
    x = np.ascontiguousarray(x)
    nmax = np.ascontiguousarray(nmax, dtype=np.uint8)
    off = offsets(nmax)
    out = np.empty(int(off[-1]), dtype=x.dtype)
    bad = lib().boys_oracle_ragged(table(x.dtype), _ptr(x), _ptr(nmax), _ptr(off), x.size,
                                   _ptr(out))
    return out, off, bad


def split(n: int, nbar: int, x, layout: str = "soa", table_path=None):
    x = np.ascontiguousarray(x)
    N = x.size
    out = np.empty((n + 1, N) if layout == "soa" else (N, n + 1), dtype=x.dtype)
    bad = lib().boys_oracle_split(table(x.dtype, table_path), n, nbar, _ptr(x), N, _ptr(out),
                                  0 if layout == "soa" else 1)
    return out, bad


def hermite(L: int, bra, ket):
    """Fused consumer restatement: pref * R_{tuv} (t+u+v <= L) for every
    (bra pair, ket pair); pair records (p, Px, Py, Pz, K).  Returns
    (values [Nb][Nk][NH], first_bad)."""
    bra = np.ascontiguousarray(bra, dtype=np.float64).reshape(-1, 5)
    ket = np.ascontiguousarray(ket, dtype=np.float64).reshape(-1, 5)
    NH = (L + 1) * (L + 2) * (L + 3) // 6
    out = np.empty((bra.shape[0], ket.shape[0], NH))
    bad = lib().boys_oracle_hermite(table(np.float64), L, _ptr(bra), bra.shape[0], _ptr(ket),
                                    ket.shape[0], _ptr(out))
    return out, bad


def qtilde(n: int, x):
    x = np.ascontiguousarray(x)
    out = np.empty_like(x)
    lib().boys_oracle_qtilde(table(x.dtype), n, _ptr(x), x.size, _ptr(out))
    return out


def expneg(x):
    x = np.ascontiguousarray(x)
    out = np.empty_like(x)
    lib().boys_oracle_expneg(int(x.dtype == np.float32), _ptr(x), x.size, _ptr(out))
    return out


def threads() -> int:
    return lib().boys_oracle_threads()
