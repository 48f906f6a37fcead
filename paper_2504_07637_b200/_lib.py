"""ctypes binding of libboys.so (the C ABI declared in include/boys.h).

There is no CPU fallback: if the library cannot be loaded, or no CUDA device
is present, every entry point raises.  This is the reference-side binding a
Python caller uses (INTEGRATION.md shows the same binding for other hosts).
"""

from __future__ import annotations

import ctypes as C
import threading

from . import build as _build

BOYS_OK, BOYS_E_DOMAIN, BOYS_E_ORDER, BOYS_E_LAYOUT, BOYS_E_DTYPE, BOYS_E_ALIGN, BOYS_E_CUDA, \
    BOYS_E_ARG = range(8)
BOYS_F64, BOYS_F32 = 0, 1
BOYS_SOA, BOYS_AOS = 0, 1

# every symbol include/boys.h declares (tests check the export table)
EXPORTS = (
    "boys_max_order", "boys_version", "boys_eval_dense", "boys_eval_ragged",
    "boys_ragged_offsets", "boys_eval_split", "boys_domain_result", "boys_eval_dense_host", "boys_eval_ragged_host",
    "boys_launch_count", "boys_status_str", "boys_last_cuda_error",
    "boys_table_checksum", "boys_table_row_bytes", "boys_table_create", "boys_table_destroy",
    "boys_table_max_order", "boys_eval_dense_table", "boys_eval_split_table", "boys_shard_error",
    "boys_hermite_coulomb",
)

_lock = threading.Lock()
_lib = None


class BoysError(RuntimeError):
    """Non-domain failure reported by libboys (CUDA error, bad argument)."""


def load(build_if_missing: bool = True) -> C.CDLL:
    """Load (building first if stale and nvcc is available) libboys.so."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        import os
        override = os.environ.get("BOYS_LIB")      # experiments: an alternative build
        path = _build.LIB if not override else __import__("pathlib").Path(override)
        if not override and build_if_missing and _build.stale():
            try:
                _build.build_libboys()
            except Exception as e:   # noqa: BLE001
                if not path.exists():
                    raise RuntimeError(f"libboys.so missing and could not be built: {e}") from e
        if not path.exists():
            raise RuntimeError(f"libboys.so not found at {path}; run __graft_entry__.build()")
        L = C.CDLL(str(path))
        vp, i64, i32 = C.c_void_p, C.c_int64, C.c_int
        L.boys_max_order.restype = i32
        L.boys_max_order.argtypes = [i32]
        L.boys_version.restype = C.c_char_p
        L.boys_eval_dense.restype = i32
        L.boys_eval_dense.argtypes = [i32, i32, vp, i64, vp, i32, vp, vp, vp]
        L.boys_eval_ragged.restype = i32
        L.boys_eval_ragged.argtypes = [i32, vp, vp, vp, i64, vp, vp, vp]
        L.boys_ragged_offsets.restype = i32
        L.boys_ragged_offsets.argtypes = [vp, i64, vp, vp]
        L.boys_eval_split.restype = i32
        L.boys_eval_split.argtypes = [i32, i32, i32, vp, i64, vp, i32, vp, vp]
        L.boys_domain_result.restype = i32
        L.boys_domain_result.argtypes = [vp, C.POINTER(i64), vp]
        L.boys_eval_dense_host.restype = i32
        L.boys_eval_dense_host.argtypes = [i32, i32, vp, i64, vp, i32, C.POINTER(i64)]
        L.boys_eval_ragged_host.restype = i32
        L.boys_eval_ragged_host.argtypes = [i32, vp, vp, i64, vp, i64, C.POINTER(i64)]
        L.boys_table_checksum.restype = C.c_char_p
        L.boys_table_checksum.argtypes = [i32]
        L.boys_table_row_bytes.restype = C.c_size_t
        L.boys_table_row_bytes.argtypes = [i32]
        L.boys_table_create.restype = i32
        L.boys_table_create.argtypes = [i32, vp, i32, C.c_size_t, C.POINTER(vp)]
        L.boys_table_destroy.restype = i32
        L.boys_table_destroy.argtypes = [vp]
        L.boys_table_max_order.restype = i32
        L.boys_table_max_order.argtypes = [vp]
        L.boys_eval_dense_table.restype = i32
        L.boys_eval_dense_table.argtypes = [vp, i32, vp, i64, vp, i32, vp, vp, vp]
        L.boys_eval_split_table.restype = i32
        L.boys_eval_split_table.argtypes = [vp, i32, i32, vp, i64, vp, i32, vp, vp]
        L.boys_shard_error.restype = i32
        L.boys_shard_error.argtypes = [i32, vp, vp, vp, i64, vp, vp]
        L.boys_hermite_coulomb.restype = i32
        L.boys_hermite_coulomb.argtypes = [i32, vp, i64, vp, i64, vp, vp, vp]
        L.boys_launch_count.restype = i64
        L.boys_status_str.restype = C.c_char_p
        L.boys_status_str.argtypes = [i32]
        L.boys_last_cuda_error.restype = C.c_char_p
        _lib = L
        return L


def status_str(code: int) -> str:
    return load().boys_status_str(code).decode()


def check(code: int) -> None:
    if code == BOYS_OK:
        return
    msg = status_str(code)
    if code == BOYS_E_CUDA:
        msg += ": " + load().boys_last_cuda_error().decode()
    if code in (BOYS_E_ORDER, BOYS_E_LAYOUT, BOYS_E_DTYPE, BOYS_E_ARG, BOYS_E_ALIGN):
        raise ValueError(msg)
    raise BoysError(msg)


def launch_count() -> int:
    return int(load().boys_launch_count())
