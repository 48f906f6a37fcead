"""The C-ABI library loads and exports every symbol include/boys.h declares;
the product path has no CPU fallback and never touches oracle/.  (No compute
calls here: this file runs without a GPU.)"""

import ctypes
import re
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
HEADER = ROOT / "include" / "boys.h"


def declared_functions():
    text = HEADER.read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(boys_[a-z_0-9]+)\s*\(", text)))


def test_header_declares_expected_surface():
    from paper_2504_07637_b200 import _lib
    assert declared_functions() == sorted(_lib.EXPORTS)


def test_library_loads_and_exports_every_symbol():
    from paper_2504_07637_b200 import _lib
    L = _lib.load()
    for name in declared_functions():
        assert hasattr(L, name), name
    from paper_2504_07637_b200 import coeffs as C
    assert L.boys_max_order(_lib.BOYS_F64) == max(C.load_default("double53").orders()) >= 16
    assert L.boys_max_order(_lib.BOYS_F32) == max(C.load_default("single24").orders()) >= 8
    assert L.boys_max_order(7) == -1
    assert b"sm_100a" in L.boys_version()
    for code in range(8):
        assert L.boys_status_str(code)


def test_argument_errors_without_gpu():
    """Argument validation happens before any CUDA call."""
    from paper_2504_07637_b200 import _lib
    L = _lib.load()
    x = np.zeros(4)
    p = x.ctypes.data_as(ctypes.c_void_p)
    m64, m32 = L.boys_max_order(_lib.BOYS_F64), L.boys_max_order(_lib.BOYS_F32)
    assert L.boys_eval_dense(_lib.BOYS_F64, m64 + 1, p, 4, p, 0, None, None, None) == _lib.BOYS_E_ORDER
    assert L.boys_eval_dense(_lib.BOYS_F32, m32 + 1, p, 4, p, 0, None, None, None) == _lib.BOYS_E_ORDER
    assert L.boys_eval_dense(_lib.BOYS_F64, 2, p, 4, p, 5, None, None, None) == _lib.BOYS_E_LAYOUT
    assert L.boys_eval_dense(9, 2, p, 4, p, 0, None, None, None) == _lib.BOYS_E_DTYPE
    assert L.boys_eval_dense(_lib.BOYS_F64, 2, None, 4, p, 0, None, None, None) == _lib.BOYS_E_ARG
    assert L.boys_eval_dense(_lib.BOYS_F64, 2, p, -1, p, 0, None, None, None) == _lib.BOYS_E_ARG
    assert L.boys_eval_dense(_lib.BOYS_F64, 2, p, 0, p, 0, None, None, None) == _lib.BOYS_OK
    bad = ctypes.c_void_p(x.ctypes.data + 4)
    assert L.boys_eval_dense(_lib.BOYS_F64, 2, bad, 4, p, 0, None, None, None) == _lib.BOYS_E_ALIGN
    assert L.boys_eval_split(_lib.BOYS_F64, 4, 4, p, 4, p, 0, None, None) == _lib.BOYS_E_ARG
    # ragged host-buffer entry
    n8 = np.zeros(4, dtype=np.uint8)
    pn = n8.ctypes.data_as(ctypes.c_void_p)
    fb = ctypes.c_int64(7)
    assert L.boys_eval_ragged_host(9, p, pn, 4, p, 4, ctypes.byref(fb)) == _lib.BOYS_E_DTYPE
    assert L.boys_eval_ragged_host(_lib.BOYS_F64, p, pn, -1, p, 4, None) == _lib.BOYS_E_ARG
    assert L.boys_eval_ragged_host(_lib.BOYS_F64, p, pn, 4, p, -1, None) == _lib.BOYS_E_ARG
    assert L.boys_eval_ragged_host(_lib.BOYS_F64, None, pn, 4, p, 4, None) == _lib.BOYS_E_ARG
    assert L.boys_eval_ragged_host(_lib.BOYS_F64, p, None, 4, p, 4, None) == _lib.BOYS_E_ARG
    assert L.boys_eval_ragged_host(_lib.BOYS_F64, p, pn, 0, p, 0, ctypes.byref(fb)) == _lib.BOYS_OK
    assert fb.value == -1


def test_no_cpu_fallback():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2504_07637_b200 import boys
    with pytest.raises(RuntimeError, match="CUDA"):
        boys(3, np.array([1.0, 2.0]))


def test_product_never_imports_oracle():
    pkg = ROOT / "paper_2504_07637_b200"
    bad = re.compile(r"^\s*(from\s+oracle|import\s+oracle)|liboracle|libquad|boys_oracle_|"
                     r"boys_(ld|quad)_downward", re.M)
    for f in list(pkg.rglob("*.py")) + list(pkg.rglob("*.cu")) + list(pkg.rglob("*.cuh")):
        assert not bad.search(f.read_text()), f
    nm = (pkg / "libboys.so").read_bytes()
    assert b"boys_oracle" not in nm


def test_oracle_library_exports():
    from oracle import oracle as O
    L = O.lib()
    for s in ("boys_oracle_load", "boys_oracle_dense", "boys_oracle_ragged", "boys_oracle_split",
              "boys_oracle_qtilde", "boys_oracle_expneg"):
        assert hasattr(L, s)


def test_c_example_compiles_and_links(tmp_path):
    """include/boys.h is plain C and libboys.so links from a C host
    (examples/c_host.c; the GPU test runs it)."""
    import shutil
    import subprocess
    if shutil.which("gcc") is None:
        pytest.skip("gcc absent")
    from paper_2504_07637_b200 import build as B
    exe = tmp_path / "c_host"
    subprocess.run(["gcc", "-O2", "-std=c11", "-Wall", "-Werror", "-I", str(ROOT / "include"),
                    str(ROOT / "examples" / "c_host.c"), "-L", str(B.PKG), "-lboys",
                    f"-Wl,-rpath,{B.PKG}", "-o", str(exe)], check=True)
    r = subprocess.run([str(exe)], capture_output=True, text=True)
    assert r.returncode == 64 and "usage" in r.stderr


def test_compiled_table_checksum_without_gpu():
    """libboys reports the digest of the table it was compiled with; it equals
    coeffs.table_checksum of the shipped datasets (the boundary compares a
    caller's table against it)."""
    from paper_2504_07637_b200 import _lib, coeffs as C
    L = _lib.load()
    for dt, prof in ((_lib.BOYS_F64, "double53"), (_lib.BOYS_F32, "single24")):
        kt = C.build_kernel_table(C.load_default(prof))
        assert L.boys_table_checksum(dt).decode() == C.table_checksum(kt)
        assert L.boys_table_row_bytes(dt) * len(kt.rows) == len(C.pack_rows(kt))
