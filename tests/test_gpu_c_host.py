"""A plain C program (examples/c_host.c) linked against libboys through
include/boys.h only -- the drop-in a compiled host would make -- produces the
same bits as the CPU oracle for the dense and ragged host-buffer entries and
reports the reference's domain / order errors."""

import shutil
import subprocess

import numpy as np
import pytest

from paper_2504_07637_b200 import build as B, workloads as W

pytestmark = pytest.mark.gpu
ROOT = B.PKG.parent


@pytest.mark.skipif(shutil.which("gcc") is None, reason="gcc absent")
def test_c_host_program(tmp_path, oracle):
    exe = tmp_path / "c_host"
    subprocess.run(["gcc", "-O2", "-std=c11", "-Wall", "-I", str(ROOT / "include"),
                    str(ROOT / "examples" / "c_host.c"), "-L", str(B.PKG), "-lboys",
                    f"-Wl,-rpath,{B.PKG}", "-o", str(exe)], check=True)
    x, n = W.cfg4_batch(1 << 18, chunk=5)
    x, n = x.numpy(), n.numpy()
    N = x.size
    x.tofile(tmp_path / "x.bin")
    n.tofile(tmp_path / "n.bin")
    r = subprocess.run([str(exe), str(tmp_path / "x.bin"), str(tmp_path / "n.bin"),
                        str(tmp_path / "d.bin"), str(tmp_path / "r.bin"), str(N)],
                       capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr
    assert "ok:" in r.stdout
    dense = np.fromfile(tmp_path / "d.bin", dtype=np.float64).reshape(N, 17)
    ragged = np.fromfile(tmp_path / "r.bin", dtype=np.float64)
    ref_d, _ = oracle.dense(16, x, "aos")
    ref_r, _, _ = oracle.ragged(x, n)
    assert np.array_equal(dense.view(np.int64), ref_d.view(np.int64))
    assert np.array_equal(ragged.view(np.int64), ref_r.view(np.int64))
