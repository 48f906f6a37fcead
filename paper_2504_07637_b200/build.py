"""Build libboys.so in-tree for sm_100a (nvcc cross-compiles without a GPU)."""

from __future__ import annotations

import os
import shutil
import subprocess
from pathlib import Path

PKG = Path(__file__).resolve().parent
CSRC = PKG / "csrc"
LIB = PKG / "libboys.so"
PROBE_LIB = PKG / "libboys_probe.so"
# translation units of libboys (compiled in parallel, linked into one .so)
UNITS = [CSRC / "dense.cu", CSRC / "ragged.cu", CSRC / "split.cu", CSRC / "table.cu",
         CSRC / "shard.cu", CSRC / "hermite.cu", CSRC / "abi.cu"]
SOURCES = UNITS + [CSRC / "boys_device.cuh", CSRC / "boys_launch.h", CSRC / "boys_eval.cuh",
                   CSRC / "boys_tables.inc", PKG.parent / "include" / "boys.h"]

ARCH_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-fmad=false",            # belt and braces: the evaluator uses explicit __*_rn intrinsics
    "-Xcompiler", "-fPIC",
]
NVCC_FLAGS = ARCH_FLAGS + ["-shared"]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if cand and Path(cand).exists():
            return cand
    raise RuntimeError("nvcc not found: cannot build libboys.so")


def stale() -> bool:
    if not LIB.exists():
        return True
    t = LIB.stat().st_mtime
    return any(s.stat().st_mtime > t for s in SOURCES if s.exists())


def build_libboys(force: bool = False, verbose: bool = False) -> Path:
    if not force and not stale():
        return LIB
    from concurrent.futures import ThreadPoolExecutor
    objdir = PKG / "build"
    objdir.mkdir(exist_ok=True)

    def compile_unit(src: Path) -> Path:
        obj = objdir / (src.stem + ".o")
        cmd = [nvcc(), *ARCH_FLAGS, "-c", "-o", str(obj), str(src)]
        if verbose:
            print(" ".join(cmd), flush=True)
        subprocess.run(cmd, check=True)
        return obj

    with ThreadPoolExecutor(max_workers=len(UNITS)) as pool:
        objs = list(pool.map(compile_unit, UNITS))
    cmd = [nvcc(), *NVCC_FLAGS, "-o", str(LIB) + ".tmp", *map(str, objs)]
    if verbose:
        print(" ".join(cmd), flush=True)
    subprocess.run(cmd, check=True)
    os.replace(str(LIB) + ".tmp", LIB)
    return LIB


def build_probe(force: bool = False, verbose: bool = False) -> Path:
    """FP64 peak probe (measurement helper for the roofline denominator)."""
    src = CSRC / "probe.cu"
    if not force and PROBE_LIB.exists() and PROBE_LIB.stat().st_mtime >= src.stat().st_mtime:
        return PROBE_LIB
    cmd = [nvcc(), *NVCC_FLAGS, "-o", str(PROBE_LIB), str(src)]
    if verbose:
        print(" ".join(cmd), flush=True)
    subprocess.run(cmd, check=True)
    return PROBE_LIB


if __name__ == "__main__":
    print(build_libboys(force=True, verbose=True))
    print(build_probe(force=True, verbose=True))
