"""Parity of every kernel variant reachable through an environment knob
(the A/B switches in csrc/boys_launch.h are read once per process, so
tests/test_gpu_knobs.py runs this script once per setting).

Checks dense SoA/AoS (even/odd N, several orders, f64/f32), ragged (f64/f32,
including a high-order tail) and split against the CPU oracle, bit for bit.
Prints "ok" and exits 0 on success."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle import oracle as O  # noqa: E402
from paper_2504_07637_b200 import boys, boys_ragged, eval_with_split, workloads as W  # noqa: E402


def same(a, b, what):
    a = np.asarray(a)
    assert a.shape == b.shape, what
    ok = (a.view(np.uint8) == b.view(np.uint8)).all() or np.array_equal(a, b, equal_nan=True)
    assert ok, f"{what}: not bit-identical"


def main():
    dev = torch.device("cuda:0")
    for dt in (np.float64, np.float32):
        for N in (1 << 16, (1 << 16) + 3):
            x = W.cfg3_x(N, chunk=9).numpy().astype(dt)
            xd = torch.from_numpy(x).to(dev)
            for n in (0, 1, 5, 8, 12, 16):
                for lay in ("soa", "aos"):
                    got = boys(n, xd, layout=lay).cpu().numpy()
                    ref, _ = O.dense(n, x, lay)
                    same(got, ref, f"dense {dt.__name__} N={N} n={n} {lay}")
            got = eval_with_split(16, 8, xd, layout="aos").cpu().numpy()
            ref, _ = O.split(16, 8, x, "aos")
            same(got, ref, f"split {dt.__name__} N={N}")
    xr, nr = W.cfg4_batch((1 << 16) + 77, chunk=2)
    nr[-40:] = 24                                   # high-order fallback chunks
    got, _ = boys_ragged(xr.to(dev), nr.to(dev))
    ref, _, _ = O.ragged(xr.numpy(), nr.numpy())
    same(got.cpu().numpy(), ref, "ragged f64")
    xf, nf = W.cfg4f32_batch(1 << 16, chunk=2)
    got, _ = boys_ragged(xf.to(dev), nf.to(dev))
    ref, _, _ = O.ragged(xf.numpy(), nf.numpy())
    same(got.cpu().numpy(), ref, "ragged f32")
    print("ok")


if __name__ == "__main__":
    main()
