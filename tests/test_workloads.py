"""Host logic: the seeded BASELINE workload generators (stated distributions,
exact strata proportions, determinism, chunk keys) and the roofline model."""

import math

import numpy as np
import torch

from paper_2504_07637_b200 import roofline as R, workloads as W


def test_cfg1_strata():
    x = W.cfg1_x(1 << 16).numpy()
    assert x.size == 1 << 16
    assert (x == 0).sum() >= (1 << 14)                        # 25% exactly zero
    assert ((x > 1) & (x <= 40)).sum() >= (1 << 14) * 0.9
    assert x.max() <= 1e4 and x.min() >= 0


def test_cfg3_cutoff_stratum():
    x = W.cfg3_x(1 << 16).numpy()
    near = np.abs(x / W.Z16_53 - 1) <= 1e-3
    assert near.sum() >= 0.1 * x.size
    assert x.min() >= 1e-12 and x.max() <= 1e5


def test_determinism_and_chunk_keys():
    a = W.cfg5_x(4096, chunk=3)
    b = W.cfg5_x(4096, chunk=3)
    c = W.cfg5_x(4096, chunk=4)
    assert torch.equal(a, b) and not torch.equal(a, c)


def test_cfg4_distribution():
    x, n = W.cfg4_batch(1 << 16)
    assert x.dtype == torch.float64 and n.dtype == torch.uint8
    assert int(n.max()) <= 12
    p = np.bincount(n.numpy(), minlength=13) / n.numel()
    w = np.array([1 / (k + 1) for k in range(13)])
    assert np.abs(p - w / w.sum()).max() < 0.01                # P(n) ~ 1/(n+1)
    xf, nf = W.cfg4f32_batch(1 << 16)
    assert xf.dtype == torch.float32 and int(nf.max()) <= 8


def test_roofline_model():
    assert R.dense_bytes_per_point(16) == 144 and R.dense_bytes_per_point(0) == 16
    assert R.pw(16) == 4 and R.pw(13) == 5 and R.pw(1) == 0
    # survey's model values: n=0: 79-80, n=16: ~131
    assert 75 <= R.ops_per_point(0) <= 85 and 125 <= R.ops_per_point(16) <= 140
    assert R.ops_per_point(8, below_cut=False) < R.ops_per_point(8)
    assert R.ragged_bytes(10, 41) == 10 * 8 + 10 + 11 * 8 + 41 * 8
