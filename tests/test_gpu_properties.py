"""Property-based GPU parity (hypothesis): random sizes, orders, layouts and
adversarial x mixtures must be bit-identical to the CPU oracle; SPEC
invariants hold on the GPU outputs."""

import numpy as np
import pytest
import torch
from hypothesis import HealthCheck, given, settings, strategies as st

from paper_2504_07637_b200 import boys, boys_ragged, max_order

pytestmark = pytest.mark.gpu

SPECIAL = [0.0, 5e-324, 2.2250738585072014e-308, 1e-300, 1e-12, 0.5, 1.0, 34.38, 57.74, 74.5,
           86.0, 88.0, 100.0, 707.99, 708.0, 708.01, 745.0, 1e4, 1e6, 1e15, 1e18, 1e20, 1e300]


def xs_strategy(max_n=3000):
    finite = st.floats(min_value=0.0, max_value=1e308, allow_nan=False, allow_infinity=False)
    small = st.floats(min_value=0.0, max_value=120.0, allow_nan=False)
    return st.lists(st.one_of(small, small, finite, st.sampled_from(SPECIAL)), min_size=0,
                    max_size=max_n)


@settings(max_examples=60, deadline=None, suppress_health_check=list(HealthCheck))
@given(xs=xs_strategy(), dtype=st.sampled_from([np.float64, np.float32]),
       order=st.integers(min_value=0, max_value=36), layout=st.sampled_from(["soa", "aos"]))
def test_dense_random_bit_exact(oracle, xs, dtype, order, layout):
    n = min(order, max_order(dtype))
    x = np.array(xs, dtype=np.float64)
    if dtype == np.float32:
        x = np.minimum(x, 3.0e38)
    x = x.astype(dtype)
    got = boys(n, torch.from_numpy(x).cuda(), layout=layout).cpu().numpy()
    ref, bad = oracle.dense(n, x, layout)
    assert bad == -1
    assert got.shape == ref.shape
    assert np.array_equal(got.view(np.uint8), ref.view(np.uint8))


@settings(max_examples=40, deadline=None, suppress_health_check=list(HealthCheck))
@given(xs=xs_strategy(2000), dtype=st.sampled_from([np.float64, np.float32]),
       seed=st.integers(0, 2 ** 31), cap=st.sampled_from([2, 12, 16, 36]))
def test_ragged_random_bit_exact(oracle, xs, dtype, seed, cap):
    x = np.array(xs, dtype=np.float64)
    if dtype == np.float32:
        x = np.minimum(x, 3.0e38)
    x = x.astype(dtype)
    nm = np.random.default_rng(seed).integers(0, min(cap, max_order(dtype)) + 1,
                                              size=x.size).astype(np.uint8)
    if x.size == 0:
        return
    got, off = boys_ragged(torch.from_numpy(x).cuda(), torch.from_numpy(nm).cuda())
    ref, roff, bad = oracle.ragged(x, nm)
    assert bad == -1 and np.array_equal(off.cpu().numpy(), roff)
    assert np.array_equal(got.cpu().numpy().view(np.uint8), ref.view(np.uint8))


@settings(max_examples=30, deadline=None, suppress_health_check=list(HealthCheck))
@given(xs=st.lists(st.floats(min_value=1e-6, max_value=1e5, allow_nan=False), min_size=1,
                   max_size=2000), n=st.integers(1, 16))
def test_invariants_on_gpu(xs, n):
    x = torch.tensor(xs, dtype=torch.float64, device="cuda")
    F = boys(n, x).cpu().numpy()
    m = np.arange(n + 1)[:, None]
    big = np.asarray(xs) > 1e4
    ok = F > 0
    assert ok[:, ~big].all()                             # 0 < F_m
    assert (F <= 1.0 / (2 * m + 1)).all()                # F_m <= 1/(2m+1)
    pos = F[1:] > 0
    assert (F[1:][pos] < F[:-1][pos]).all()              # strictly decreasing in m
