"""Fused consumer: McMurchie-Davidson Hermite Coulomb
integrals with F_m consumed in registers (boys_hermite_coulomb), bit-identical
to the CPU restatement (oracle boys_oracle_hermite) for L = 0..4."""

import numpy as np
import pytest
import torch

from paper_2504_07637_b200 import hermite_coulomb, workloads as W
from paper_2504_07637_b200 import _lib

pytestmark = pytest.mark.gpu
DEV = torch.device("cuda:0")


def _pairs(n, seed):
    return W.shell_pairs(n, seed=seed, device=DEV)


@pytest.mark.parametrize("L", [0, 1, 2, 3, 4])
def test_hermite_bit_exact(oracle, L):
    bra, ket = _pairs(37, 1), _pairs(53, 2)           # 1961 quartets: a ragged last tile
    got = hermite_coulomb(L, bra, ket).cpu().numpy()
    ref, bad = oracle.hermite(L, bra.cpu().numpy(), ket.cpu().numpy())
    assert bad == -1
    assert got.shape == ref.shape == (37, 53, (L + 1) * (L + 2) * (L + 3) // 6)
    assert np.array_equal(got.view(np.int64), ref.view(np.int64))


def test_hermite_edges_and_bulk_tiles(oracle):
    # coincident centres (x = 0), far pairs (x past every cut-off, e^-x = 0),
    # many full 128-quartet tiles (bulk stores) plus a tail
    bra, ket = _pairs(300, 3), _pairs(301, 4)
    ket[:5, 1:4] = bra[:5, 1:4]                        # P == Q for some quartets
    ket[5:9, 1:4] += 1e4                               # very large |P - Q|
    got = hermite_coulomb(4, bra, ket).cpu().numpy()
    ref, bad = oracle.hermite(4, bra.cpu().numpy(), ket.cpu().numpy())
    assert bad == -1
    assert np.array_equal(got.view(np.int64), ref.view(np.int64))
    # R_000 = pref F_0 > 0; at P == Q every odd-index term vanishes
    assert np.all(got[:, :, 0] > 0)
    assert np.all(got[0, 0, 1:4] == 0)


def test_hermite_errors_and_nan_rows(oracle):
    bra, ket = _pairs(4, 5), _pairs(3, 6)
    bad_ket = ket.clone()
    bad_ket[1, 0] = -1.0                               # negative exponent
    with pytest.raises(ValueError, match="quartet 1"):
        hermite_coulomb(2, bra, bad_ket)
    out = hermite_coulomb(2, bra, bad_ket, check=False).cpu().numpy()
    assert np.isnan(out[:, 1]).all() and np.isfinite(out[:, [0, 2]]).all()
    with pytest.raises(ValueError, match="lmax"):
        hermite_coulomb(5, bra, ket)
    with pytest.raises(ValueError, match="shape"):
        hermite_coulomb(1, bra[:, :4], ket)
    lib = _lib.load()
    assert lib.boys_hermite_coulomb(9, None, 1, None, 1, None, None, None) == _lib.BOYS_E_ORDER
    empty = torch.empty((0, 5), dtype=torch.float64, device=DEV)
    assert hermite_coulomb(3, empty, ket).shape == (0, 3, 20)


def test_hermite_consumes_the_same_F(oracle):
    """R_000 / pref equals F_0 of the dense evaluator at the same x, bit for
    bit (the fused kernel runs the same Boys evaluator in registers)."""
    from paper_2504_07637_b200 import boys
    bra, ket = _pairs(64, 7), _pairs(64, 8)
    R = hermite_coulomb(0, bra, ket).cpu().numpy()[:, :, 0]
    b, k = bra.cpu().numpy(), ket.cpu().numpy()
    p, q = b[:, None, 0], k[None, :, 0]
    X = b[:, None, 1] - k[None, :, 1]
    Y = b[:, None, 2] - k[None, :, 2]
    Z = b[:, None, 3] - k[None, :, 3]
    pq = p + q
    a = (p * q) / pq

    def fma(u, v, w):                                  # exactly rounded u*v + w
        from fractions import Fraction
        return np.array([float(Fraction(float(i)) * Fraction(float(j)) + Fraction(float(k)))
                         for i, j, k in zip(u.ravel(), v.ravel(), w.ravel())]).reshape(u.shape)

    r2 = fma(Z, Z, fma(Y, Y, X * X))
    x = (a * r2).reshape(-1)
    F0 = boys(0, torch.from_numpy(x).to(DEV)).cpu().numpy()[0].reshape(64, 64)
    pref = (((float.fromhex("0x1.17e50a9dc6553p+5") / ((p * q) * np.sqrt(pq))) * b[:, None, 4]) * k[None, :, 4])
    assert np.array_equal((pref * F0).view(np.int64), R.view(np.int64))
