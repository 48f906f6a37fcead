"""GPU outputs against the reference oracle's golden vectors (refmath
boys_downward at Precision(96)), to the paper's Table I bars (eps_bar - 2)."""

import numpy as np
import pytest
import torch

import accuracy as A
from paper_2504_07637_b200 import boys, boys_ragged

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("tag,dtype", [("f64", np.float64), ("f32", np.float32)])
def test_table1_scans_on_gpu(tag, dtype):
    d = A.load(f"scan_{tag}.npz")
    for key in d.files:
        if not key.startswith("x"):
            continue
        n = int(key[1:])
        x = d[key].astype(dtype)
        gold = d[f"F{n}"]
        got = boys(n, torch.from_numpy(x).cuda(), layout="aos").cpu().numpy()
        bits = [A.bits(A.rel_err(got[:, m], gold[:, m], dtype)) for m in range(n + 1)]
        for m, b in enumerate(bits):
            assert b >= A.bar(n, m, dtype), f"{tag} n={n} m={m}: {b:.2f}"
        assert bits[0] >= bits[n] - 1     # recursion improves accuracy (acceptance 7)


@pytest.mark.parametrize("name,n", [("cfg1", 0), ("cfg2", 8), ("cfg3", 16), ("cfg5", 12)])
def test_config_samples_on_gpu(name, n):
    d = A.load("configs.npz")
    x, gold = d[f"{name}_x"], d[f"{name}_F"]
    got = boys(n, torch.from_numpy(x).cuda(), layout="soa").cpu().numpy().T
    ok = A.representable(gold, np.float64)
    for m in range(n + 1):
        r = A.rel_err(got[:, m], gold[:, m])[ok[:, m]]
        assert A.bits(r) >= A.bar(n, m, np.float64), f"{name} F_{m}"


@pytest.mark.parametrize("tag,dtype", [("cfg4", np.float64), ("cfg4f32", np.float32)])
def test_ragged_sample_on_gpu(tag, dtype):
    d = A.load("configs.npz")
    x, nm, gold = d[f"{tag}_x"].astype(dtype), d[f"{tag}_n"], d[f"{tag}_F"]
    got, off = boys_ragged(torch.from_numpy(x).cuda(), torch.from_numpy(nm).cuda())
    got, off = got.cpu().numpy(), off.cpu().numpy()
    r = A.rel_err(got, gold, dtype)
    for i in range(x.size):
        n = int(nm[i])
        for m in range(n + 1):
            k = off[i] + m
            if dtype == np.float64 and abs(gold[k, 0]) < np.finfo(np.float64).tiny:
                continue
            assert A.bits(r[k:k + 1]) >= A.bar(n, m, dtype), f"elem {i} n={n} m={m}"
