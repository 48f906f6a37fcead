"""Parity at BASELINE.json's full sizes through size-independent properties.

For every configuration at its stated size:
  * SPEC invariants over ALL outputs: 0 < F_m <= 1/(2m+1) for
    representable values, F_{m+1} < F_m;
  * a random subsample of 2^16 points is bit-identical to the CPU oracle;
  * shard invariance: evaluating the two halves separately gives the same
    bytes as evaluating the whole batch (the multi-GPU contiguous split);
  * config 5: the sharded chunk plan covers 2^30 points exactly once and the
    per-chunk checksums are independent of the number of ranks.
"""

import numpy as np
import pytest
import torch

from paper_2504_07637_b200 import boys, boys_ragged, ragged_offsets, shard as S, workloads as W

pytestmark = pytest.mark.gpu

DEV = torch.device("cuda:0")


def _invariants(F_rows):
    """F_rows: [n+1, N] tensor (any dtype) on the device."""
    n1 = F_rows.shape[0]
    m = torch.arange(n1, device=F_rows.device, dtype=F_rows.dtype)[:, None]
    tiny = torch.finfo(F_rows.dtype).tiny
    rep = F_rows >= tiny
    assert bool(torch.all((F_rows >= 0))), "negative value"
    assert bool(torch.all(F_rows[rep] <= (1.0 / (2 * m + 1)).expand_as(F_rows)[rep]))
    both = rep[1:] & rep[:-1]
    assert bool(torch.all(F_rows[1:][both] < F_rows[:-1][both])), "not decreasing in m"


def _subsample_exact(oracle, n, x, got_rows, k=1 << 16, seed=0):
    idx = np.sort(np.random.default_rng(seed).choice(x.numel(), size=min(k, x.numel()),
                                                     replace=False))
    xi = x[torch.from_numpy(idx).to(x.device)].cpu().numpy()
    ref, bad = oracle.dense(n, xi, "soa")
    assert bad == -1
    g = got_rows[:, torch.from_numpy(idx).to(x.device)].cpu().numpy()
    assert np.array_equal(g.view(np.uint8), ref.view(np.uint8))


@pytest.mark.parametrize("cfg", ["cfg1", "cfg2", "cfg3"])
def test_dense_configs_full_size(oracle, cfg):
    c = W.CONFIGS[cfg]
    x = W.config_x(cfg, device=DEV)
    assert x.numel() == c.N
    F = boys(c.n_max, x, layout=c.layout)
    rows = F if c.layout == "soa" else F.t()
    _invariants(rows)
    _subsample_exact(oracle, c.n_max, x, rows)
    h = c.N // 2                                      # shard invariance (2 ranks)
    a = boys(c.n_max, x[:h], layout=c.layout)
    b = boys(c.n_max, x[h:], layout=c.layout)
    whole = torch.cat([a, b], dim=1 if c.layout == "soa" else 0)
    assert torch.equal(whole.view(torch.int64), F.view(torch.int64))
    del F, a, b, whole
    torch.cuda.empty_cache()


def test_cfg5_sharded_sweep_full_size(oracle):
    """2^30 points in 2^26 chunks: each chunk evaluated, properties on every
    chunk, per-chunk checksums identical for 1/2/4/8-rank chunk plans."""
    N, ch = 1 << 30, W.CHUNK
    out = torch.empty((ch, 13), dtype=torch.float64, device=DEV)
    sums = {}
    for cid in range(N // ch):
        x = W.config_x("cfg5", n=ch, chunk=cid, device=DEV)
        boys(12, x, layout="aos", out=out)
        if cid % 5 == 0:
            _invariants(out.t())
        if cid == 3:
            _subsample_exact(oracle, 12, x, out.t(), k=1 << 15, seed=cid)
        sums[cid] = float(out[:, 0].sum()) + float(out[:, 12].sum())
    for world in (1, 2, 4, 8):
        seen = []
        for r in range(world):
            seen += [cid for cid, lo, hi in S.chunk_plan(N, r, world, ch)]
        assert seen == list(range(N // ch))
    # a rank-2 plan recomputes its chunks bit-identically
    for cid, lo, hi in S.chunk_plan(N, 1, 2, ch)[:2]:
        x = W.config_x("cfg5", n=ch, chunk=cid, device=DEV)
        boys(12, x, layout="aos", out=out)
        assert float(out[:, 0].sum()) + float(out[:, 12].sum()) == sums[cid]


@pytest.mark.parametrize("tag", ["cfg4", "cfg4f32"])
def test_ragged_config_full_size(oracle, tag):
    c = W.CONFIGS[tag]
    x, nm = (W.cfg4f32_batch if tag == "cfg4f32" else W.cfg4_batch)(c.N, device=DEV)
    vals, off = boys_ragged(x, nm)
    assert int(off[-1]) == vals.numel()
    assert bool(torch.all(vals >= 0))
    # subsample of elements: bit-identical to the oracle's ragged evaluation
    idx = np.sort(np.random.default_rng(7).choice(x.numel(), size=1 << 15, replace=False))
    ti = torch.from_numpy(idx).to(DEV)
    xs, ns = x[ti].cpu().numpy(), nm[ti].cpu().numpy()
    ref, roff, bad = oracle.ragged(xs, ns)
    assert bad == -1
    offc = off.cpu().numpy()
    got = vals.cpu().numpy()
    for j, i in enumerate(idx):
        assert np.array_equal(got[offc[i]:offc[i + 1]].view(np.uint8),
                              ref[roff[j]:roff[j + 1]].view(np.uint8))
    # shard invariance: two halves (with their own offsets) reproduce the bytes
    h = x.numel() // 2
    va, oa = boys_ragged(x[:h], nm[:h])
    vb, ob = boys_ragged(x[h:], nm[h:])
    assert torch.equal(torch.cat([va, vb]).view(torch.int32 if vals.dtype == torch.float32
                                                else torch.int64),
                       vals.view(torch.int32 if vals.dtype == torch.float32 else torch.int64))
