"""Parity at BASELINE.json's full sizes: EVERY output byte against the CPU oracle.

For every configuration at its stated size:
  * the whole output is compared byte for byte with the oracle (oracle/,
    OpenMP on the host), slice by slice (2^22 points per slice, so host
    memory stays bounded): cfg1, cfg2, cfg3, cfg4 (fp64 and the fp32 n <= 8
    subset) in full, cfg5 on four of its sixteen 2^26-point chunks (the chunk
    plan of the sharded sweep covers all sixteen, see below);
  * SPEC invariants over all outputs: 0 < F_m <= 1/(2m+1) for
    representable values, F_{m+1} < F_m;
  * shard invariance: evaluating the two halves separately gives the same
    bytes as evaluating the whole batch (the multi-GPU contiguous split);
  * config 5: the sharded chunk plan covers 2^30 points exactly once and the
    per-chunk checksums are independent of the number of ranks.
"""

import numpy as np
import pytest
import torch

from paper_2504_07637_b200 import boys, boys_ragged, shard as S, workloads as W

pytestmark = pytest.mark.gpu

DEV = torch.device("cuda:0")
SLICE = 1 << 22


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


def _bytes_equal(got: np.ndarray, ref: np.ndarray, what: str):
    assert got.shape == ref.shape and got.dtype == ref.dtype, what
    it = np.int64 if got.dtype.itemsize == 8 else np.int32
    g, r = got.reshape(-1).view(it), ref.reshape(-1).view(it)
    if not np.array_equal(g, r):
        bad = np.nonzero(g != r)[0]
        raise AssertionError(f"{what}: {bad.size} values differ, first at flat index {bad[0]}")


def _whole_output_exact(oracle, n, x, F, layout, what):
    """Every output of F (device, layout as given) against the oracle."""
    N = x.numel()
    for a in range(0, N, SLICE):
        b = min(N, a + SLICE)
        ref, bad = oracle.dense(n, x[a:b].cpu().numpy(), layout)
        assert bad == -1
        got = (F[:, a:b] if layout == "soa" else F[a:b]).contiguous().cpu().numpy()
        _bytes_equal(got, ref, f"{what} points [{a}, {b})")


@pytest.mark.parametrize("cfg", ["cfg1", "cfg2", "cfg3"])
def test_dense_configs_full_size(oracle, cfg):
    c = W.CONFIGS[cfg]
    x = W.config_x(cfg, device=DEV)
    assert x.numel() == c.N
    F = boys(c.n_max, x, layout=c.layout)
    rows = F if c.layout == "soa" else F.t()
    _invariants(rows)
    _whole_output_exact(oracle, c.n_max, x, F, c.layout, cfg)
    h = c.N // 2                                      # shard invariance (2 ranks)
    a = boys(c.n_max, x[:h], layout=c.layout)
    b = boys(c.n_max, x[h:], layout=c.layout)
    whole = torch.cat([a, b], dim=1 if c.layout == "soa" else 0)
    assert torch.equal(whole.view(torch.int64), F.view(torch.int64))
    del F, a, b, whole
    torch.cuda.empty_cache()


def test_cfg5_sharded_sweep_full_size(oracle):
    """2^30 points in 2^26 chunks: each chunk evaluated, properties on every
    fifth chunk, every output byte of chunks 0, 3, 12 and 15 against the oracle,
    per-chunk checksums identical for 1/2/4/8-rank chunk plans."""
    N, ch = 1 << 30, W.CHUNK
    out = torch.empty((ch, 13), dtype=torch.float64, device=DEV)
    sums = {}
    for cid in range(N // ch):
        x = W.config_x("cfg5", n=ch, chunk=cid, device=DEV)
        boys(12, x, layout="aos", out=out)
        if cid % 5 == 0:
            _invariants(out.t())
        if cid in (0, 3, 12, 15):
            _whole_output_exact(oracle, 12, x, out, "aos", f"cfg5 chunk {cid}")
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
    # every element, slice by slice: bit-identical to the oracle's ragged evaluation
    offc = off.cpu().numpy()
    N = x.numel()
    for a in range(0, N, SLICE):
        b = min(N, a + SLICE)
        ref, roff, bad = oracle.ragged(x[a:b].cpu().numpy(), nm[a:b].cpu().numpy())
        assert bad == -1
        assert np.array_equal(offc[a:b + 1] - offc[a], roff)
        got = vals[int(offc[a]):int(offc[b])].cpu().numpy()
        _bytes_equal(got, ref, f"{tag} elements [{a}, {b})")
    # shard invariance: two halves (with their own offsets) reproduce the bytes
    h = x.numel() // 2
    va, oa = boys_ragged(x[:h], nm[:h])
    vb, ob = boys_ragged(x[h:], nm[h:])
    assert torch.equal(torch.cat([va, vb]).view(torch.int32 if vals.dtype == torch.float32
                                                else torch.int64),
                       vals.view(torch.int32 if vals.dtype == torch.float32 else torch.int64))
