"""Boundary behaviour added in round 2, on the GPU, through the C ABI:

* coefficient tables at the boundary: a KernelTable /
  Dataset / dataset path equal to the compiled table takes the compiled
  kernels; a different one (a perturbed dataset) is uploaded and its values
  equal the CPU oracle loaded with the same dataset file, bit for bit;
* the ragged entry with an output that is only element-aligned (out=buf[1:]);
* the linear offsets scan (sizes around its 4096-element tiles, unaligned
  orders, the full cfg4 size);
* boys_shard_error (the per-shard error statistic) against numpy.
"""

import ctypes as C

import numpy as np
import pytest
import torch

from paper_2504_07637_b200 import (EvalRequest, boys, boys_ragged, coeffs as CF, eval_batch,
                                   eval_fn, eval_with_split, ragged_offsets, workloads as W)
from paper_2504_07637_b200 import _lib
from paper_2504_07637_b200.kernel import _table_handle, table_checksum

pytestmark = pytest.mark.gpu


def _perturbed(tmp_path, profile="double53", orders=(3, 5, 8, 16)):
    """The shipped dataset with a few reals moved by a relative 2^-30 (a
    different, still valid table); saved through coeffs.save (checksummed)."""
    ds = CF.load_default(profile)
    for n in orders:
        r = ds.records[n]
        f = (lambda v: float(np.float32(v * (1 + 2.0 ** -20)))) if profile == "single24" \
            else (lambda v: v * (1 + 2.0 ** -30))
        r.q2 = f(r.q2)
        r.c = f(r.c)
        y, a = r.u_quads[0]
        r.u_quads[0] = (f(y), a)
    p = tmp_path / f"perturbed_{profile}.dat"
    CF.save(ds, p)
    return ds, p


def _x(dtype, N=20000, seed=3):
    rng = np.random.default_rng(seed)
    x = np.concatenate([rng.uniform(0, 80, N // 2), np.exp(rng.uniform(-25, 12, N - N // 2))])
    return np.concatenate([[0.0, 1e-300, 30.0, 74.5, 800.0, 1e20], x]).astype(dtype)


def test_compiled_table_checksum_matches_dataset():
    for dt, prof in ((torch.float64, "double53"), (torch.float32, "single24")):
        kt = CF.build_kernel_table(CF.load_default(prof))
        assert table_checksum(dt) == CF.table_checksum(kt)
        # the shipped table, however it is passed, selects the compiled kernels
        for t in (CF.load_default(prof), kt, CF.default_path(prof)):
            assert _table_handle(t, dt, torch.device("cuda")) is None


@pytest.mark.parametrize("layout", ["soa", "aos"])
def test_uploaded_table_matches_oracle_with_that_dataset(oracle, tmp_path, layout):
    ds, path = _perturbed(tmp_path)
    x = _x(np.float64)
    xd = torch.from_numpy(x).cuda()
    for n in (0, 3, 5, 8, 16, 24, 36):
        got = boys(n, xd, layout=layout, table=ds).cpu().numpy()
        ref, bad = oracle.dense(n, x, layout, table_path=path)
        assert bad == -1
        assert np.array_equal(got.view(np.int64), ref.view(np.int64)), n
        base = boys(n, xd, layout=layout).cpu().numpy()
        if n in (3, 5, 8, 16):
            assert not np.array_equal(got, base), f"n={n}: perturbation had no effect"
        else:
            assert np.array_equal(got.view(np.int64), base.view(np.int64)), n


def test_uploaded_table_eval_batch_eval_fn_split(oracle, tmp_path):
    ds, path = _perturbed(tmp_path)
    x = _x(np.float64, N=5000)
    res = eval_batch(EvalRequest(n=8, xs=x, layout="point-major"), table=path)
    ref, _, ex = oracle.dense(8, x, "aos", expx=True, table_path=path)
    assert np.array_equal(res.values.view(np.int64), ref.view(np.int64))
    assert np.array_equal(res.expx.view(np.int64), ex.view(np.int64))
    fn, ex2 = eval_fn(5, torch.from_numpy(x).cuda(), table=CF.build_kernel_table(ds))
    r5, _ = oracle.dense(5, x, "soa", table_path=path)
    assert np.array_equal(fn.cpu().numpy().view(np.int64), r5[5].view(np.int64))
    for lay in ("soa", "aos"):
        sp = eval_with_split(16, 8, torch.from_numpy(x).cuda(), table=ds, layout=lay)
        rs, _ = oracle.split(16, 8, x, lay, table_path=path)
        assert np.array_equal(sp.cpu().numpy().view(np.int64), rs.view(np.int64)), lay


def test_uploaded_table_f32_and_domain(oracle, tmp_path):
    ds, path = _perturbed(tmp_path, "single24", orders=(2, 8))
    x = _x(np.float32)
    got = boys(8, torch.from_numpy(x).cuda(), layout="aos", table=ds).cpu().numpy()
    ref, _ = oracle.dense(8, x, "aos", table_path=path)
    assert np.array_equal(got.view(np.int32), ref.view(np.int32))
    # host input with a custom table keeps float32
    fn, _ = eval_fn(8, x[:100], table=ds)
    assert fn.dtype == torch.float32
    bad = x[:64].copy()
    bad[7] = -1.0
    with pytest.raises(ValueError, match=r"\[7\]"):
        boys(4, torch.from_numpy(bad).cuda(), table=ds)


def test_table_errors(tmp_path):
    ds32, _ = _perturbed(tmp_path, "single24", orders=(2,))
    x = torch.from_numpy(_x(np.float64, N=100)).cuda()
    with pytest.raises(ValueError, match="profile"):
        boys(2, x, table=ds32)                      # single24 table, float64 x
    with pytest.raises(TypeError):
        boys(2, x, table=42)
    ds, _ = _perturbed(tmp_path)
    n = torch.zeros(x.numel(), dtype=torch.uint8, device="cuda")
    with pytest.raises(ValueError, match="compiled table"):
        boys_ragged(x, n, table=ds)
    # a table cut to orders 0..4 rejects higher orders
    short = CF.Dataset(profile="double53", records={k: ds.records[k] for k in range(5)})
    with pytest.raises(ValueError, match="maximum"):
        boys(6, x, table=short)
    # the ABI refuses a wrong row size and out-of-range factor counts
    lib = _lib.load()
    h = C.c_void_p()
    rows = CF.pack_rows(CF.build_kernel_table(ds))
    buf = C.create_string_buffer(rows, len(rows))
    assert lib.boys_table_create(_lib.BOYS_F64, C.cast(buf, C.c_void_p), 37, 300,
                                 C.byref(h)) == _lib.BOYS_E_ARG
    bad = bytearray(rows)
    bad[336:340] = (99).to_bytes(4, "little")       # order 0: u quads = 99
    bb = C.create_string_buffer(bytes(bad), len(bad))
    assert lib.boys_table_create(_lib.BOYS_F64, C.cast(bb, C.c_void_p), 37, 352,
                                 C.byref(h)) == _lib.BOYS_E_ARG


@pytest.mark.parametrize("dtype", [torch.float64, torch.float32])
def test_ragged_element_aligned_out(oracle, dtype):
    x, nm = W.cfg4_batch(1 << 14, chunk=5, device="cuda")
    if dtype == torch.float32:
        keep = nm <= 8
        x, nm = x[keep].to(torch.float32), nm[keep]
    off = ragged_offsets(nm)
    total = int(off[-1].item())
    ref, _, _ = oracle.ragged(x.cpu().numpy(), nm.cpu().numpy())
    for shift in (1, 2, 3):
        buf = torch.full((total + 4,), 7.0, dtype=dtype, device="cuda")
        out = buf[shift:shift + total]
        boys_ragged(x, nm, off, out=out)
        got = buf.cpu().numpy()
        assert np.array_equal(got[shift:shift + total].view(np.uint8), ref.view(np.uint8)), shift
        assert (got[:shift] == 7.0).all() and (got[shift + total:] == 7.0).all()


def test_ragged_strided_offsets_made_contiguous(oracle):
    x, nm = W.cfg4_batch(4096, chunk=6, device="cuda")
    off = ragged_offsets(nm)
    wide = torch.zeros(2 * off.numel(), dtype=torch.int64, device="cuda")
    wide[::2] = off
    got, _ = boys_ragged(x, nm, wide[::2])
    ref, _, _ = oracle.ragged(x.cpu().numpy(), nm.cpu().numpy())
    assert np.array_equal(got.cpu().numpy().view(np.int64), ref.view(np.int64))


@pytest.mark.parametrize("N", [1, 15, 16, 17, 4095, 4096, 4097, 8192, 8192 + 5, (1 << 20) + 3,
                               4096 * 4096, 4096 * 4096 + 4096 * 3 - 1, 3 * 4096 * 1024 + 1])
def test_offsets_scan_sizes(N):
    g = torch.Generator(device="cuda").manual_seed(N)
    nm = torch.randint(0, 37, (N + 1,), generator=g, device="cuda", dtype=torch.uint8)
    for sl in (nm[:N], nm[1:]):                        # 16-byte aligned and unaligned
        got = ragged_offsets(sl).cpu().numpy()
        ref = np.zeros(N + 1, dtype=np.int64)
        np.cumsum(sl.cpu().numpy().astype(np.int64) + 1, out=ref[1:])
        assert np.array_equal(got, ref)


def test_offsets_scan_full_cfg4_size():
    x, nm = W.cfg4_batch(1 << 27, device="cuda")
    del x
    got = ragged_offsets(nm)
    ref = torch.zeros((1 << 27) + 1, dtype=torch.int64, device="cuda")
    torch.cumsum(nm.to(torch.int64) + 1, 0, out=ref[1:])
    assert torch.equal(got, ref)
    # no allocation per call: the launch issues the scan's four kernels only
    # (totals, totals scan, tiles, the tiles overlapping the parked totals)
    l0 = _lib.launch_count()
    ragged_offsets(nm)
    assert _lib.launch_count() - l0 == 4


@pytest.mark.parametrize("dtype", [torch.float64, torch.float32])
def test_shard_error_kernel(dtype):
    rng = np.random.default_rng(11)
    K = 5000
    hi = np.exp(rng.uniform(-60, 60, K))
    if dtype == torch.float32:
        hi = np.exp(rng.uniform(-30, 30, K))
        hi[:10] = 1e-40                              # below FLT_MIN: absolute vs FLT_MIN
    lo = hi * rng.uniform(-1e-17, 1e-17, K)
    vals = (hi * (1 + rng.uniform(-1e-12, 1e-12, K))).astype(np.float64 if dtype == torch.float64
                                                             else np.float32)
    pos = rng.permutation(K).astype(np.int64)
    v = np.empty(K, dtype=vals.dtype)
    v[pos] = vals
    tiny = np.finfo(vals.dtype).tiny
    e = np.abs((vals.astype(np.float64) - hi) - lo)
    ref = (e / np.maximum(np.abs(hi), tiny)).max()
    err = torch.zeros(1, dtype=torch.float64, device="cuda")
    vd = torch.from_numpy(v).cuda()
    pd = torch.from_numpy(pos).cuda()
    gd = torch.from_numpy(np.stack([hi, lo], 1)).cuda()
    dt = _lib.BOYS_F64 if dtype == torch.float64 else _lib.BOYS_F32
    _lib.check(_lib.load().boys_shard_error(dt, C.c_void_p(vd.data_ptr()), C.c_void_p(pd.data_ptr()),
                                            C.c_void_p(gd.data_ptr()), K,
                                            C.c_void_p(err.data_ptr()), None))
    assert float(err.item()) == ref
    # NaN output -> +inf; folding keeps the max
    vd[pos[3]] = float("nan")
    _lib.check(_lib.load().boys_shard_error(dt, C.c_void_p(vd.data_ptr()), C.c_void_p(pd.data_ptr()),
                                            C.c_void_p(gd.data_ptr()), K,
                                            C.c_void_p(err.data_ptr()), None))
    assert float(err.item()) == float("inf")
