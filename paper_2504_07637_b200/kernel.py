"""Python face of the batched Boys evaluator: the reference's SPEC'd ``kernel``
module over the libboys C ABI.

Reference interface -> here
  eval_batch(EvalRequest{n, xs, layout}, KernelTable) -> EvalResult{values, expx}
                                                     SPEC.md:279-286, 316-324  -> eval_batch
  eval_fn(n, x, table) -> (fn, expx)                 SPEC.md:298-306           -> eval_fn
  eval_with_split(n, n_bar, x, table)                SPEC.md:325-333           -> eval_with_split
  boys_downward(n, x, prec) -> [F_0..F_n]            refmath.py:330-341        -> boys (batched)
  ragged per-element orders                                  -> boys_ragged

Semantics kept from the reference: index m <-> F_m; order checks raise
ValueError (refmath.py:104-108); x must be finite and >= 0, otherwise the
whole batch raises ValueError listing the offending indices (SPEC.md:320,
refmath.py:111-115).  Output dtype = input dtype (float64 / float32).

Device tensors are computed in place on the current CUDA stream; host inputs
(numpy arrays, lists, CPU tensors) go through the pipelined host-buffer entry
point and come back on the host.  There is no CPU implementation here.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import Any

import numpy as np
import torch

from . import _lib as L

_LAYOUTS = {"soa": L.BOYS_SOA, "order-major": L.BOYS_SOA,
            "aos": L.BOYS_AOS, "point-major": L.BOYS_AOS}
_DTYPES = {torch.float64: L.BOYS_F64, torch.float32: L.BOYS_F32}


def _layout(layout: str) -> int:
    try:
        return _LAYOUTS[layout]
    except KeyError:
        raise ValueError(f"unknown layout {layout!r} (use 'soa'/'order-major' or "
                         f"'aos'/'point-major')") from None


def max_order(dtype=torch.float64) -> int:
    dt = _DTYPES.get(_torch_dtype(dtype))
    if dt is None:
        raise ValueError(f"unsupported dtype {dtype}")
    return int(L.load().boys_max_order(dt))


def _torch_dtype(dtype):
    if isinstance(dtype, torch.dtype):
        return dtype
    return {np.dtype(np.float64): torch.float64, np.dtype(np.float32): torch.float32}.get(
        np.dtype(dtype))


def _check_order(n, dtype) -> None:
    if not isinstance(n, (int, np.integer)) or isinstance(n, bool) or n < 0:
        raise ValueError(f"order must be a non-negative integer, got {n!r}")
    mx = max_order(dtype)
    if n > mx:
        raise ValueError(f"order {n} exceeds the supported maximum {mx} for {dtype}")


def _stream_ptr(device) -> int:
    return torch.cuda.current_stream(device).cuda_stream


def _ptr(t: torch.Tensor):
    return C.c_void_p(t.data_ptr()) if t is not None else None


def _domain_error(x: torch.Tensor, first: int):
    xb = x.detach().reshape(-1)
    bad = (~(torch.isfinite(xb) & (xb >= 0))).nonzero().reshape(-1)
    idx = bad[:10].tolist() or [first]
    more = f" (and {bad.numel() - 10} more)" if bad.numel() > 10 else ""
    raise ValueError(f"argument must be finite and >= 0; offending indices {idx}{more}")


def _as_device_x(x) -> torch.Tensor:
    if not isinstance(x, torch.Tensor):
        raise TypeError("expected a torch.Tensor")
    if x.dtype not in _DTYPES:
        raise ValueError(f"x must be float64 or float32, got {x.dtype}")
    return x.contiguous().reshape(-1)


# ----------------------------------------------------------------------------
# coefficient tables at the boundary
# ----------------------------------------------------------------------------

_PROFILE = {torch.float64: "double53", torch.float32: "single24"}
_handles = {}          # (sha256, device index) -> boys_table* (kept for the process)


def _kernel_table(table, dtype):
    """table (coeffs.Dataset / coeffs.KernelTable / dataset path) -> KernelTable
    of dtype's profile; ValueError for another profile or a malformed table."""
    from . import coeffs as CF
    if isinstance(table, (str, bytes)) or hasattr(table, "__fspath__"):
        table = CF.load(table)
    if isinstance(table, CF.Dataset):
        table = CF.build_kernel_table(table)
    if not isinstance(table, CF.KernelTable):
        raise TypeError(f"table must be a coeffs.Dataset, coeffs.KernelTable or a dataset path, "
                        f"got {type(table).__name__}")
    want = _PROFILE[dtype]
    if table.profile != want:
        raise ValueError(f"table profile {table.profile!r} does not match {dtype} "
                         f"(needs {want!r})")
    return table


def table_checksum(dtype=torch.float64) -> str:
    """SHA-256 of the compiled-in table (coeffs.table_checksum of the shipped dataset)."""
    dt = _DTYPES[_torch_dtype(dtype)]
    return L.load().boys_table_checksum(dt).decode()


def _table_handle(table, dtype, device):
    """None -> the compiled tables; a table equal to them (same checksum) ->
    None as well; any other table -> a device copy (uploaded once per device)."""
    if table is None:
        return None
    from . import coeffs as CF
    kt = _kernel_table(table, dtype)
    digest = CF.table_checksum(kt)
    if digest == table_checksum(dtype):
        return None
    key = (digest, torch.device(device).index)
    h = _handles.get(key)
    if h is None:
        rows = CF.pack_rows(kt)
        lib = L.load()
        nb = lib.boys_table_row_bytes(_DTYPES[dtype])
        if nb * len(kt.rows) != len(rows):
            raise ValueError("table row layout does not match libboys")
        buf = C.create_string_buffer(rows, len(rows))
        hp = C.c_void_p()
        with torch.cuda.device(device):
            L.check(lib.boys_table_create(_DTYPES[dtype], C.cast(buf, C.c_void_p), len(kt.rows),
                                          nb, C.byref(hp)))
        h = _handles[key] = hp
    return h


def _boys_device(n_max: int, x: torch.Tensor, layout: str, out, expx: bool, check: bool,
                 table=None):
    lay = _layout(layout)
    _check_order(n_max, x.dtype)
    th = _table_handle(table, x.dtype, x.device)
    if th is not None and n_max > L.load().boys_table_max_order(th):
        raise ValueError(f"order {n_max} exceeds the table's maximum "
                         f"{L.load().boys_table_max_order(th)}")
    xf = _as_device_x(x)
    N = xf.numel()
    shape = (n_max + 1, N) if lay == L.BOYS_SOA else (N, n_max + 1)
    if out is None:
        out = torch.empty(shape, dtype=x.dtype, device=x.device)
    elif (tuple(out.shape) != shape or out.dtype != x.dtype or out.device != x.device
          or not out.is_contiguous()):
        raise ValueError(f"out must be a contiguous {x.dtype} tensor of shape {shape}")
    ex = torch.empty(N, dtype=x.dtype, device=x.device) if expx else None
    dom = torch.full((1,), -1, dtype=torch.int64, device=x.device) if check else None
    with torch.cuda.device(x.device):
        if th is None:
            L.check(L.load().boys_eval_dense(_DTYPES[x.dtype], n_max, _ptr(xf), N, _ptr(out),
                                             lay, _ptr(ex), _ptr(dom),
                                             C.c_void_p(_stream_ptr(x.device))))
        else:
            L.check(L.load().boys_eval_dense_table(th, n_max, _ptr(xf), N, _ptr(out), lay,
                                                   _ptr(ex), _ptr(dom),
                                                   C.c_void_p(_stream_ptr(x.device))))
    if check:
        first = int(dom.item())
        if first >= 0:
            _domain_error(xf, first)
    return out, ex


def _boys_host(n_max: int, x, layout: str, out):
    lay = _layout(layout)
    was_tensor = isinstance(x, torch.Tensor)
    xn = x.detach().cpu().numpy() if was_tensor else np.asarray(x)
    if xn.dtype not in (np.float64, np.float32):
        xn = xn.astype(np.float64)
    xn = np.ascontiguousarray(xn.reshape(-1))
    _check_order(n_max, xn.dtype)
    N = xn.size
    shape = (n_max + 1, N) if lay == L.BOYS_SOA else (N, n_max + 1)
    if out is None:
        res = np.empty(shape, dtype=xn.dtype)
    else:
        res = out.numpy() if isinstance(out, torch.Tensor) else out
        if res.shape != shape or res.dtype != xn.dtype or not res.flags.c_contiguous:
            raise ValueError(f"out must be a contiguous {xn.dtype} array of shape {shape}")
    if not torch.cuda.is_available():
        raise RuntimeError("libboys needs a CUDA device (there is no CPU implementation)")
    first = C.c_int64(-1)
    code = L.load().boys_eval_dense_host(
        L.BOYS_F64 if xn.dtype == np.float64 else L.BOYS_F32, n_max,
        xn.ctypes.data_as(C.c_void_p), N, res.ctypes.data_as(C.c_void_p), lay, C.byref(first))
    if code == L.BOYS_E_DOMAIN:
        bad = np.nonzero(~(np.isfinite(xn) & (xn >= 0)))[0]
        raise ValueError(f"argument must be finite and >= 0; offending indices "
                         f"{bad[:10].tolist()}" + (f" (and {bad.size - 10} more)"
                                                     if bad.size > 10 else ""))
    L.check(code)
    if out is not None:
        return out
    return torch.from_numpy(res) if was_tensor else res


def _to_device(x):
    """Host input (numpy / list / scalar / CPU tensor) -> CUDA tensor, keeping
    float32 and float64 (anything else becomes float64)."""
    if isinstance(x, torch.Tensor):
        t = x.detach()
        if t.dtype not in _DTYPES:
            t = t.to(torch.float64)
        return t.cuda()
    a = np.asarray(x)
    if a.dtype not in (np.float64, np.float32):
        a = a.astype(np.float64)
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def boys(n_max: int, x, *, layout: str = "soa", out=None, check: bool = True, table=None):
    """F_0..F_{n_max}(x) for every element of x (the batched boys_downward).

    x: CUDA tensor (float64 or float32) -> CUDA tensor, computed on the current
    stream; numpy array / list / CPU tensor -> host result via the pipelined
    host-buffer path.  Shape [n_max+1, N] ('soa') or [N, n_max+1] ('aos').
    ``check=False`` skips the batch domain check (no host sync).  ``table``:
    a coeffs.Dataset / KernelTable / dataset path; None or the compiled table
    -> the compiled kernels, any other -> the uploaded-table path.
    """
    if isinstance(x, torch.Tensor) and x.is_cuda:
        return _boys_device(n_max, x, layout, out, False, check, table)[0]
    if table is not None:
        dt = _torch_dtype(np.asarray(x).dtype if not isinstance(x, torch.Tensor) else x.dtype)
        if _table_handle(table, dt or torch.float64, torch.device("cuda")) is not None:
            xd = _to_device(x)
            res = _boys_device(n_max, xd, layout, None, False, check, table)[0].cpu()
            if out is not None:
                (out if isinstance(out, torch.Tensor) else torch.from_numpy(out)).copy_(res)
                return out
            return res if isinstance(x, torch.Tensor) else res.numpy()
    return _boys_host(n_max, x, layout, out)


@dataclass(frozen=True)
class EvalRequest:
    """order n, arguments xs, layout."""

    n: int
    xs: Any
    layout: str = "order-major"


@dataclass
class EvalResult:
    """values (n+1) x |xs| (or |xs| x (n+1)) and e^{-x}."""

    values: Any
    expx: Any


def eval_batch(req: EvalRequest, table=None) -> EvalResult:
    """SPEC.md:316-324.  ``table`` (coeffs.Dataset / KernelTable / dataset
    path): None or the compiled table -> the compiled kernels; a different
    table is uploaded once and evaluated by the run-time-table kernel."""
    x = req.xs
    if not (isinstance(x, torch.Tensor) and x.is_cuda):
        x = _to_device(x)
        vals, ex = _boys_device(req.n, x, req.layout, None, True, True, table)
        return EvalResult(values=vals.cpu().numpy(), expx=ex.cpu().numpy())
    vals, ex = _boys_device(req.n, x, req.layout, None, True, True, table)
    return EvalResult(values=vals, expx=ex)


def eval_fn(n: int, x, table=None):
    """(F_n(x), e^{-x}) for a batch (or a scalar) x, in x's
    dtype (float32 stays float32)."""
    scalar = np.isscalar(x) or (isinstance(x, torch.Tensor) and x.dim() == 0)
    if isinstance(x, torch.Tensor) and x.is_cuda:
        xt = x
    elif isinstance(x, torch.Tensor):
        xt = _to_device(x.reshape(-1))
    else:
        xt = _to_device(np.atleast_1d(np.asarray(x)))
    vals, ex = _boys_device(n, xt.reshape(-1), "soa", None, True, True, table)
    fn = vals[n]
    if scalar:
        return float(fn[0]), float(ex[0])
    return fn, ex


def eval_with_split(n: int, n_bar: int, x, table=None, layout: str = "soa", check: bool = True,
                    out=None):
    """F_{n_bar+1..n} from the order-n seed, F_{0..n_bar} from
    the order-n_bar seed (two recursions).  ``table`` as in eval_batch.
    ``out``: optional preallocated device tensor of the result's shape
    (device inputs only)."""
    xt = x if isinstance(x, torch.Tensor) and x.is_cuda else _to_device(x)
    _check_order(n, xt.dtype)
    if not isinstance(n_bar, (int, np.integer)) or not 0 <= n_bar < n:
        raise ValueError(f"need 0 <= n_bar < n, got n_bar={n_bar!r}, n={n}")
    th = _table_handle(table, xt.dtype, xt.device)
    if th is not None and n > L.load().boys_table_max_order(th):
        raise ValueError(f"order {n} exceeds the table's maximum "
                         f"{L.load().boys_table_max_order(th)}")
    lay = _layout(layout)
    xf = _as_device_x(xt)
    N = xf.numel()
    shape = (n + 1, N) if lay == L.BOYS_SOA else (N, n + 1)
    if out is None:
        out = torch.empty(shape, dtype=xt.dtype, device=xt.device)
    elif (tuple(out.shape) != shape or out.dtype != xt.dtype or out.device != xt.device
          or not out.is_contiguous()):
        raise ValueError(f"out must be a contiguous {xt.dtype} tensor of shape {shape}")
    dom = torch.full((1,), -1, dtype=torch.int64, device=xt.device) if check else None
    with torch.cuda.device(xt.device):
        if th is None:
            L.check(L.load().boys_eval_split(_DTYPES[xt.dtype], n, n_bar, _ptr(xf), N, _ptr(out),
                                             lay, _ptr(dom), C.c_void_p(_stream_ptr(xt.device))))
        else:
            L.check(L.load().boys_eval_split_table(th, n, n_bar, _ptr(xf), N, _ptr(out), lay,
                                                   _ptr(dom), C.c_void_p(_stream_ptr(xt.device))))
    if check and int(dom.item()) >= 0:
        _domain_error(xf, int(dom.item()))
    return out if isinstance(x, torch.Tensor) and x.is_cuda else out.cpu().numpy()


def ragged_offsets(n_max: torch.Tensor, out: torch.Tensor = None) -> torch.Tensor:
    """Exclusive prefix sum of n_i + 1 (N+1 entries), computed on the device.
    ``out``: optional preallocated contiguous int64 tensor of N+1 entries."""
    nm = n_max.contiguous().reshape(-1)
    if nm.dtype != torch.uint8 or not nm.is_cuda:
        raise ValueError("n_max must be a CUDA uint8 tensor")
    if out is None:
        off = torch.empty(nm.numel() + 1, dtype=torch.int64, device=nm.device)
    else:
        if (out.dtype != torch.int64 or out.numel() != nm.numel() + 1 or out.device != nm.device
                or not out.is_contiguous()):
            raise ValueError("out must be a contiguous int64 tensor of N+1 entries on n_max's device")
        off = out.reshape(-1)
    with torch.cuda.device(nm.device):
        L.check(L.load().boys_ragged_offsets(_ptr(nm), nm.numel(), _ptr(off),
                                             C.c_void_p(_stream_ptr(nm.device))))
    return off


def _boys_ragged_host(x, n_max, out, return_offsets: bool):
    """Host buffers -> boys_eval_ragged_host (pipelined copies + kernel).  The
    offsets are the exclusive prefix sum of n_max + 1 (include/boys.h)."""
    was_tensor = isinstance(x, torch.Tensor)
    xn = x.detach().cpu().numpy() if was_tensor else np.asarray(x)
    if xn.dtype not in (np.float64, np.float32):
        xn = xn.astype(np.float64)
    xn = np.ascontiguousarray(xn.reshape(-1))
    nn = n_max.detach().cpu().numpy() if isinstance(n_max, torch.Tensor) else np.asarray(n_max)
    nn = np.ascontiguousarray(nn.reshape(-1))
    if nn.dtype != np.uint8 or nn.size != xn.size:
        raise ValueError("n_max must be a uint8 array with one entry per x")
    N = xn.size
    if out is None:
        res = np.empty(int(nn.sum(dtype=np.int64)) + N, dtype=xn.dtype)
    else:
        res = out.numpy() if isinstance(out, torch.Tensor) else out
        if res.dtype != xn.dtype or res.ndim != 1 or not res.flags.c_contiguous:
            raise ValueError(f"out must be a contiguous 1-D {xn.dtype} array")
    if not torch.cuda.is_available():
        raise RuntimeError("libboys needs a CUDA device (there is no CPU implementation)")
    first = C.c_int64(-1)
    code = L.load().boys_eval_ragged_host(
        L.BOYS_F64 if xn.dtype == np.float64 else L.BOYS_F32, xn.ctypes.data_as(C.c_void_p),
        nn.ctypes.data_as(C.c_void_p), N, res.ctypes.data_as(C.c_void_p), res.size, C.byref(first))
    if code == L.BOYS_E_DOMAIN:
        i = int(first.value)
        mx = max_order(torch.float64 if xn.dtype == np.float64 else torch.float32)
        if int(nn[i]) > mx:
            raise ValueError(f"order {int(nn[i])} at index {i} exceeds the supported maximum {mx}")
        bad = np.nonzero(~(np.isfinite(xn) & (xn >= 0)))[0]
        raise ValueError(f"argument must be finite and >= 0; offending indices "
                         f"{bad[:10].tolist()}" + (f" (and {bad.size - 10} more)"
                                                     if bad.size > 10 else ""))
    if code == L.BOYS_E_ARG and out is not None:
        raise ValueError("out holds fewer values than sum(n_max + 1)")
    L.check(code)
    off = None
    if return_offsets:
        off = np.zeros(N + 1, dtype=np.int64)
        np.cumsum(nn.astype(np.int64) + 1, out=off[1:])
    vals = out if out is not None else (torch.from_numpy(res) if was_tensor else res)
    if was_tensor and off is not None:
        off = torch.from_numpy(off)
    return vals, off


def boys_ragged(x: torch.Tensor, n_max: torch.Tensor, offsets: torch.Tensor = None, *,
                out: torch.Tensor = None, check: bool = True, return_offsets: bool = True,
                table=None):
    """Per-element orders: element i gets F_0..F_{n_max[i]}(x_i) at
    values[offsets[i] : offsets[i+1]].  Returns (values, offsets).

    x on a CUDA device: computed on the current stream (offsets as given, or
    the exclusive prefix sum of n_max + 1).  x (and n_max) on the host: the
    pipelined host-buffer path; results come back on the host, offsets are the
    exclusive prefix sum (None with return_offsets=False).  ``table``: ragged
    batches run the compiled tables only; a different table raises ValueError."""
    if table is not None:
        dt = x.dtype if isinstance(x, torch.Tensor) else _torch_dtype(np.asarray(x).dtype)
        if _table_handle(table, dt or torch.float64, torch.device("cuda")) is not None:
            raise ValueError("ragged batches evaluate the compiled table only; use eval_batch "
                             "per order for a different table")
    if not (isinstance(x, torch.Tensor) and x.is_cuda):
        return _boys_ragged_host(x, n_max, out, return_offsets)
    xf = _as_device_x(x)
    nm = n_max.contiguous().reshape(-1)
    if nm.dtype != torch.uint8 or nm.numel() != xf.numel() or nm.device != xf.device:
        raise ValueError("n_max must be a uint8 tensor on x's device with one entry per x")
    if offsets is None:
        offsets = ragged_offsets(nm)
    else:
        offsets = offsets.contiguous().reshape(-1)
    if offsets.dtype != torch.int64 or offsets.numel() != xf.numel() + 1 or \
            offsets.device != xf.device:
        raise ValueError("offsets must be an int64 tensor of N+1 entries on x's device")
    if out is None:
        out = torch.empty(int(offsets[-1].item()), dtype=xf.dtype, device=xf.device)
    else:
        if out.dtype != xf.dtype or out.device != xf.device or not out.is_contiguous():
            raise ValueError(f"out must be a contiguous {xf.dtype} tensor on x's device")
        # check=True already synchronises for the domain flag; the size check
        # (one 8-byte read) keeps a short `out` from being written past its end.
        # check=False: the caller guarantees out.numel() >= offsets[-1].
        if check and out.numel() < int(offsets[-1].item()):
            raise ValueError("out holds fewer values than offsets[-1]")
    dom = torch.full((1,), -1, dtype=torch.int64, device=xf.device) if check else None
    with torch.cuda.device(xf.device):
        L.check(L.load().boys_eval_ragged(_DTYPES[xf.dtype], _ptr(xf), _ptr(nm), _ptr(offsets),
                                          xf.numel(), _ptr(out), _ptr(dom),
                                          C.c_void_p(_stream_ptr(xf.device))))
    if check and int(dom.item()) >= 0:
        first = int(dom.item())
        mx = max_order(xf.dtype)
        if int(nm[first].item()) > mx:
            raise ValueError(f"order {int(nm[first].item())} at index {first} exceeds the "
                             f"supported maximum {mx}")
        _domain_error(xf, first)
    return out, offsets


def hermite_coulomb(lmax: int, bra: torch.Tensor, ket: torch.Tensor, *, out: torch.Tensor = None,
                    check: bool = True) -> torch.Tensor:
    """Fused consumer of F_m (SPEC.md:16, 353 name downstream
    integral code as the caller): McMurchie-Davidson Hermite Coulomb integrals
    for every (bra pair, ket pair), with F_0..F_L evaluated and consumed in
    registers (include/boys.h boys_hermite_coulomb).  lmax = L of the formulas.

    bra: [Nb, 5], ket: [Nk, 5] float64 CUDA tensors of pair records
    (p, Px, Py, Pz, K).  Returns [Nb, Nk, NH] with NH = (L+1)(L+2)(L+3)/6:
    2 pi^{5/2} / (p q sqrt(p+q)) K_i K_j R_{tuv}(a = pq/(p+q), P-Q), t+u+v <= L,
    canonical order (t+u+v ascending, then t descending, then u descending)."""
    if not isinstance(lmax, (int, np.integer)) or not 0 <= lmax <= 4:
        raise ValueError(f"lmax must be an integer in [0, 4], got {lmax!r}")
    for name, t in (("bra", bra), ("ket", ket)):
        if (not isinstance(t, torch.Tensor) or not t.is_cuda or t.dtype != torch.float64
                or t.dim() != 2 or t.shape[1] != 5):
            raise ValueError(f"{name} must be a float64 CUDA tensor of shape [N, 5]")
    if bra.device != ket.device:
        raise ValueError("bra and ket must be on the same device")
    bra, ket = bra.contiguous(), ket.contiguous()
    NH = (lmax + 1) * (lmax + 2) * (lmax + 3) // 6
    shape = (bra.shape[0], ket.shape[0], NH)
    if out is None:
        out = torch.empty(shape, dtype=torch.float64, device=bra.device)
    elif (tuple(out.shape) != shape or out.dtype != torch.float64 or out.device != bra.device
          or not out.is_contiguous()):
        raise ValueError(f"out must be a contiguous float64 tensor of shape {shape}")
    dom = torch.full((1,), -1, dtype=torch.int64, device=bra.device) if check else None
    with torch.cuda.device(bra.device):
        L.check(L.load().boys_hermite_coulomb(int(lmax), _ptr(bra), bra.shape[0], _ptr(ket), ket.shape[0],
                                              _ptr(out), _ptr(dom), C.c_void_p(_stream_ptr(bra.device))))
    if check and int(dom.item()) >= 0:
        q = int(dom.item())
        raise ValueError(f"invalid pair data (x not finite/non-negative, or exponent <= 0) at "
                         f"quartet {q} (bra {q // ket.shape[0]}, ket {q % ket.shape[0]})")
    return out
