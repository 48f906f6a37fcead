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


def _boys_device(n_max: int, x: torch.Tensor, layout: str, out, expx: bool, check: bool):
    lay = _layout(layout)
    _check_order(n_max, x.dtype)
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
        L.check(L.load().boys_eval_dense(_DTYPES[x.dtype], n_max, _ptr(xf), N, _ptr(out), lay,
                                         _ptr(ex), _ptr(dom), C.c_void_p(_stream_ptr(x.device))))
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


def boys(n_max: int, x, *, layout: str = "soa", out=None, check: bool = True):
    """F_0..F_{n_max}(x) for every element of x (the batched boys_downward).

    x: CUDA tensor (float64 or float32) -> CUDA tensor, computed on the current
    stream; numpy array / list / CPU tensor -> host result via the pipelined
    host-buffer path.  Shape [n_max+1, N] ('soa') or [N, n_max+1] ('aos').
    ``check=False`` skips the batch domain check (no host sync).
    """
    if isinstance(x, torch.Tensor) and x.is_cuda:
        return _boys_device(n_max, x, layout, out, False, check)[0]
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
    """SPEC.md:316-324.  ``table`` is accepted for signature parity; the
    kernel tables are compiled into libboys (see coeffs.gen_header)."""
    x = req.xs
    if not (isinstance(x, torch.Tensor) and x.is_cuda):
        x = torch.as_tensor(np.asarray(x)).cuda()
        vals, ex = _boys_device(req.n, x, req.layout, None, True, True)
        return EvalResult(values=vals.cpu().numpy(), expx=ex.cpu().numpy())
    vals, ex = _boys_device(req.n, x, req.layout, None, True, True)
    return EvalResult(values=vals, expx=ex)


def eval_fn(n: int, x, table=None):
    """(F_n(x), e^{-x}) for a batch (or a scalar) x."""
    scalar = np.isscalar(x) or (isinstance(x, torch.Tensor) and x.dim() == 0)
    xt = x if isinstance(x, torch.Tensor) and x.is_cuda else torch.as_tensor(
        np.atleast_1d(np.asarray(x, dtype=np.float64))).cuda()
    vals, ex = _boys_device(n, xt.reshape(-1), "soa", None, True, True)
    fn = vals[n]
    if scalar:
        return float(fn[0]), float(ex[0])
    return fn, ex


def eval_with_split(n: int, n_bar: int, x, layout: str = "soa", check: bool = True, out=None):
    """F_{n_bar+1..n} from the order-n seed, F_{0..n_bar} from
    the order-n_bar seed (two recursions).  ``out``: optional preallocated
    device tensor of the result's shape (device inputs only)."""
    xt = x if isinstance(x, torch.Tensor) and x.is_cuda else torch.as_tensor(
        np.asarray(x)).cuda()
    _check_order(n, xt.dtype)
    if not isinstance(n_bar, (int, np.integer)) or not 0 <= n_bar < n:
        raise ValueError(f"need 0 <= n_bar < n, got n_bar={n_bar!r}, n={n}")
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
        L.check(L.load().boys_eval_split(_DTYPES[xt.dtype], n, n_bar, _ptr(xf), N, _ptr(out), lay,
                                         _ptr(dom), C.c_void_p(_stream_ptr(xt.device))))
    if check and int(dom.item()) >= 0:
        _domain_error(xf, int(dom.item()))
    return out if isinstance(x, torch.Tensor) and x.is_cuda else out.cpu().numpy()


def ragged_offsets(n_max: torch.Tensor) -> torch.Tensor:
    """Exclusive prefix sum of n_i + 1 (N+1 entries), computed on the device."""
    nm = n_max.contiguous().reshape(-1)
    if nm.dtype != torch.uint8 or not nm.is_cuda:
        raise ValueError("n_max must be a CUDA uint8 tensor")
    off = torch.empty(nm.numel() + 1, dtype=torch.int64, device=nm.device)
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
                out: torch.Tensor = None, check: bool = True, return_offsets: bool = True):
    """Per-element orders: element i gets F_0..F_{n_max[i]}(x_i) at
    values[offsets[i] : offsets[i+1]].  Returns (values, offsets).

    x on a CUDA device: computed on the current stream (offsets as given, or
    the exclusive prefix sum of n_max + 1).  x (and n_max) on the host: the
    pipelined host-buffer path; results come back on the host, offsets are the
    exclusive prefix sum (None with return_offsets=False)."""
    if not (isinstance(x, torch.Tensor) and x.is_cuda):
        return _boys_ragged_host(x, n_max, out, return_offsets)
    xf = _as_device_x(x)
    nm = n_max.contiguous().reshape(-1)
    if nm.dtype != torch.uint8 or nm.numel() != xf.numel() or nm.device != xf.device:
        raise ValueError("n_max must be a uint8 tensor on x's device with one entry per x")
    if offsets is None:
        offsets = ragged_offsets(nm)
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
