"""Data-parallel sharding of a Boys sweep across ranks (BASELINE config 5).

The x array partitions into independent points, so ranks own contiguous
shards and exchange nothing on the data path.  The only
collective is a gather of one fp64 per rank: the shard's max relative error
against a golden subsample (reference-oracle values uploaded before timing),
reduced to the job maximum on every rank.

One process per GPU (torchrun); the process group is set up by the caller
(``nccl`` on GPUs, ``gloo`` in the CPU tests).
"""

from __future__ import annotations

from dataclasses import dataclass, field
from typing import Callable, Optional

import torch

CHUNK = 1 << 26


def shard_range(N: int, rank: int, world: int) -> tuple:
    """Contiguous [lo, hi) of rank `rank`; sizes differ by at most one."""
    if not 0 <= rank < world:
        raise ValueError(f"rank {rank} outside world {world}")
    base, rem = divmod(N, world)
    lo = rank * base + min(rank, rem)
    return lo, lo + base + (1 if rank < rem else 0)


def chunk_plan(N: int, rank: int, world: int, chunk: int = CHUNK) -> list:
    """The rank's contiguous slice as (chunk_id, lo, hi) pieces, each inside a
    single global chunk so every piece can be regenerated from its
    (seed, chunk_id) key alone (shard-invariant inputs)."""
    lo, hi = shard_range(N, rank, world)
    out = []
    while lo < hi:
        cid = lo // chunk
        end = min(hi, (cid + 1) * chunk)
        out.append((cid, lo, end))
        lo = end
    return out


def max_rel_error(values: torch.Tensor, gold_hi: torch.Tensor, gold_lo: torch.Tensor) -> torch.Tensor:
    """max |v - (hi + lo)| / |hi| over representable references (device op)."""
    v = values.to(torch.float64)
    err = ((v - gold_hi) - gold_lo).abs()
    tiny = torch.finfo(values.dtype).tiny
    ok = gold_hi.abs() >= tiny
    rel = torch.where(ok, err / gold_hi.abs().clamp_min(tiny), torch.zeros_like(err))
    return rel.max() if rel.numel() else torch.zeros((), dtype=torch.float64, device=v.device)


def gather_max(local: torch.Tensor) -> tuple:
    """all_gather of one fp64 per rank -> (per-rank list, max).  Works with
    NCCL (device tensor) and gloo (CPU tensor)."""
    import torch.distributed as dist
    t = local.reshape(1).to(torch.float64)
    if not dist.is_available() or not dist.is_initialized():
        return [float(t.item())], float(t.item())
    world = dist.get_world_size()
    buf = torch.empty(world, dtype=torch.float64, device=t.device)
    dist.all_gather_into_tensor(buf, t)
    vals = buf.cpu().tolist()
    return vals, max(vals)


@dataclass
class SweepResult:
    points: int
    values: int
    per_rank_err: list = field(default_factory=list)
    max_err: float = 0.0
    checksum: float = 0.0


def golden_error(n: int, gold_x: torch.Tensor, gold_F: torch.Tensor, rank: int, world: int,
                 evaluate: Callable) -> torch.Tensor:
    """Rank's slice (rank::world) of the golden subsample -> max relative error
    over all orders.  gold_F: [M, n+1, 2] double-double references."""
    xs = gold_x[rank::world]
    g = gold_F[rank::world]
    if xs.numel() == 0:
        return torch.zeros((), dtype=torch.float64, device=gold_x.device)
    vals = evaluate(n, xs)                     # [M', n+1] (point-major)
    return max_rel_error(vals, g[..., 0], g[..., 1])


def run_sweep(n: int, N: int, rank: int, world: int, make_x: Callable, evaluate: Callable,
              gold: Optional[tuple] = None, chunk: int = CHUNK) -> SweepResult:
    """Evaluate the rank's contiguous shard chunk by chunk; optional golden
    error check gathered across ranks.  ``evaluate(n, x) -> [len(x), n+1]``
    (the GPU kernel in production; the tests inject the CPU oracle)."""
    pts = 0
    csum = 0.0
    for cid, lo, hi in chunk_plan(N, rank, world, chunk):
        x_full = make_x(cid)
        x = x_full[lo - cid * chunk: hi - cid * chunk]
        vals = evaluate(n, x)
        pts += x.numel()
        csum += float(vals[:, 0].double().sum())
    res = SweepResult(points=pts, values=pts * (n + 1), checksum=csum)
    if gold is not None:
        gx, gF = gold
        e = golden_error(n, gx, gF, rank, world, evaluate)
        res.per_rank_err, res.max_err = gather_max(e)
    return res
