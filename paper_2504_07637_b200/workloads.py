"""Seeded synthetic inputs for the five BASELINE.json configurations.

The configurations name no public dataset; these generators reproduce the
stated distributions (BASELINE.json "configs").  Every chunk
of at most 2^26 points is keyed by (seed, chunk) so any rank can regenerate
any chunk (contiguous sharding is then shard-invariant).  Within a chunk the
strata are drawn in their exact proportions and then permuted with the same
key, so warps see mixed strata (the realistic worst case for divergence).

Generation runs with torch on the requested device (fast on the GPU); the
values depend on the device's RNG, and tests always compare implementations
on the same generated x, never against stored x.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import torch

CHUNK = 1 << 26
Z16_53 = float.fromhex("0x1.2a06fd39e20e6p+6")   # z_{16,53} = 74.506825355932591


@dataclass(frozen=True)
class Config:
    name: str
    n_max: int            # -1 for ragged
    N: int
    layout: str           # 'soa' | 'aos' | 'ragged'
    dtype: torch.dtype
    desc: str


CONFIGS = {
    "cfg1": Config("cfg1", 0, 1 << 20, "soa", torch.float64,
                   "F_0 only (n_max=0), fp64, N=2^20: 25% 0, 25% U[0,1], 25% U[1,40], "
                   "25% logU[1e-10,1e4]; out F_0[N]"),
    "cfg2": Config("cfg2", 8, 1 << 24, "soa", torch.float64,
                   "n_max=8 fp64, N=2^24: 50% U[0,30], 50% logU[1e-8,1e4]; SoA [9][N]"),
    "cfg3": Config("cfg3", 16, 1 << 26, "aos", torch.float64,
                   "n_max=16 fp64, N=2^26: 90% logU[1e-12,1e5], 10% within +-1e-3 rel of "
                   "z_{16,53}; AoS [N][17]"),
    "cfg4": Config("cfg4", -1, 1 << 27, "ragged", torch.float64,
                   "ERI-like ragged batch, fp64, N=2^27 quartets, n_i in 0..12 with "
                   "P(n) ~ 1/(n+1), x = rho |P-Q|^2"),
    "cfg4f32": Config("cfg4f32", -1, 1 << 27, "ragged", torch.float32,
                      "cfg4 fp32 variant on the n_i <= 8 subset"),
    "cfg5": Config("cfg5", 12, 1 << 30, "aos", torch.float64,
                   "n_max=12 fp64, N=2^30 logU[1e-10,1e4], 2^26-point chunks sharded "
                   "contiguously over ranks; AoS [N][13]"),
}


def _gen(seed: int, chunk: int, device) -> torch.Generator:
    g = torch.Generator(device=device)
    g.manual_seed((seed * 1_000_003 + chunk) & 0x7FFF_FFFF_FFFF_FFFF)
    return g


def _u(g, n, lo, hi, device):
    return torch.rand(n, generator=g, device=device, dtype=torch.float64) * (hi - lo) + lo


def _logu(g, n, lo, hi, device):
    a, b = math.log(lo), math.log(hi)
    return torch.exp(_u(g, n, a, b, device))


def _strata(g, n, parts, device):
    """parts: list of (fraction, sampler(k) -> tensor); exact counts, then permute."""
    counts = [int(round(f * n)) for f, _ in parts]
    counts[-1] = n - sum(counts[:-1])
    xs = torch.cat([s(k) for (_, s), k in zip(parts, counts)])
    return xs[torch.randperm(n, generator=g, device=device)]


def cfg1_x(n=1 << 20, seed=1, chunk=0, device="cpu"):
    g = _gen(seed, chunk, device)
    return _strata(g, n, [
        (0.25, lambda k: torch.zeros(k, dtype=torch.float64, device=device)),
        (0.25, lambda k: _u(g, k, 0.0, 1.0, device)),
        (0.25, lambda k: _u(g, k, 1.0, 40.0, device)),
        (0.25, lambda k: _logu(g, k, 1e-10, 1e4, device)),
    ], device)


def cfg2_x(n=1 << 24, seed=2, chunk=0, device="cpu"):
    g = _gen(seed, chunk, device)
    return _strata(g, n, [
        (0.5, lambda k: _u(g, k, 0.0, 30.0, device)),
        (0.5, lambda k: _logu(g, k, 1e-8, 1e4, device)),
    ], device)


def cfg3_x(n=1 << 26, seed=3, chunk=0, device="cpu"):
    g = _gen(seed, chunk, device)
    return _strata(g, n, [
        (0.9, lambda k: _logu(g, k, 1e-12, 1e5, device)),
        (0.1, lambda k: Z16_53 * (1.0 + _u(g, k, -1e-3, 1e-3, device))),
    ], device)


def cfg5_x(n=CHUNK, seed=5, chunk=0, device="cpu"):
    g = _gen(seed, chunk, device)
    return _logu(g, n, 1e-10, 1e4, device)


def cfg4_batch(n=1 << 27, seed=4, chunk=0, device="cpu", sub=1 << 22):
    """ERI-like quartets -> (x float64 [n], n_max uint8 [n]).

    alpha..delta log-uniform [0.05, 1e4]; centres uniform in a 20-bohr cube;
    P = (aA + bB)/(a+b), Q = (cC + dD)/(c+d), rho = (a+b)(c+d)/(a+b+c+d),
    x = rho |P - Q|^2; n_i in 0..12 with P(n) proportional to 1/(n+1).
    Generated in sub-chunks to bound memory.
    """
    g = _gen(seed, chunk, device)
    w = torch.tensor([1.0 / (k + 1) for k in range(13)], dtype=torch.float64, device=device)
    xs, ns = [], []
    for s in range(0, n, sub):
        k = min(sub, n - s)
        e = _logu(g, 4 * k, 0.05, 1e4, device).view(4, k)
        c = _u(g, 12 * k, 0.0, 20.0, device).view(4, 3, k)
        a, b, cc, d = e[0], e[1], e[2], e[3]
        P = (a * c[0] + b * c[1]) / (a + b)
        Q = (cc * c[2] + d * c[3]) / (cc + d)
        rho = (a + b) * (cc + d) / (a + b + cc + d)
        xs.append(rho * ((P - Q) ** 2).sum(0))
        ns.append(torch.multinomial(w, k, replacement=True, generator=g).to(torch.uint8))
    return torch.cat(xs), torch.cat(ns)


def cfg4f32_batch(n=1 << 27, seed=4, chunk=0, device="cpu"):
    """fp32 variant: the n_i <= 8 subset of the cfg4 batch, x rounded to fp32."""
    x, nm = cfg4_batch(n, seed, chunk, device)
    keep = nm <= 8
    return x[keep].to(torch.float32), nm[keep]


def shell_pairs(n, seed=6, chunk=0, device="cpu"):
    """Primitive shell-pair records for the fused consumer (hermite_coulomb):
    [n, 5] float64 (p, Px, Py, Pz, K) from two primitives with exponents
    log-uniform [0.05, 50], centre A uniform in a 20-bohr cube and B within
    1.5 bohr of it per axis (pairs that survive Schwarz-type screening):
    p = a + b, P = (aA + bB)/p, K = exp(-ab/p |A-B|^2)."""
    g = _gen(seed, chunk, device)
    e = _logu(g, 2 * n, 0.05, 50.0, device).view(2, n)
    A = _u(g, 3 * n, 0.0, 20.0, device).view(3, n)
    B = A + _u(g, 3 * n, -1.5, 1.5, device).view(3, n)
    a, b = e[0], e[1]
    p = a + b
    P = (a * A + b * B) / p
    K = torch.exp(-(a * b / p) * ((A - B) ** 2).sum(0))
    return torch.stack([p, P[0], P[1], P[2], K], dim=1).contiguous()


def config_x(name: str, n: int = None, seed: int = None, chunk: int = 0, device="cpu"):
    """Dense-config inputs (cfg1/2/3/5) with the config's default size/seed."""
    fn = {"cfg1": cfg1_x, "cfg2": cfg2_x, "cfg3": cfg3_x, "cfg5": cfg5_x}[name]
    kw = {"chunk": chunk, "device": device}
    if n is not None:
        kw["n"] = n
    if seed is not None:
        kw["seed"] = seed
    return fn(**kw)
