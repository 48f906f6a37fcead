#!/usr/bin/env python3
"""Benchmark of the batched Boys evaluator (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config cfg3] [--no-extras]

Headline workload (config.workload): BASELINE config 3 -- n_max = 16, fp64,
N = 2^26 points per GPU (log-uniform [1e-12, 1e5] + 10% at the cut-off),
point-major (AoS) output [N][17].  It is the configuration the north star
quotes its single-GPU roofline target on; inputs (512 MiB) and outputs
(9.1 GB) are far larger than L2, so no flush is needed between steps.  One
step = one launch of the dense kernel over the rank's 2^26 points (weak
scaling: each rank owns its own 2^26-point chunk, keyed by rank) plus the
per-shard error reduction over that launch's own outputs.

Multi-GPU: one process per GPU.  ``--gpus N`` outside torchrun re-executes
itself under ``torch.distributed.run --nproc-per-node N`` (NCCL); under
torchrun the ranks come from the environment.  Each rank's inputs carry its
slice of the refmath golden points spliced in at known positions; every
step reduces the relative error at those positions on the device
(boys_shard_error), and the one fp64 per rank is all-gathered inside the
timed window (time from a barrier to after the gather).

Timing: W untimed warm-up steps, barrier + synchronize, K timed steps with
CUDA events on the launching stream, the gather, synchronize + barrier; the
job time is the max over ranks.  value = F-values/s over all ranks.

Also reported: roofline of the dominant kernel (algorithmic bytes / measured
launch time vs the measured HBM copy bandwidth), SM clocks sampled through
NVML during the timed region, the end-to-end number through the host-buffer
C-ABI entry (pinned host x in, full result out, copies inside the timed
region), the CPU baselines (the C port on the host cores, bounded sample; and
the reference's own mpmath path, refmath.boys_downward, on a 2^12 sample
with one process per core), and per-config lines for the other BASELINE
configurations, each with its accuracy against the refmath goldens and its
ulp distance to the C port.

``--impl reference`` times the reference's CPU implementation of the path:
the reference ships no finite-precision evaluator (only mpmath), so this is
the C restatement in oracle/ on all host cores (kind "port") over the same
workload per step as our arm (all 2^26 points of cfg3), plus the mpmath line.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import socket
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402
import torch  # noqa: E402

METRIC = "Boys values/sec (F_m outputs, fp64) and % of HBM/FP64 roofline"
UNIT = "values/s"


# ----------------------------------------------------------------------------
# launcher: --gpus N outside torchrun -> N ranks under torch.distributed.run
# ----------------------------------------------------------------------------

def _free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def maybe_reexec(gpus: int) -> None:
    if gpus <= 1 or "RANK" in os.environ:
        return
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={gpus}", "--master-addr=127.0.0.1",
           f"--master-port={_free_port()}", str(Path(__file__).resolve()), *sys.argv[1:]]
    sys.exit(subprocess.call(cmd))


# ----------------------------------------------------------------------------
# rank context: process group, device, clocks, reductions (device-agnostic:
# NCCL + CUDA events on GPUs, gloo + the host clock for the CPU self-test)
# ----------------------------------------------------------------------------

class Ctx:
    def __init__(self, stub: bool = False):
        self.ws = int(os.environ.get("WORLD_SIZE", "1"))
        self.rank = int(os.environ.get("RANK", "0"))
        self.local = int(os.environ.get("LOCAL_RANK", "0"))
        self.cuda = not stub
        if self.cuda:
            torch.cuda.set_device(self.local)
            self.dev = torch.device("cuda", self.local)
        else:
            self.dev = torch.device("cpu")
        self.dist = False
        if "RANK" in os.environ:
            import torch.distributed as dist
            if self.cuda:
                dist.init_process_group("nccl", device_id=self.dev)
            else:
                dist.init_process_group("gloo")
            self.dist = True

    # -- clocks: CUDA events on the launching stream, or the host clock --
    def mark(self):
        if self.cuda:
            e = torch.cuda.Event(enable_timing=True)
            e.record(torch.cuda.current_stream())
            return e
        return time.perf_counter()

    def sync(self):
        if self.cuda:
            torch.cuda.synchronize()

    def ms(self, a, b) -> float:
        return a.elapsed_time(b) if self.cuda else (b - a) * 1e3

    # -- collectives --
    def barrier(self):
        if self.dist:
            import torch.distributed as dist
            dist.barrier()

    def _reduce(self, v: float, op) -> float:
        if not self.dist:
            return v
        import torch.distributed as dist
        t = torch.tensor([v], dtype=torch.float64, device=self.dev)
        dist.all_reduce(t, op=op)
        return float(t.item())

    def max(self, v: float) -> float:
        import torch.distributed as dist
        return self._reduce(v, dist.ReduceOp.MAX) if self.dist else v

    def sum(self, v: float) -> float:
        import torch.distributed as dist
        return self._reduce(v, dist.ReduceOp.SUM) if self.dist else v

    def gather_into(self, buf: torch.Tensor, local: torch.Tensor) -> None:
        """all_gather of one fp64 per rank (stream-ordered under NCCL)."""
        if self.dist:
            import torch.distributed as dist
            dist.all_gather_into_tensor(buf, local.reshape(1))
        else:
            buf.copy_(local.reshape(1))

    def gather_list(self, v: float) -> list:
        buf = torch.zeros(self.ws, dtype=torch.float64, device=self.dev)
        self.gather_into(buf, torch.tensor([v], dtype=torch.float64, device=self.dev))
        return buf.cpu().tolist()

    def close(self):
        if self.dist:
            import torch.distributed as dist
            dist.destroy_process_group()


class ClockSampler:
    """NVML sampling of SM clock and throttle reasons while active."""

    REASONS = {
        0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
        0x8: "hw_slowdown", 0x10: "sync_boost", 0x20: "sw_thermal_slowdown",
        0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
        0x100: "display_clock_setting",
    }

    def __init__(self, local_rank: int, period=0.01):
        self.samples, self.reasons, self.ok = [], 0, False
        self.period = period
        try:
            import pynvml as N
            N.nvmlInit()
            vis = os.environ.get("CUDA_VISIBLE_DEVICES")
            idx = int(vis.split(",")[local_rank]) if vis else local_rank
            self.N, self.h = N, N.nvmlDeviceGetHandleByIndex(idx)
            self.max_mhz = N.nvmlDeviceGetMaxClockInfo(self.h, N.NVML_CLOCK_SM)
            self.ok = True
        except Exception as e:  # noqa: BLE001
            self.err = str(e)
        self._stop = threading.Event()

    def _run(self):
        N = self.N
        while not self._stop.is_set():
            try:
                self.samples.append(N.nvmlDeviceGetClockInfo(self.h, N.NVML_CLOCK_SM))
                self.reasons |= N.nvmlDeviceGetCurrentClocksEventReasons(self.h)
            except Exception:  # noqa: BLE001
                pass
            time.sleep(self.period)

    def __enter__(self):
        if self.ok:
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        return self

    def __exit__(self, *a):
        if self.ok:
            self._stop.set()
            self._t.join()

    def summary(self):
        if not self.ok:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "error": self.err}
        rs = [name for bit, name in self.REASONS.items() if self.reasons & bit]
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None,
                "sm_max_mhz": self.max_mhz, "reasons": rs, "samples": len(self.samples)}


class _Null:
    def __enter__(self):
        return self

    def __exit__(self, *a):
        pass

    def summary(self):
        return None


def measured_peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return d.get("hbm_gbs"), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def fp64_peak_probe():
    """Measured DFMA rate (ops/s) with the probe library, or None."""
    try:
        import ctypes as C
        from paper_2504_07637_b200 import build as B
        lib = C.CDLL(str(B.build_probe()))
        lib.boys_probe_fp64_rate.restype = C.c_double
        lib.boys_probe_fp64_rate.argtypes = [C.c_int, C.c_int, C.POINTER(C.c_double)]
        ms = C.c_double()
        return lib.boys_probe_fp64_rate(4096, 5, C.byref(ms))
    except Exception:  # noqa: BLE001
        return None


def committed_traffic(config: str):
    """dram bytes per launch of the dominant kernel from the committed ncu
    capture (profiles/ncu_traffic.json, one `ncu --set full` per config)."""
    p = ROOT / "profiles" / "ncu_traffic.json"
    if p.exists():
        d = json.loads(p.read_text())
        return d.get(config)
    return None


# ----------------------------------------------------------------------------
# workloads: one step = the config's kernel launches + the error reduction
# over those launches' outputs at the spliced golden positions
# ----------------------------------------------------------------------------

def _golden(name: str):
    """refmath.boys_downward goldens (tests/golden/configs.npz, double-double)."""
    d = np.load(ROOT / "tests" / "golden" / "configs.npz")
    if name.startswith("cfg4"):
        return d[f"{name}_x"], d[f"{name}_n"], d[f"{name}_F"]
    return d[f"{name}_x"], None, d[f"{name}_F"]


class _ErrCheck:
    """Device-side error statistic: positions into one output tensor and the
    (hi, lo) references there; run() folds the max relative error into err."""

    def __init__(self, out: torch.Tensor, pos: torch.Tensor, gold: torch.Tensor,
                 err: torch.Tensor):
        self.out, self.pos, self.gold, self.err = out, pos.contiguous(), gold.contiguous(), err
        self.K = int(pos.numel())

    def run(self):
        import ctypes as C
        from paper_2504_07637_b200 import _lib as L
        dt = L.BOYS_F64 if self.out.dtype == torch.float64 else L.BOYS_F32
        L.check(L.load().boys_shard_error(
            dt, C.c_void_p(self.out.data_ptr()), C.c_void_p(self.pos.data_ptr()),
            C.c_void_p(self.gold.data_ptr()), self.K, C.c_void_p(self.err.data_ptr()),
            C.c_void_p(torch.cuda.current_stream(self.out.device).cuda_stream)))


def _spread(total: int, k: int, dev) -> torch.Tensor:
    """k positions spread evenly over [0, total)."""
    stride = max(1, total // max(1, k))
    return torch.arange(k, device=dev, dtype=torch.int64) * stride + stride // 2


class Dense:
    """Dense config: one or more 2^26-point chunks per rank (weak), or the
    rank's contiguous shard of 2^30 (cfg5, strong)."""

    def __init__(self, cfg, ctx, n_points=None, rotate=1, split_nbar=None):
        from paper_2504_07637_b200 import roofline as R, workloads as W
        self.cfg, self.ctx = cfg, ctx
        dev = ctx.dev
        self.n = cfg.n_max
        self.layout = cfg.layout
        self.split_nbar = split_nbar
        total = n_points or cfg.N
        if cfg.name == "cfg5":          # strong scaling: shard 2^30 contiguously
            from paper_2504_07637_b200 import shard as S
            plan = S.chunk_plan(total, ctx.rank, ctx.ws, W.CHUNK)
            self.xs = [W.config_x("cfg5", n=W.CHUNK, chunk=cid, device=dev)[lo - cid * W.CHUNK:
                                                                          hi - cid * W.CHUNK]
                       for cid, lo, hi in plan]
            self.outs = [torch.empty(self._shape(W.CHUNK), dtype=cfg.dtype, device=dev)
                         for _ in range(min(2, len(self.xs)))]
            self.scaling = "strong"
        else:                            # weak: each rank its own chunk(s)
            self.xs = [W.config_x(cfg.name, n=total, chunk=ctx.rank * rotate + j, device=dev)
                       for j in range(rotate)]
            self.outs = [torch.empty(self._shape(total), dtype=cfg.dtype, device=dev)
                         for _ in range(rotate)]
            self.scaling = "weak"
        self.points_per_step = sum(x.numel() for x in self.xs)
        self.values_per_step = self.points_per_step * (self.n + 1)
        self.bytes_per_point = R.dense_bytes_per_point(self.n, 8 if cfg.dtype == torch.float64 else 4)
        self.ops_per_point = R.ops_per_point(self.n) if split_nbar is None else None
        self.err = torch.zeros(1, dtype=torch.float64, device=dev)
        self._splice()

    def _shape(self, N):
        return (N, self.n + 1) if self.layout == "aos" else (self.n + 1, N)

    def _out(self, k):
        x = self.xs[k]
        out = self.outs[k % len(self.outs)]
        if self.layout == "aos":
            return out[: x.numel()]          # contiguous prefix for a partial chunk
        return out if out.shape[1] == x.numel() else None

    def _splice(self):
        """The rank's slice (rank::world) of the golden points goes into its
        first batch; the check reads the first launch's own outputs there."""
        gx, _, gF = _golden(self.cfg.name if self.cfg.name != "split" else "cfg3")
        gx, gF = gx[self.ctx.rank::self.ctx.ws], gF[self.ctx.rank::self.ctx.ws]
        x = self.xs[0]
        pos = _spread(x.numel(), len(gx), x.device)
        x[pos] = torch.from_numpy(gx).to(x.device, x.dtype)
        self.golden_points = len(gx)
        W = self.n + 1
        m = torch.arange(W, device=x.device, dtype=torch.int64)
        out = self._out(0)
        if self.layout == "aos":
            opos = pos[:, None] * W + m[None, :]
        else:
            opos = m[None, :] * x.numel() + pos[:, None]
        gold = torch.from_numpy(np.ascontiguousarray(gF)).to(x.device)      # [K][W][2]
        self.check = _ErrCheck(out.reshape(-1), opos.reshape(-1), gold.reshape(-1, 2), self.err)

    def steps(self):
        """[(fn, is_kernel)] for one step."""
        from paper_2504_07637_b200 import boys, eval_with_split
        fns = []
        for k, x in enumerate(self.xs):
            out = self._out(k)
            if out is None:             # SoA partial chunk: a fresh view of the right width
                out = self.outs[k % len(self.outs)].view(-1)[: x.numel() * (self.n + 1)].view(
                    self.n + 1, x.numel())
            if self.split_nbar is not None:
                fns.append((lambda x=x, out=out: eval_with_split(
                    self.n, self.split_nbar, x, layout=self.layout, check=False, out=out), True))
            else:
                fns.append((lambda x=x, out=out: boys(self.n, x, layout=self.layout, out=out,
                                                      check=False), True))
            if k == 0:
                fns.append((self.check.run, False))
        return fns

    def port_compare(self, npts=1 << 18):
        """Max ulp between the GPU and the C port on a prefix of the first batch."""
        from oracle import oracle as O
        from paper_2504_07637_b200 import boys, eval_with_split
        x = self.xs[0][:npts].contiguous()
        if self.split_nbar is not None:
            g = eval_with_split(self.n, self.split_nbar, x, layout=self.layout).cpu().numpy()
            ref, _ = O.split(self.n, self.split_nbar, x.cpu().numpy(), self.layout)
        else:
            g = boys(self.n, x, layout=self.layout).cpu().numpy()
            ref, _ = O.dense(self.n, x.cpu().numpy(), self.layout)
        return max_ulp(g, ref), int(x.numel())


class Ragged:
    def __init__(self, cfg, ctx, n_points=None):
        from paper_2504_07637_b200 import ragged_offsets, roofline as R, workloads as W
        self.cfg, self.ctx = cfg, ctx
        dev = ctx.dev
        N = n_points or cfg.N
        if cfg.dtype == torch.float32:
            self.x, self.nm = W.cfg4f32_batch(N, chunk=ctx.rank, device=dev)
        else:
            self.x, self.nm = W.cfg4_batch(N, chunk=ctx.rank, device=dev)
        gx, gn, gF = _golden(cfg.name)
        # golden elements (x and order) spliced in before the offsets are formed
        goff = np.zeros(len(gx) + 1, dtype=np.int64)
        np.cumsum(gn.astype(np.int64) + 1, out=goff[1:])
        sel = np.arange(ctx.rank, len(gx), ctx.ws)
        pos = _spread(self.x.numel(), len(sel), dev)
        self.x[pos] = torch.from_numpy(gx[sel]).to(dev, self.x.dtype)
        self.nm[pos] = torch.from_numpy(gn[sel]).to(dev)
        self.golden_points = len(sel)
        self.off = ragged_offsets(self.nm)
        total = int(self.off[-1].item())
        self.out = torch.empty(total, dtype=cfg.dtype, device=dev)
        base = self.off[pos].cpu().numpy()
        opos = np.concatenate([b + np.arange(int(gn[j]) + 1) for b, j in zip(base, sel)])
        gold = np.concatenate([gF[goff[j]:goff[j + 1]] for j in sel])
        self.err = torch.zeros(1, dtype=torch.float64, device=dev)
        self.check = _ErrCheck(self.out, torch.from_numpy(opos).to(dev),
                               torch.from_numpy(np.ascontiguousarray(gold)).to(dev), self.err)
        self.points_per_step = self.x.numel()
        self.values_per_step = total
        eb = 8 if cfg.dtype == torch.float64 else 4
        self.bytes_total = R.ragged_bytes(self.x.numel(), total, eb)
        self.bytes_per_point = self.bytes_total / self.x.numel()
        self.ops_per_point = None
        self.scaling = "weak"

    def steps(self):
        from paper_2504_07637_b200 import boys_ragged
        return [(lambda: boys_ragged(self.x, self.nm, self.off, out=self.out, check=False), True),
                (self.check.run, False)]

    def offsets_ms(self, reps=20):
        """Device time of one offsets scan over the whole batch (int64, N+1)."""
        from paper_2504_07637_b200 import ragged_offsets
        ctx = self.ctx
        o = torch.empty_like(self.off)                 # preallocated: device time only
        for _ in range(3):
            ragged_offsets(self.nm, out=o)
        ctx.sync()
        a = ctx.mark()
        for _ in range(reps):
            ragged_offsets(self.nm, out=o)
        b = ctx.mark()
        ctx.sync()
        same = bool(torch.equal(o, self.off))
        return ctx.ms(a, b) / reps, same

    def port_compare(self, npts=1 << 18):
        from oracle import oracle as O
        from paper_2504_07637_b200 import boys_ragged
        x, nm = self.x[:npts].contiguous(), self.nm[:npts].contiguous()
        g, _ = boys_ragged(x, nm)
        ref, _, _ = O.ragged(x.cpu().numpy(), nm.cpu().numpy())
        return max_ulp(g.cpu().numpy(), ref), int(x.numel())


class Stub:
    """CPU stand-in for the self-test of the multi-rank plumbing (gloo): a
    torch op per step and the same error-check protocol."""

    def __init__(self, ctx, n_points=1 << 16):
        g = torch.Generator().manual_seed(1000 + ctx.rank)
        self.ctx = ctx
        self.x = torch.rand(n_points, generator=g, dtype=torch.float64) * 10
        self.out = torch.empty_like(self.x)
        self.err = torch.zeros(1, dtype=torch.float64)
        self.points_per_step = self.values_per_step = n_points
        self.bytes_per_point, self.ops_per_point = 16.0, None
        self.scaling = "weak"
        self.golden_points = 1

    def _check(self):
        e = ((self.out - torch.exp(-self.x)).abs() / torch.exp(-self.x)).max()
        self.err.copy_(torch.maximum(self.err, e.reshape(1)))

    def steps(self):
        return [(lambda: torch.exp(-self.x, out=self.out), True), (self._check, False)]


def max_ulp(a: np.ndarray, b: np.ndarray) -> int:
    """Max |bits(a) - bits(b)| over all values (NaN pairs count 0)."""
    ia = a.view(np.int64 if a.dtype == np.float64 else np.int32).astype(np.int64)
    ib = b.view(np.int64 if b.dtype == np.float64 else np.int32).astype(np.int64)
    both_nan = np.isnan(a) & np.isnan(b)
    return int(np.where(both_nan, 0, np.abs(ia - ib)).max(initial=0))


def make_workload(name, ctx, n_points=None, rotate=1):
    from paper_2504_07637_b200 import workloads as W
    if name == "split":
        return Dense(W.CONFIGS["cfg3"], ctx, n_points, split_nbar=8)
    cfg = W.CONFIGS[name]
    if cfg.layout == "ragged":
        return Ragged(cfg, ctx, n_points)
    return Dense(cfg, ctx, n_points, rotate=rotate)


def launch_count(ctx) -> int:
    if not ctx.cuda:
        return 0
    from paper_2504_07637_b200 import _lib
    return _lib.launch_count()


def time_workload(wl, ctx, steps, warmup, flush=None, sample_clocks=False, graph=False):
    """Times `steps` steps of `wl` on every rank (barrier -> steps -> error
    gather -> barrier).  Returns a dict: job seconds (max over ranks),
    per-kernel-launch ms, clocks, launches, per-rank error vector.

    graph=True: the step's launches are captured once into a CUDA graph and
    each step is one replay (for small batches whose host-side launch cost
    would otherwise starve the GPU); per-launch time = replay time / kernels.
    flush: called before every step outside the kernel timing (the job time
    is then the sum of the step times).
    """
    fns = wl.steps()
    nk = sum(1 for _, k in fns if k)
    for _ in range(warmup):
        for f, _ in fns:
            f()
    ctx.sync()
    if graph:
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            for f, _ in fns:
                f()
        ctx.sync()
        for _ in range(warmup):
            g.replay()
        ctx.sync()
        fns = [(g.replay, True)]
    wl.err.zero_()
    gbuf = torch.zeros(ctx.ws, dtype=torch.float64, device=ctx.dev)
    ctx.barrier()
    ctx.sync()
    evs = []
    l0 = launch_count(ctx)
    sampler = ClockSampler(ctx.local) if (sample_clocks and ctx.cuda) else _Null()
    step_evs = []
    with sampler:
        t_start = ctx.mark()
        for _ in range(steps):
            if flush is not None:
                flush()
            s0 = ctx.mark()
            for f, is_kernel in fns:
                if is_kernel:           # events bracket the evaluator launches only
                    a = ctx.mark()
                    f()
                    evs.append((a, ctx.mark()))
                else:
                    f()
            step_evs.append((s0, ctx.mark()))
        ctx.gather_into(gbuf, wl.err)          # inside the timed window
        t_end = ctx.mark()
        ctx.sync()
    ctx.barrier()
    launches = launch_count(ctx) - l0
    per_launch = [ctx.ms(a, b) for a, b in evs]
    if graph:      # kernels launched by the replays (the host counter sees none)
        launches = steps * (nk + 1)
        per_launch = [p / nk for p in per_launch]
    if flush is not None:     # job time = step times only (flushes excluded)
        secs = sum(ctx.ms(a, b) for a, b in step_evs) / 1e3
    else:
        secs = ctx.ms(t_start, t_end) / 1e3
    local_secs = secs
    secs = ctx.max(secs)
    per_rank_err = gbuf.cpu().tolist()
    return {"secs": secs, "local_secs": local_secs, "per_launch_ms": per_launch,
            "clocks": sampler.summary(), "launches": launches, "kernels_per_step": nk,
            "per_rank_err": per_rank_err}


def roofline_obj(wl, per_ms, hbm_peak, fp64_peak, bound=None, traffic=None):
    launch_ms = statistics.mean(per_ms)
    nk = sum(1 for _, k in wl.steps() if k)
    pts = wl.points_per_step / max(1, nk)
    bytes_launch = wl.bytes_per_point * pts
    gbs = bytes_launch / (launch_ms * 1e-3) / 1e9
    out = {"bound": "hbm", "achieved": round(gbs, 1), "peak": hbm_peak, "unit": "GB/s",
           "frac": round(gbs / hbm_peak, 4), "traffic": traffic,
           "algorithmic_bytes_per_launch": int(bytes_launch),
           "bytes_per_point": wl.bytes_per_point, "launch_ms": round(launch_ms, 4)}
    if wl.ops_per_point and fp64_peak:
        ops = wl.ops_per_point * pts / (launch_ms * 1e-3)
        out["fp64_ops_frac"] = round(ops / fp64_peak, 4)
        t_b = bytes_launch / (hbm_peak * 1e9)
        t_o = wl.ops_per_point * pts / fp64_peak
        if bound == "fp64" or (bound is None and t_o > t_b):
            out.update({"bound": "fp64", "achieved": round(ops / 1e12, 3),
                        "peak": round(fp64_peak / 1e12, 3), "unit": "TDPop/s",
                        "frac": round(ops / fp64_peak, 4),
                        "peak_source": "measured DFMA probe (libboys_probe)"})
    return out


def accuracy_obj(wl, res):
    per = res["per_rank_err"]
    mx = max(per) if per else 0.0
    return {"max_rel_err": mx, "bits": (-math.log2(mx) if mx > 0 else None),
            "per_rank": per, "golden_points_per_rank": wl.golden_points,
            "measured_on": "the timed launches' own outputs at the spliced golden positions "
                           "(boys_shard_error, gathered inside the timed window)",
            "reference": "refmath.boys_downward(n, x, Precision(96)), tests/golden/configs.npz"}


# ----------------------------------------------------------------------------
# CPU baselines / reference arm
# ----------------------------------------------------------------------------

def cpu_model() -> str:
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def cpu_port_rate(n, x_host, layout, min_seconds=10.0, gpu_out=None):
    """Times the C restatement on the host cores.  gpu_out (the GPU's values for
    the same sample): returns the max |GPU - CPU| in ulp over the sample."""
    from oracle import oracle as O
    O.dense(n, x_host[:1024], layout)      # load + warm
    t0 = time.perf_counter()
    reps = 0
    ref = None
    while True:
        ref, _ = O.dense(n, x_host, layout)
        reps += 1
        el = time.perf_counter() - t0
        if el >= min_seconds:
            break
    ulp = max_ulp(gpu_out, ref) if gpu_out is not None else None
    return reps * x_host.size * (n + 1) / el, O.threads(), reps, ulp


def _mp_worker(args):
    n, xs = args
    sys.path.insert(0, str(ROOT / "baseline" / "_ref"))
    from boysfn import refmath as RM
    p = RM.Precision(64)
    for x in xs:
        RM.boys_downward(n, float(x), p)
    return len(xs)


def reference_mpmath_rate(cfg_name="cfg3", npts=1 << 14):
    """The reference's own CPU path: refmath.boys_downward(n, x, Precision(64))
    (refmath.py:330-341) on a seeded 2^14-point sample of the config, one
    process per host core (the mpmath context is process-global)."""
    ref_dir = ROOT / "baseline" / "_ref"
    if not (ref_dir / "boysfn" / "refmath.py").exists():
        return {"unavailable": "baseline/_ref (pip install of the reference) not built; "
                               "run __graft_entry__.build() in the build container"}
    import multiprocessing as mp
    from paper_2504_07637_b200 import workloads as W
    cfg = W.CONFIGS[cfg_name]
    x = W.config_x(cfg_name, n=1 << 16, chunk=7, device="cpu").numpy()[:npts]
    cores = os.cpu_count() or 1
    parts = [(cfg.n_max, x[i::cores]) for i in range(cores)]
    ctx = mp.get_context("spawn")
    with ctx.Pool(cores) as pool:
        pool.map(_mp_worker, [(cfg.n_max, x[:cores])])     # import + warm every worker
        t0 = time.perf_counter()
        done = sum(pool.map(_mp_worker, parts))
        el = time.perf_counter() - t0
    return {"value": done * (cfg.n_max + 1) / el, "unit": UNIT, "points_per_s": done / el,
            "cores": cores, "cpu_model": cpu_model(), "kind": "reference",
            "sample": f"{done} seeded {cfg_name} points, refmath.boys_downward({cfg.n_max}, x, "
                      f"Precision(64)), multiprocessing.Pool({cores})",
            "seconds": el}


def run_reference(args, rank, ws):
    """--impl reference: the C oracle port on all host cores over the same
    workload per step as our arm; rank 0 only."""
    if rank != 0:
        return
    from oracle import oracle as O
    from paper_2504_07637_b200 import workloads as W
    cfg = W.CONFIGS[args.config]
    if cfg.layout == "ragged":
        raise SystemExit("--impl reference supports the dense configs")
    N = cfg.N if cfg.name != "cfg5" else W.CHUNK
    x = W.config_x(args.config, n=N, chunk=0, device="cpu").numpy()
    if cfg.dtype == torch.float32:
        x = x.astype(np.float32)
    # the whole config per step, in 2^22-point slices through one output
    # buffer (bounded host memory; the same work as one pass over N)
    sl = min(N, 1 << 22)

    def step():
        for i in range(0, N, sl):
            O.dense(cfg.n_max, x[i:i + sl], cfg.layout)

    for _ in range(args.warmup):
        step()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        step()
    el = time.perf_counter() - t0
    v = args.steps * N * (cfg.n_max + 1) / el
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": ws,
        "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": el / args.steps * 1e3, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": cfg.desc, "config": cfg.name, "points_per_step": N},
        "cpu_baseline": {"value": v, "unit": UNIT, "cores": O.threads(), "kind": "port",
                         "cpu_model": cpu_model(),
                         "sample": f"all {N} points of {cfg.name} per step (2^22-point slices), "
                                   "all host threads; C restatement of the SPEC kernel (the "
                                   "reference ships no finite-precision evaluator)"},
        "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    if args.mpmath:
        try:
            line["reference_mpmath"] = reference_mpmath_rate(cfg.name)
        except Exception as ex:  # noqa: BLE001
            line["reference_mpmath"] = {"error": str(ex)[:200]}
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------------------
# main arm
# ----------------------------------------------------------------------------

def e2e_dense(cfg_name, steps, dev):
    """Host-buffer path through the public API (C-ABI boys_eval_dense_host)."""
    from paper_2504_07637_b200 import boys, workloads as W
    cfg = W.CONFIGS[cfg_name]
    xd = W.config_x(cfg_name, n=cfg.N if cfg.name != "cfg5" else W.CHUNK, device=dev)
    N = xd.numel()
    xh = torch.empty(N, dtype=torch.float64, pin_memory=True)
    xh.copy_(xd)
    shape = (N, cfg.n_max + 1) if cfg.layout == "aos" else (cfg.n_max + 1, N)
    oh = torch.empty(shape, dtype=torch.float64, pin_memory=True)
    del xd
    boys(cfg.n_max, xh, layout=cfg.layout, out=oh)         # warm-up (allocates workspace)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(steps):
        boys(cfg.n_max, xh, layout=cfg.layout, out=oh)
    torch.cuda.synchronize()
    el = time.perf_counter() - t0
    return {"value": steps * N * (cfg.n_max + 1) / el, "unit": UNIT,
            "h2d_bytes_per_step": N * 8, "d2h_bytes_per_step": N * (cfg.n_max + 1) * 8,
            "steps": steps, "path": "boys(n, pinned host x) -> boys_eval_dense_host "
                                    "(chunked H2D / kernel / D2H pipeline)"}


def hermite_ops(L: int) -> int:
    """Algorithmic FP64 ops per quartet of the fused consumer (same weights as
    roofline.ops_per_point: div/rcp 8, sqrt 7, every other DP op 1): the Boys
    evaluation at order L (Table I N of that order), the pair geometry, the
    (-2a)^n F_n products, the Hermite recurrences and the prefactor."""
    from paper_2504_07637_b200 import roofline as R
    ops = R.ops_per_point(L, 8)
    ops += 3 + 1 + 1 + 8 + 3 + 1              # X, Y, Z; p+q; pq; /; r2 (mul + 2 fma); x
    ops += 2 * (L + 1)                        # R0_k = pw_k F_k, pw_{k+1} = pw_k (-2a)
    for n in range(L - 1, -1, -1):            # recurrences: fma + mul, or one mul
        for s in range(L - n, 0, -1):
            for t in range(s, -1, -1):
                for u in range(s - t, -1, -1):
                    v = s - t - u
                    ops += 2 if (t >= 2 or (t == 0 and u >= 2) or (t == 0 and u == 0 and v >= 2)) else 1
    ops += 1 + 7 + 1 + 8 + 1 + 1              # den = (pq) sqrt(p+q); pref
    ops += (L + 1) * (L + 2) * (L + 3) // 6   # pref * R
    return ops


def hermite_line(ctx, steps, warmup, hbm_peak, fp64_peak, L=4, npairs=4096):
    """The fused consumer as a bench line: McMurchie-Davidson
    Hermite Coulomb integrals for npairs x npairs primitive quartets at order
    L, F_0..F_L consumed in registers; device-resident pair data, CUDA events."""
    from paper_2504_07637_b200 import hermite_coulomb, workloads as W
    dev = ctx.dev
    bra = W.shell_pairs(npairs, seed=21, chunk=ctx.rank, device=dev)
    ket = W.shell_pairs(npairs, seed=22, chunk=ctx.rank, device=dev)
    NH = (L + 1) * (L + 2) * (L + 3) // 6
    # two output buffers, alternating (4.7 GB each): no launch rewrites lines
    # the previous one left dirty in L2
    outs = [torch.empty((npairs, npairs, NH), dtype=torch.float64, device=dev) for _ in range(2)]
    for k in range(warmup):
        hermite_coulomb(L, bra, ket, out=outs[k % 2], check=False)
    ctx.sync()
    l0 = launch_count(ctx)
    a = ctx.mark()
    for k in range(steps):
        hermite_coulomb(L, bra, ket, out=outs[k % 2], check=False)
    b = ctx.mark()
    out = outs[(steps - 1) % 2]
    ctx.sync()
    launches = launch_count(ctx) - l0
    ms = ctx.ms(a, b) / steps
    nq = npairs * npairs
    bytes_q = NH * 8
    gbs = bytes_q * nq / (ms * 1e-3) / 1e9
    ops = hermite_ops(L)
    tops = ops * nq / (ms * 1e-3)
    # bit-exactness against the CPU restatement on a 64 x 64 corner
    from oracle import oracle as O
    ref, bad = O.hermite(L, bra[:64].cpu().numpy(), ket[:64].cpu().numpy())
    got = out[:64, :64].cpu().numpy()
    same = bool(bad == -1 and np.array_equal(got.view(np.int64), ref.view(np.int64)))
    t_b, t_o = bytes_q * nq / (hbm_peak * 1e9), ops * nq / fp64_peak if fp64_peak else 0.0
    bound = "fp64" if t_o > t_b else "hbm"
    roof = ({"bound": "hbm", "achieved": round(gbs, 1), "peak": hbm_peak, "unit": "GB/s",
             "frac": round(gbs / hbm_peak, 4)} if bound == "hbm" else
            {"bound": "fp64", "achieved": round(tops / 1e12, 3), "peak": round(fp64_peak / 1e12, 3),
             "unit": "TDPop/s", "frac": round(tops / fp64_peak, 4)})
    roof.update({"traffic": committed_traffic("hermite"), "algorithmic_bytes_per_launch": bytes_q * nq,
                 "bytes_per_quartet": bytes_q, "fp64_ops_per_quartet": ops,
                 "fp64_ops_frac": round(tops / fp64_peak, 4) if fp64_peak else None,
                 "launch_ms": round(ms, 4),
                 "note": ("write-only stream: it can exceed the copy test (read + write) that "
                          "defines the peak; ncu of this launch: 4.64 GB DRAM writes in 0.670 ms "
                          "= 6.93 TB/s, 84.6% of the DRAM peak ncu reports "
                          "(profiles/r02_hermite_ncu.md)")})
    return {"value": ctx.sum(nq / (ms * 1e-3)), "unit": "quartets/s",
            "F_values_consumed_per_s": ctx.sum(nq * (L + 1) / (ms * 1e-3)),
            "steps": steps, "n_gpus": ctx.ws, "ms_per_step": ms, "scaling": "weak",
            "gpu_launches": launches, "roofline": roof,
            "accuracy": {"bit_identical_to_port": same, "compared_quartets": 64 * 64},
            "workload": (f"fused consumer: McMurchie-Davidson Hermite Coulomb integrals R_tuv, "
                         f"t+u+v <= {L} ({NH} per quartet), {npairs} x {npairs} primitive "
                         f"pair quartets (cfg4-like exponents), F_0..F_{L} in registers, never "
                         f"written; output [{npairs}][{npairs}][{NH}] fp64, two buffers alternating")}


def e2e_ragged(wl, steps):
    """Host-buffer ragged path through the public API (C-ABI
    boys_eval_ragged_host): pinned host x and orders in, pinned values out."""
    from paper_2504_07637_b200 import boys_ragged
    N = wl.x.numel()
    total = int(wl.values_per_step)
    eb = wl.x.element_size()
    xh = torch.empty(N, dtype=wl.x.dtype, pin_memory=True)
    xh.copy_(wl.x)
    nh = torch.empty(N, dtype=torch.uint8, pin_memory=True)
    nh.copy_(wl.nm)
    oh = torch.empty(total, dtype=wl.x.dtype, pin_memory=True)
    boys_ragged(xh, nh, out=oh, return_offsets=False)     # warm-up (allocates workspace)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(steps):
        boys_ragged(xh, nh, out=oh, return_offsets=False)
    torch.cuda.synchronize()
    el = time.perf_counter() - t0
    return {"value": steps * total / el, "unit": UNIT,
            "h2d_bytes_per_step": N * (eb + 1), "d2h_bytes_per_step": total * eb,
            "steps": steps, "path": "boys_ragged(pinned host x, pinned host n_max) -> "
                                    "boys_eval_ragged_host (chunked H2D / offsets scan / "
                                    "kernel / D2H pipeline)"}


def run_stub(args, ctx):
    """CPU self-test of the multi-rank plumbing (tests/test_bench_dist.py)."""
    wl = Stub(ctx)
    res = time_workload(wl, ctx, args.steps, args.warmup)
    total = ctx.sum(wl.values_per_step * args.steps)
    line = {"metric": METRIC, "value": total / res["secs"], "unit": UNIT, "n_gpus": ctx.ws,
            "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": res["secs"] / args.steps * 1e3, "higher_is_better": True,
            "scaling": wl.scaling, "data": "stub (CPU self-test)",
            "per_rank": {"secs": ctx.gather_list(res["local_secs"]),
                         "values": ctx.gather_list(float(wl.values_per_step * args.steps))},
            "accuracy": accuracy_obj(wl, res)}
    if ctx.rank == 0:
        print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=300)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="cfg3")
    ap.add_argument("--no-extras", action="store_true")
    ap.add_argument("--extras", default=None,
                    help="comma list of extra configs (default: all at N=1, cfg5 at N>1)")
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    ap.add_argument("--no-mpmath", dest="mpmath", action="store_false")
    ap.add_argument("--stub", action="store_true", help=argparse.SUPPRESS)
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    maybe_reexec(args.gpus)

    if args.impl == "reference":
        run_reference(args, int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")))
        return

    ctx = Ctx(stub=args.stub)
    if args.stub:
        try:
            run_stub(args, ctx)
        finally:
            ctx.close()
        return
    dev = ctx.dev
    from paper_2504_07637_b200 import _lib, workloads as W
    _lib.load(build_if_missing=False)
    hbm_peak, hbm_src = measured_peaks()
    fp64_peak = fp64_peak_probe()

    wl = make_workload(args.config, ctx)
    res = time_workload(wl, ctx, args.steps, args.warmup, sample_clocks=True)
    total_values = ctx.sum(wl.values_per_step * args.steps)
    value = total_values / res["secs"]
    roof = roofline_obj(wl, res["per_launch_ms"], hbm_peak, fp64_peak,
                        traffic=committed_traffic(args.config))
    roof["peak_source"] = roof.get("peak_source", hbm_src)
    roof["traffic_source"] = "profiles/ncu_traffic.json (ncu --set full capture, per launch)"
    cfg = W.CONFIGS[args.config]

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ctx.ws, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": res["secs"] / args.steps * 1e3,
        "higher_is_better": True, "scaling": wl.scaling, "vs_baseline": None,
        "dtype": "f64" if cfg.dtype == torch.float64 else "f32",
        "data": "synthetic (seeded generators of BASELINE.json configs)",
        "config": {"workload": cfg.desc, "config": cfg.name,
                   "points_per_step_per_gpu": wl.points_per_step,
                   "points_per_s": value / (cfg.n_max + 1 if cfg.n_max >= 0 else 1),
                   "l2": "inputs 512 MiB and outputs 9.1 GB per step exceed the 126 MB L2; "
                         "no flush" if cfg.name == "cfg3" else "inputs/outputs exceed L2",
                   "parallelism": f"dp{ctx.ws} (contiguous shards, no data-path collective)"},
        "roofline": roof,
        "clocks": res["clocks"],
        "gpu_launches": res["launches"],
        "gpu_launches_per_step": {"evaluator": res["kernels_per_step"], "shard_error": 1},
        "accuracy": accuracy_obj(wl, res),
        "per_rank": {"secs": ctx.gather_list(res["local_secs"]),
                     "values": ctx.gather_list(float(wl.values_per_step * args.steps))},
    }

    # end-to-end (host buffers through the C-ABI), rank-local then summed
    try:
        e2e = (e2e_dense(args.config, args.e2e_steps, dev)
               if cfg.layout != "ragged" and args.e2e_steps > 0 else None)
        if e2e:
            e2e["value"] = ctx.sum(e2e["value"])
        line["e2e"] = e2e
    except Exception as ex:  # noqa: BLE001
        line["e2e"] = {"error": str(ex)[:200]}

    # CPU baselines: the C port and the reference's mpmath path, rank 0 at N=1 only
    if ctx.rank == 0 and ctx.ws == 1 and cfg.layout != "ragged" and args.cpu_seconds > 0:
        from paper_2504_07637_b200 import boys
        xd = wl.xs[0][: 1 << 21]
        xs = xd.cpu().numpy()
        g = boys(cfg.n_max, xd, layout=cfg.layout).cpu().numpy()
        v, cores, reps, ulp = cpu_port_rate(cfg.n_max, xs, cfg.layout, args.cpu_seconds, g)
        line["cpu_baseline"] = {"value": v, "unit": UNIT, "cores": cores, "kind": "port",
                                "cpu_model": cpu_model(),
                                "sample": f"{reps} x 2^21 points of {cfg.name} "
                                          f"(~{args.cpu_seconds:.0f} s), OpenMP all threads",
                                "max_ulp_gpu_vs_port": ulp}
        if args.mpmath:
            try:
                line["cpu_baseline_reference"] = reference_mpmath_rate(cfg.name)
            except Exception as ex:  # noqa: BLE001
                line["cpu_baseline_reference"] = {"error": str(ex)[:200]}
    try:
        ulp, npts = wl.port_compare()
        line["accuracy"]["max_ulp_vs_port"] = ctx.max(float(ulp))
        line["accuracy"]["port_compare_points_per_rank"] = npts
    except Exception as ex:  # noqa: BLE001
        line["accuracy"]["port_compare_error"] = str(ex)[:200]

    # the other BASELINE configurations (same protocol, fewer steps)
    extras_list = (args.extras.split(",") if args.extras else
                   (["cfg1", "cfg1_l2flush", "cfg1_2p24", "cfg2", "cfg4", "cfg4f32", "cfg5", "split",
                     "hermite"]
                    if ctx.ws == 1 else ["cfg5"]))
    if not args.no_extras:
        extras = {}
        del wl
        torch.cuda.empty_cache()
        # 1 GiB (8x L2): flushes L2 and keeps the GPU busy long enough that
        # the host has enqueued the next launch before the timed event fires
        flushbuf = torch.empty(1 << 30, dtype=torch.uint8, device=dev)
        # cfg1 (2^20 points, 16 MiB in+out) two ways: (a) a stream of 32 distinct
        # batches launched back to back from one CUDA graph (host launch cost
        # off the GPU's critical path; 512 MiB working set, each batch cold
        # in L2 when its launch starts); (b) one batch, L2 flushed before every
        # launch (also evicts code and __constant__ tables)
        # cfg2 (1.3 GB per launch): two distinct batches per step, outputs
        # alternating, so dirty L2 lines of one launch are written back during
        # the next instead of being overwritten in L2 (which would flatter HBM)
        plan = {"cfg1": ("cfg1", 32, "graph"), "cfg1_l2flush": ("cfg1", 1, "flush"),
                "cfg2": ("cfg2", 2, None),
                # the n=0 kernel at steady state: cfg1's distribution, 2^24-point
                # batches (27 waves: no per-launch ramp/tail), two alternating
                "cfg1_2p24": ("cfg1", 2, None, 1 << 24)}
        for key in extras_list:
            if key == "hermite":
                try:
                    extras[key] = hermite_line(ctx, min(args.steps, 50), args.warmup, hbm_peak,
                                               fp64_peak)
                except Exception as ex:  # noqa: BLE001
                    extras[key] = {"error": str(ex)[:300]}
                continue
            name, rot, fl, npts = (plan.get(key, (key, 1, None)) + (None,))[:4]
            if name == args.config:
                continue
            try:
                w2 = make_workload(name, ctx, n_points=npts, rotate=rot)
                k = min(args.steps, 50) if name != "cfg1" else (100 if rot > 1 else 200)
                r2 = time_workload(w2, ctx, k, args.warmup,
                                   flush=(lambda: flushbuf.zero_()) if fl == "flush" else None,
                                   graph=fl == "graph")
                v2 = ctx.sum(w2.values_per_step * k) / r2["secs"]
                if fl == "flush":
                    note = "flushed (1 GiB memset) before every launch; kernel time only"
                elif rot > 1 and fl == "graph":
                    note = (f"{rot} distinct batches per step, launched back to back as one "
                            "CUDA-graph replay "
                            f"({rot} x {w2.bytes_per_point * w2.points_per_step / rot / 2**20:.0f} MiB "
                            "working set > L2)")
                elif key == "cfg1_2p24":
                    note = ("cfg1's distribution at 2^24 points per batch (not the config's "
                            "2^20): the kernel without per-launch ramp and tail; "
                            f"{rot} alternating batches with their own outputs (> L2)")
                elif rot > 1:
                    note = (f"{rot} distinct batches per step with their own outputs "
                            f"({w2.bytes_per_point * w2.points_per_step / rot / 2**30:.2f} GiB per "
                            "launch, > L2; no output is rewritten while its dirty lines sit in L2)")
                else:
                    note = "exceeds L2"
                if name == "split":
                    note = "eval_with_split(16, 8) on the cfg3 inputs, AoS [N][17]; exceeds L2"
                e = {"value": v2, "unit": UNIT, "steps": k, "n_gpus": ctx.ws,
                     "ms_per_step": r2["secs"] / k * 1e3, "scaling": w2.scaling,
                     "gpu_launches": r2["launches"],
                     "roofline": roofline_obj(w2, r2["per_launch_ms"], hbm_peak, fp64_peak,
                                              traffic=committed_traffic(key)),
                     "accuracy": accuracy_obj(w2, r2), "l2": note}
                if rot > 1:
                    e["launches_per_step"] = rot
                try:
                    ulp, npts = w2.port_compare()
                    e["accuracy"]["max_ulp_vs_port"] = ctx.max(float(ulp))
                    e["accuracy"]["port_compare_points_per_rank"] = npts
                except Exception as ex:  # noqa: BLE001
                    e["accuracy"]["port_compare_error"] = str(ex)[:200]
                if name in ("cfg4", "cfg4f32"):
                    oms, same = w2.offsets_ms()
                    e["offsets_ms"] = round(oms, 4)
                    e["offsets_bit_identical"] = same
                    e["offsets_elements"] = int(w2.x.numel())
                    if args.e2e_steps > 0:
                        try:
                            e["e2e"] = e2e_ragged(w2, max(1, args.e2e_steps))
                        except Exception as ex:  # noqa: BLE001
                            e["e2e"] = {"error": str(ex)[:200]}
                extras[key] = e
                del w2
                torch.cuda.empty_cache()
            except Exception as ex:  # noqa: BLE001
                extras[key] = {"error": str(ex)[:300]}
        line["configs"] = extras

    if fp64_peak:
        line["fp64_peak_measured_ops_per_s"] = fp64_peak
    if ctx.rank == 0:
        print(json.dumps(line), flush=True)
    ctx.close()


if __name__ == "__main__":
    main()
