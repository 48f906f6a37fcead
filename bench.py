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
scaling: each rank owns its own 2^26-point chunk, keyed by rank).

Timing: W untimed warm-up steps, barrier + synchronize, K timed steps with
CUDA events on the launching stream, synchronize + barrier; the job time is
the max over ranks.  value = F-values/s over all ranks.

Also reported: roofline of the dominant kernel (algorithmic bytes / measured
launch time vs the measured HBM copy bandwidth), SM clocks sampled through
NVML during the timed region, the end-to-end number through the host-buffer
C-ABI entry (pinned host x in, full result out, copies inside the timed
region), the CPU baseline (the C oracle on the host cores, bounded sample),
and per-config lines for the other BASELINE configurations.

``--impl reference`` times the reference's CPU implementation of the path:
the reference ships no finite-precision evaluator (only mpmath), so this is
the C restatement in oracle/ running on all host cores (kind "port"), on a
bounded sample of the same workload per step.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
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
# infrastructure
# ----------------------------------------------------------------------------

def _dist_on() -> bool:
    import torch.distributed as dist
    return dist.is_available() and dist.is_initialized()


def dist_setup(gpus: int):
    """One process per GPU.  Under torchrun (RANK set) the NCCL group is
    created even at world size 1, so the barrier / max-over-ranks / gather
    paths are the same code at every N."""
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if "RANK" in os.environ:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    return rank, ws, local


def barrier(ws):
    if _dist_on():
        import torch.distributed as dist
        dist.barrier()


def max_over_ranks(v: float, ws: int) -> float:
    if not _dist_on():
        return v
    import torch.distributed as dist
    t = torch.tensor([v], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def sum_over_ranks(v: float, ws: int) -> float:
    if not _dist_on():
        return v
    import torch.distributed as dist
    t = torch.tensor([v], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())


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
    """dram bytes per launch of the dominant kernel from the committed ncu summary."""
    p = ROOT / "profiles" / "ncu_traffic.json"
    if p.exists():
        d = json.loads(p.read_text())
        return d.get(config)
    return None


# ----------------------------------------------------------------------------
# workloads
# ----------------------------------------------------------------------------

class Dense:
    """Dense config: one or more 2^26-point chunks per rank."""

    def __init__(self, cfg, rank, ws, dev, n_points=None, rotate=1):
        from paper_2504_07637_b200 import workloads as W
        self.cfg = cfg
        self.n = cfg.n_max
        self.layout = cfg.layout
        total = n_points or cfg.N
        if cfg.name == "cfg5":          # strong scaling: shard 2^30 contiguously
            from paper_2504_07637_b200 import shard as S
            plan = S.chunk_plan(total, rank, ws, W.CHUNK)
            self.chunks = [cid for cid, _, _ in plan]
            self.xs = [W.config_x("cfg5", n=W.CHUNK, chunk=cid, device=dev)[lo - cid * W.CHUNK:
                                                                          hi - cid * W.CHUNK]
                       for cid, lo, hi in plan]
            self.outs = [torch.empty(self._shape(W.CHUNK), dtype=torch.float64, device=dev)
                         for _ in range(2)]
            self.scaling = "strong"
        else:                            # weak: each rank its own chunk(s)
            # rotate > 1: that many distinct batches (and outputs) per step, so a
            # small config streams through a working set larger than L2
            self.xs = [W.config_x(cfg.name, n=total, chunk=rank * rotate + j, device=dev)
                       for j in range(rotate)]
            self.outs = [torch.empty(self._shape(total), dtype=torch.float64, device=dev)
                         for _ in range(rotate)]
            self.scaling = "weak"
        self.points_per_step = sum(x.numel() for x in self.xs)
        self.values_per_step = self.points_per_step * (self.n + 1)
        from paper_2504_07637_b200 import roofline as R
        self.bytes_per_point = R.dense_bytes_per_point(self.n)
        self.ops_per_point = R.ops_per_point(self.n)

    def _shape(self, N):
        return (N, self.n + 1) if self.layout == "aos" else (self.n + 1, N)

    def launches(self):
        from paper_2504_07637_b200 import boys
        for k, x in enumerate(self.xs):
            out = self.outs[k % len(self.outs)]
            if self.layout == "aos":
                out = out[: x.numel()]          # contiguous prefix for a partial chunk
            yield lambda x=x, out=out: boys(self.n, x, layout=self.layout, out=out, check=False)


class Ragged:
    def __init__(self, cfg, rank, ws, dev, n_points=None):
        from paper_2504_07637_b200 import ragged_offsets, roofline as R, workloads as W
        N = n_points or cfg.N
        if cfg.dtype == torch.float32:
            self.x, self.nm = W.cfg4f32_batch(N, chunk=rank, device=dev)
        else:
            self.x, self.nm = W.cfg4_batch(N, chunk=rank, device=dev)
        self.off = ragged_offsets(self.nm)
        total = int(self.off[-1].item())
        self.out = torch.empty(total, dtype=cfg.dtype, device=dev)
        self.points_per_step = self.x.numel()
        self.values_per_step = total
        eb = 8 if cfg.dtype == torch.float64 else 4
        self.bytes_total = R.ragged_bytes(self.x.numel(), total, eb)
        self.bytes_per_point = self.bytes_total / self.x.numel()
        self.ops_per_point = None
        self.scaling = "weak"

    def launches(self):
        from paper_2504_07637_b200 import boys_ragged
        yield lambda: boys_ragged(self.x, self.nm, self.off, out=self.out, check=False)


class Split(Dense):
    """eval_with_split(16, 8) on the cfg3 inputs, point-major [N][17] (the
    SPEC's two-seed accuracy option; same bytes per point as cfg3)."""

    def __init__(self, rank, ws, dev):
        from paper_2504_07637_b200 import workloads as W
        super().__init__(W.CONFIGS["cfg3"], rank, ws, dev)
        self.n_bar = 8

    def launches(self):
        from paper_2504_07637_b200 import eval_with_split
        x, out = self.xs[0], self.outs[0]
        yield lambda: eval_with_split(self.n, self.n_bar, x, layout="aos", check=False, out=out)


def make_workload(name, rank, ws, dev, n_points=None, rotate=1):
    from paper_2504_07637_b200 import workloads as W
    cfg = W.CONFIGS[name]
    if cfg.layout == "ragged":
        return Ragged(cfg, rank, ws, dev, n_points)
    return Dense(cfg, rank, ws, dev, n_points, rotate=rotate)


def time_workload(wl, steps, warmup, ws, local, flush=None, sample_clocks=False, graph=False):
    """Returns (job seconds (max over ranks), per-launch ms list, clocks, launches).

    graph=True: the step's launches are captured once into a CUDA graph and
    each step is one replay (for small batches whose host-side launch cost
    would otherwise starve the GPU); per-launch time = replay time / launches.
    """
    from paper_2504_07637_b200 import _lib
    fns = list(wl.launches())
    for _ in range(warmup):
        for f in fns:
            f()
    torch.cuda.synchronize()
    if graph:
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            for f in fns:
                f()
        torch.cuda.synchronize()
        for _ in range(warmup):
            g.replay()
        torch.cuda.synchronize()
        fns = [g.replay]
    barrier(ws)
    torch.cuda.synchronize()
    stream = torch.cuda.current_stream()
    evs = []
    l0 = _lib.launch_count()
    sampler = ClockSampler(local) if sample_clocks else None
    ctx = sampler if sampler else _Null()
    with ctx:
        t_start = torch.cuda.Event(enable_timing=True)
        t_end = torch.cuda.Event(enable_timing=True)
        t_start.record(stream)
        for _ in range(steps):
            for f in fns:
                if flush is not None:
                    flush()
                a = torch.cuda.Event(enable_timing=True)
                b = torch.cuda.Event(enable_timing=True)
                a.record(stream)
                f()
                b.record(stream)
                evs.append((a, b))
        t_end.record(stream)
        torch.cuda.synchronize()
    barrier(ws)
    launches = _lib.launch_count() - l0
    per = [a.elapsed_time(b) for a, b in evs]
    if graph:      # kernels launched by the replays (the host counter sees none)
        nk = len(list(wl.launches()))
        launches = steps * nk
        per = [p / nk for p in per]
    if flush is not None:     # job time = kernel time only (flushes excluded)
        secs = sum(per) / 1e3
    else:
        secs = t_start.elapsed_time(t_end) / 1e3
    secs = max_over_ranks(secs, ws)
    clocks = sampler.summary() if sampler else None
    return secs, per, clocks, launches


class _Null:
    def __enter__(self):
        return self

    def __exit__(self, *a):
        pass


def roofline_obj(wl, per_ms, hbm_peak, fp64_peak, bound=None, traffic=None):
    launch_ms = statistics.mean(per_ms)
    pts = wl.points_per_step / max(1, len(list(wl.launches())))
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


# ----------------------------------------------------------------------------
# CPU baseline / reference arm (oracle port on host cores)
# ----------------------------------------------------------------------------

def cpu_port_rate(n, x_host, layout, min_seconds=10.0, gpu_out=None):
    """Times the C restatement on the host cores.  gpu_out (the GPU's values for
    the same sample): the baseline's own output is also the parity checker --
    returns the max |GPU - CPU| in ulp over the sample (0 = bit-identical)."""
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
    ulp = None
    if gpu_out is not None:
        a = gpu_out.view(np.int64).astype(np.int64)
        b = ref.view(np.int64).astype(np.int64)
        both_nan = np.isnan(gpu_out) & np.isnan(ref)
        ulp = int(np.where(both_nan, 0, np.abs(a - b)).max(initial=0))
    return reps * x_host.size * (n + 1) / el, O.threads(), reps, ulp


def run_reference(args, rank, ws):
    """--impl reference: the C oracle port on all host cores; rank 0 only."""
    if rank != 0:
        return
    from oracle import oracle as O
    from paper_2504_07637_b200 import workloads as W
    cfg = W.CONFIGS[args.config]
    sample = 1 << 20
    x = W.config_x(args.config, n=sample, chunk=0, device="cpu").numpy()
    if cfg.dtype == torch.float32:
        x = x.astype(np.float32)
    for _ in range(args.warmup):
        O.dense(cfg.n_max, x, cfg.layout)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        O.dense(cfg.n_max, x, cfg.layout)
    el = time.perf_counter() - t0
    v = args.steps * sample * (cfg.n_max + 1) / el
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": el / args.steps * 1e3, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": cfg.desc, "config": cfg.name,
                   "points_per_step": sample},
        "cpu_baseline": {"value": v, "unit": UNIT, "cores": O.threads(), "kind": "port",
                         "sample": f"{sample} points of {cfg.name} per step, all host threads; "
                                   "C restatement of the SPEC kernel (reference ships no "
                                   "finite-precision evaluator)"},
        "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
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


def golden_check(cfg_name, rank, ws, dev):
    """Max relative error vs refmath.boys_downward goldens (tests/golden,
    double-double), gathered over ranks with all_gather (1 fp64 per rank)."""
    import math
    from paper_2504_07637_b200 import boys, shard as S, workloads as W
    cfg = W.CONFIGS[cfg_name]
    if cfg.layout == "ragged":
        return None
    d = np.load(ROOT / "tests" / "golden" / "configs.npz")
    gx = torch.from_numpy(d[f"{cfg_name}_x"]).to(dev)
    gF = torch.from_numpy(d[f"{cfg_name}_F"]).to(dev)
    err = S.golden_error(cfg.n_max, gx, gF, rank, ws,
                         lambda n, x: boys(n, x.contiguous(), layout="aos"))
    per_rank, mx = S.gather_max(err)
    return {"golden_points": int(gx.numel()), "max_rel_err": mx,
            "bits": (-math.log2(mx) if mx > 0 else None), "per_rank": per_rank,
            "reference": "refmath.boys_downward(n, x, Precision(96)), tests/golden/configs.npz"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=300)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="cfg3")
    ap.add_argument("--no-extras", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)

    if args.impl == "reference":
        rank = int(os.environ.get("RANK", "0"))
        ws = int(os.environ.get("WORLD_SIZE", "1"))
        run_reference(args, rank, ws)
        return

    rank, ws, local = dist_setup(args.gpus)
    dev = torch.device("cuda", torch.cuda.current_device())
    from paper_2504_07637_b200 import _lib, workloads as W
    _lib.load(build_if_missing=False)
    hbm_peak, hbm_src = measured_peaks()
    fp64_peak = fp64_peak_probe()

    wl = make_workload(args.config, rank, ws, dev)
    secs, per, clocks, launches = time_workload(wl, args.steps, args.warmup, ws, local,
                                                sample_clocks=True)
    total_values = sum_over_ranks(wl.values_per_step * args.steps, ws)
    value = total_values / secs
    roof = roofline_obj(wl, per, hbm_peak, fp64_peak, traffic=committed_traffic(args.config))
    roof["peak_source"] = roof.get("peak_source", hbm_src)
    cfg = W.CONFIGS[args.config]

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": secs / args.steps * 1e3,
        "higher_is_better": True, "scaling": wl.scaling, "vs_baseline": None,
        "dtype": "f64" if cfg.dtype == torch.float64 else "f32",
        "data": "synthetic (seeded generators of BASELINE.json configs)",
        "config": {"workload": cfg.desc, "config": cfg.name,
                   "points_per_step_per_gpu": wl.points_per_step,
                   "points_per_s": value / (cfg.n_max + 1 if cfg.n_max >= 0 else 1),
                   "l2": "inputs 512 MiB and outputs 9.1 GB per step exceed the 126 MB L2; "
                         "no flush" if cfg.name == "cfg3" else "inputs/outputs exceed L2",
                   "parallelism": f"dp{ws} (contiguous shards, no collective)"},
        "roofline": roof,
        "clocks": clocks,
        "gpu_launches": launches,
    }

    # accuracy: each rank checks its slice of the reference-golden sample on
    # the device; one fp64 per rank is gathered (the path's only collective)
    try:
        line["accuracy"] = golden_check(args.config, rank, ws, dev)
    except Exception as ex:  # noqa: BLE001
        line["accuracy"] = {"error": str(ex)[:200]}

    # end-to-end (host buffers through the C-ABI), rank-local then summed
    try:
        e2e = (e2e_dense(args.config, args.e2e_steps, dev)
               if cfg.layout != "ragged" and args.e2e_steps > 0 else None)
        if e2e:
            e2e["value"] = sum_over_ranks(e2e["value"], ws)
        line["e2e"] = e2e
    except Exception as ex:  # noqa: BLE001
        line["e2e"] = {"error": str(ex)[:200]}

    # CPU baseline: the C oracle on the host cores, rank 0 at N=1 only
    if rank == 0 and ws == 1 and cfg.layout != "ragged" and args.cpu_seconds > 0:
        from paper_2504_07637_b200 import boys
        xd = wl.xs[0][: 1 << 21]
        xs = xd.cpu().numpy()
        g = boys(cfg.n_max, xd, layout=cfg.layout).cpu().numpy()
        v, cores, reps, ulp = cpu_port_rate(cfg.n_max, xs, cfg.layout, args.cpu_seconds, g)
        line["cpu_baseline"] = {"value": v, "unit": UNIT, "cores": cores, "kind": "port",
                                "sample": f"{reps} x 2^21 points of {cfg.name} "
                                          f"(~{args.cpu_seconds:.0f} s), OpenMP all threads",
                                "max_ulp_gpu_vs_port": ulp}

    # the other BASELINE configurations (same protocol, fewer steps)
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
        # in L2 when its launch starts; code and tables stay warm, as in a
        # real stream of batches); (b) one batch, L2 flushed before every
        # launch (also evicts code and __constant__ tables: includes the cold
        # fetch latency of an isolated launch)
        plan = [("cfg1", "cfg1", 32, "graph"), ("cfg1_l2flush", "cfg1", 1, "flush")]
        plan += [(n, n, 1, None) for n in ("cfg2", "cfg4", "cfg4f32", "cfg5", "split")]
        for key, name, rot, fl in plan:
            if name == args.config:
                continue
            try:
                w2 = (Split(rank, ws, dev) if name == "split"
                      else make_workload(name, rank, ws, dev, rotate=rot))
                k = min(args.steps, 50) if name != "cfg1" else (100 if rot > 1 else 200)
                s2, p2, _, l2 = time_workload(
                    w2, k, args.warmup, ws, local,
                    flush=(lambda: flushbuf.zero_()) if fl == "flush" else None,
                    graph=fl == "graph")
                v2 = sum_over_ranks(w2.values_per_step * k, ws) / s2
                if fl == "flush":
                    note = "flushed (1 GiB memset) before every launch; kernel time only"
                elif rot > 1:
                    note = (f"{rot} distinct batches per step, launched back to back as one "
                            "CUDA-graph replay "
                            f"({rot} x {w2.bytes_per_point * w2.points_per_step / rot / 2**20:.0f} MiB "
                            "working set > L2)")
                else:
                    note = "exceeds L2"
                if name == "split":
                    note = ("eval_with_split(16, 8) on the cfg3 inputs, AoS [N][17]; "
                            "exceeds L2")
                extras[key] = {"value": v2, "unit": UNIT, "steps": k,
                               "ms_per_step": s2 / k * 1e3, "scaling": w2.scaling,
                               "gpu_launches": l2,
                               "roofline": roofline_obj(w2, p2, hbm_peak, fp64_peak,
                                                        traffic=committed_traffic(name)),
                               "l2": note}
                if rot > 1:
                    extras[key]["launches_per_step"] = rot
                if name in ("cfg4", "cfg4f32") and args.e2e_steps > 0:
                    try:
                        extras[key]["e2e"] = e2e_ragged(w2, max(1, args.e2e_steps))
                    except Exception as ex:  # noqa: BLE001
                        extras[key]["e2e"] = {"error": str(ex)[:200]}
                del w2
                torch.cuda.empty_cache()
            except Exception as ex:  # noqa: BLE001
                extras[key] = {"error": str(ex)[:300]}
        line["configs"] = extras

    if fp64_peak:
        line["fp64_peak_measured_ops_per_s"] = fp64_peak
    if rank == 0:
        print(json.dumps(line), flush=True)
    if _dist_on():
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
