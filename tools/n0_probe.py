"""Decompose the cfg1 (n=0, 2^20 points) single-launch time: event-timed single
launches with (a) L2 flushed (x, tables and code cold), (b) the same batch
again (everything warm), (c) a fresh batch each launch with only the tables
warm (x cold), (d) back-to-back launches of distinct batches (host-launched,
no graph).  Prints one JSON line of microseconds."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2504_07637_b200 import boys, workloads as W  # noqa: E402

dev = torch.device("cuda:0")
xs = [W.config_x("cfg1", device=dev, chunk=k) for k in range(40)]
out = torch.empty_like(xs[0]).reshape(1, -1)
flush = torch.empty(1 << 30, dtype=torch.uint8, device=dev)
ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731


def one(x, pre=None):
    if pre:
        pre()
    a, b = ev(), ev()
    a.record()
    boys(0, x, out=out[:, :x.numel()], check=False)
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) * 1e3


for _ in range(5):
    one(xs[0])
res = {"env": {k: v for k, v in os.environ.items() if k.startswith("BOYS_")}}
# a spin kernel ahead of each timed launch keeps the GPU busy while the host
# enqueues it, so the events bracket GPU time only
spin = lambda: torch.cuda._sleep(400000)  # noqa: E731
res["flushed"] = round(sorted(one(xs[0], lambda: (flush.zero_(), spin())) for _ in range(30))[15], 2)
res["warm_same_batch"] = round(sorted(one(xs[0], spin) for _ in range(30))[15], 2)
res["x_cold_tables_warm"] = round(sorted(one(xs[k], spin) for k in range(1, 33))[16], 2)
tiny = xs[0][:1024].clone()
res["tiny_1024_points"] = round(sorted(one(tiny, spin) for _ in range(30))[15], 2)
torch.cuda.synchronize()
a, b = ev(), ev()
a.record()
for k in range(32):
    boys(0, xs[k], out=out, check=False)
b.record()
torch.cuda.synchronize()
res["back_to_back_per_launch"] = round(a.elapsed_time(b) * 1e3 / 32, 2)
print(json.dumps(res), flush=True)
