"""f64 small orders at 2^24 points (the FP64-bound / mixed kernels): ms per
launch, SoA n = 0..5 and AoS n = 1..3, two alternating outputs; one JSON line."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2504_07637_b200 import boys, workloads as W  # noqa: E402

N = 1 << 24
# optional: dtype (f64 | f32) and "layout:n,n,..." groups, e.g.  f32 soa:6,8,12
dt = torch.float32 if len(sys.argv) > 1 and sys.argv[1] == "f32" else torch.float64
groups = [(g.split(":")[0], tuple(int(v) for v in g.split(":")[1].split(","))) for g in sys.argv[2:]] \
    or [("soa", (0, 1, 2, 3, 4, 5)), ("aos", (1, 2, 3))]
x = W.cfg3_x(N, device="cuda").to(dt)
res = {}
for lay, orders in groups:
    for n in orders:
        shape = (n + 1, N) if lay == "soa" else (N, n + 1)
        outs = [torch.empty(shape, dtype=dt, device="cuda") for _ in range(2)]
        for k in range(3):
            boys(n, x, layout=lay, out=outs[k % 2], check=False)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for k in range(20):
            boys(n, x, layout=lay, out=outs[k % 2], check=False)
        b.record()
        torch.cuda.synchronize()
        res[f"{lay}{n}"] = round(a.elapsed_time(b) / 20, 4)
        del outs
print(json.dumps(res), flush=True)
