"""Every (dtype, layout, order) at 2^24 points with the library's own kernel
choices: back-to-back launches over two alternating outputs, CUDA events.
Writes a markdown table: ms per launch, fraction of the HBM copy peak, and of
the FP64 roofline for the FP64-bound small orders.

    python tools/order_sweep.py [--out profiles/r02_order_sweep.md]
"""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2504_07637_b200 import boys, max_order, roofline as R, workloads as W  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--out", default=None)
ap.add_argument("--log2n", type=int, default=24)
a = ap.parse_args()
peak = json.load(open(os.path.join(os.path.dirname(__file__), "..", "MEASURED_PEAKS.json")))["hbm_gbs"]
fp64 = 17.0e12
N = 1 << a.log2n
rows = []
for dt in (torch.float64, torch.float32):
    x = W.cfg3_x(N, device="cuda").to(dt)
    es = x.element_size()
    for lay in ("soa", "aos"):
        for n in range(max_order(dt) + 1):
            shape = (n + 1, N) if lay == "soa" else (N, n + 1)
            outs = [torch.empty(shape, dtype=dt, device="cuda") for _ in range(2)]
            for k in range(3):
                boys(n, x, layout=lay, out=outs[k % 2], check=False)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for k in range(10):
                boys(n, x, layout=lay, out=outs[k % 2], check=False)
            e1.record()
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / 10
            hbm = (es + es * (n + 1)) * N / (ms * 1e-3) / 1e9 / peak
            ops = R.ops_per_point(n, es) * N / (ms * 1e-3) / fp64 if dt == torch.float64 else None
            rows.append((str(dt).split(".")[-1], lay, n, ms, hbm, ops))
            del outs
    del x
    torch.cuda.empty_cache()
lines = ["| dtype | layout | n | ms / launch | % HBM copy peak | % FP64 (algorithmic ops) |",
         "|---|---|---|---|---|---|"]
for d, lay, n, ms, hbm, ops in rows:
    lines.append(f"| {d} | {lay} | {n} | {ms:.4f} | {100 * hbm:.1f} | {'' if ops is None else f'{100 * ops:.1f}'} |")
text = "\n".join(lines)
print(text)
if a.out:
    open(a.out, "w").write(f"# Order sweep: every (dtype, layout, order) at 2^{a.log2n} points\n\n"
                          "`python tools/order_sweep.py` on one B200 (default kernel choices, two "
                          "alternating outputs, 10 back-to-back launches, CUDA events; inputs: "
                          "cfg3's distribution; FP64 peak 17.0 T DP ops/s).\n\n" + text + "\n")
