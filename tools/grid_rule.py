"""Persistent grid vs one block per tile, per (order, N, layout): per-launch
microseconds of a graph-replayed stream of distinct batches (BOYS_GRID_TILES
is read once per process, so run this once per setting)."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2504_07637_b200 import _lib, boys  # noqa: E402

_lib.load(build_if_missing=False)
res = {}
CASES = [(0, "soa", 18), (0, "soa", 20), (0, "soa", 22), (0, "soa", 24),
         (4, "soa", 20), (8, "soa", 20), (8, "soa", 22), (16, "soa", 20)]
if len(sys.argv) > 1:      # e.g. "0,2,4,6,8,10,12,16:22,24"
    ns, lgs = sys.argv[1].split(":")
    LAY = os.environ.get("LAYOUT", "soa")
    CASES = [(int(n), LAY, int(lg)) for lg in lgs.split(",") for n in ns.split(",")]
DT = torch.float32 if os.environ.get("DTYPE") == "f32" else torch.float64
for n, lay, lg in CASES:
    N = 1 << lg
    rot = max(2, min(32, (1 << 29) // (N * 8 * (n + 2))))
    g = torch.Generator(device="cuda").manual_seed(n * 100 + lg)
    xs = [(torch.rand(N, dtype=torch.float64, device="cuda", generator=g) * 60).to(DT)
          for _ in range(rot)]
    shape = (n + 1, N) if lay == "soa" else (N, n + 1)
    outs = [torch.empty(shape, dtype=DT, device="cuda") for _ in range(rot)]
    for x, o in zip(xs, outs):
        boys(n, x, layout=lay, out=o, check=False)
    torch.cuda.synchronize()
    gr = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gr):
        for x, o in zip(xs, outs):
            boys(n, x, layout=lay, out=o, check=False)
    for _ in range(3):
        gr.replay()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = max(3, 2000 // rot)
    a.record()
    for _ in range(reps):
        gr.replay()
    b.record()
    torch.cuda.synchronize()
    res[f"n{n}_{lay}_2^{lg}"] = round(1e3 * a.elapsed_time(b) / (reps * rot), 2)
    del xs, outs, gr
    torch.cuda.empty_cache()
print(json.dumps({"grid_tiles": os.environ.get("BOYS_GRID_TILES", "0"),
                  "dtype": str(DT), **res}))
