"""eval_with_split timing per layout (graph-free, back-to-back launches)."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2504_07637_b200 import eval_with_split, workloads as W  # noqa: E402

res = {}
for lay in ("soa", "aos"):
    for n, nb in ((16, 8), (12, 11), (8, 4)):
        x = W.cfg3_x(1 << 24, device="cuda")
        out = torch.empty(((n + 1, x.numel()) if lay == "soa" else (x.numel(), n + 1)),
                          dtype=torch.float64, device="cuda")
        for _ in range(3):
            eval_with_split(n, nb, x, layout=lay, check=False, out=out)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(10):
            eval_with_split(n, nb, x, layout=lay, check=False, out=out)
        b.record()
        torch.cuda.synchronize()
        ms = a.elapsed_time(b) / 10
        res[f"{lay}_{n}_{nb}"] = {"ms": round(ms, 4),
                                  "hbm_frac": round((8 + 8 * (n + 1)) * x.numel() / (ms * 1e-3) / 6547e9, 3)}
print(json.dumps(res))
