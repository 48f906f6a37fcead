"""cfg4 / cfg4f32 ragged kernel timing (back-to-back launches, CUDA events),
one JSON line; the kernel variant is chosen by the environment (A/B)."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2504_07637_b200 import boys_ragged, ragged_offsets, workloads as W  # noqa: E402

res = {"env": {k: v for k, v in os.environ.items() if k.startswith("BOYS_")}}
for tag in sys.argv[1:] or ["cfg4", "cfg4f32"]:
    c = W.CONFIGS[tag]
    x, nm = (W.cfg4f32_batch if tag == "cfg4f32" else W.cfg4_batch)(c.N, device="cuda")
    off = ragged_offsets(nm)
    out = torch.empty(int(off[-1]), dtype=x.dtype, device="cuda")
    for _ in range(3):
        boys_ragged(x, nm, off, out=out, check=False)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(20):
        boys_ragged(x, nm, off, out=out, check=False)
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / 20
    es = x.element_size()
    nbytes = x.numel() * (es + 1 + 8) + out.numel() * es
    res[tag] = {"ms": round(ms, 4), "hbm_frac": round(nbytes / (ms * 1e-3) / 6547.2e9, 4),
                "values": out.numel()}
print(json.dumps(res), flush=True)
