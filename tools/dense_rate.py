"""cfg3 / cfg5-chunk / cfg2 dense kernel timing: back-to-back launches over two
alternating outputs (no output rewritten while its dirty lines sit in L2),
CUDA events; one JSON line with per-launch ms and the fraction of the
MEASURED_PEAKS copy bandwidth."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2504_07637_b200 import boys, eval_with_split, workloads as W  # noqa: E402

peak = 6543.7
try:
    peak = json.load(open(os.path.join(os.path.dirname(__file__), "..", "MEASURED_PEAKS.json")))["hbm_gbs"]
except Exception:  # noqa: BLE001
    pass
res = {"lib": os.environ.get("BOYS_LIB", "default"), "single_out": bool(os.environ.get("SINGLE_OUT"))}
for tag, cfg, n, lay, split in (("cfg3", "cfg3", 16, "aos", None), ("cfg5", "cfg5", 12, "aos", None),
                                ("cfg2", "cfg2", 8, "soa", None), ("split", "cfg3", 16, "aos", 8)):
    x = W.config_x(cfg, n=min(W.CONFIGS[cfg].N, W.CHUNK), device="cuda")
    N = x.numel()
    shape = (N, n + 1) if lay == "aos" else (n + 1, N)
    nout = 1 if os.environ.get("SINGLE_OUT") else 2
    outs = [torch.empty(shape, dtype=torch.float64, device="cuda") for _ in range(nout)]

    def run(k):
        if split is None:
            boys(n, x, layout=lay, out=outs[k % nout], check=False)
        else:
            eval_with_split(n, split, x, layout=lay, out=outs[k % nout], check=False)
    for k in range(4):
        run(k)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for k in range(20):
        run(k)
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / 20
    res[tag] = {"ms": round(ms, 4), "hbm_frac": round((8 + 8 * (n + 1)) * N / (ms * 1e-3) / peak / 1e9, 4)}
    del outs, x
    torch.cuda.empty_cache()
print(json.dumps(res), flush=True)
