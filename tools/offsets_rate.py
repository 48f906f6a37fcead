"""ragged_offsets timing at cfg4 size (2^27 orders), CUDA events, one JSON line."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2504_07637_b200 import ragged_offsets, workloads as W  # noqa: E402

x, nm = W.cfg4_batch(W.CONFIGS["cfg4"].N, device="cuda")
ref = torch.zeros(nm.numel() + 1, dtype=torch.int64, device="cuda")
torch.cumsum(nm.to(torch.int64) + 1, 0, out=ref[1:])
for _ in range(3):
    off = ragged_offsets(nm)
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(20):
    ragged_offsets(nm)
b.record()
torch.cuda.synchronize()
ms = a.elapsed_time(b) / 20
nbytes = nm.numel() + 8 * (nm.numel() + 1)
print(json.dumps({"ms": round(ms, 4), "hbm_frac": round(nbytes / (ms * 1e-3) / 6547.2e9, 3),
                  "exact": bool(torch.equal(off, ref))}), flush=True)
