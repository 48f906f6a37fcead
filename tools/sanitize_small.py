"""Small launches of every kernel path (for compute-sanitizer): dense SoA/AoS
(f64/f32, full and tail tiles, unaligned out), ragged (fast path, deferred
queue drains, high-order fallback), split, ragged offsets, host pipeline."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch
from paper_2504_07637_b200 import boys, boys_ragged, eval_with_split, max_order

dev = torch.device("cuda:0")
rng = np.random.default_rng(0)
for dt in (torch.float64, torch.float32):
    for N in (1, 255, 256, 3000):
        x = torch.from_numpy(rng.uniform(0, 90, N)).to(dev, dt)
        for n in (0, 3, 8, max_order(dt)):
            for lay in ("soa", "aos"):
                boys(n, x, layout=lay)
    base = torch.empty(3000 * 17 + 1, dtype=dt, device=dev)
    boys(16, torch.from_numpy(rng.uniform(0, 90, 3000)).to(dev, dt), layout="aos",
         out=base[1:].view(3000, 17))
    for cap in (12, max_order(dt)):
        M = 5000
        xr = torch.from_numpy(np.exp(rng.uniform(np.log(1e-3), np.log(1e4), M))).to(dev, dt)
        nr = torch.from_numpy(rng.integers(0, cap + 1, M).astype(np.uint8)).to(dev)
        boys_ragged(xr, nr)
    eval_with_split(8, 3, torch.from_numpy(rng.uniform(0, 90, 1000)).to(dev, dt))
boys(12, rng.uniform(0, 90, (1 << 22) + 5))       # host pipeline, two chunks
torch.cuda.synchronize()
print("sanitize driver ok")
