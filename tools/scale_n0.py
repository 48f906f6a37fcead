"""n=0 kernel time vs batch size: separates the fixed launch/ramp cost from the
asymptotic FP64 throughput (config 1 is 2^20 points)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
from paper_2504_07637_b200 import boys, roofline as R, workloads as W

dev = torch.device("cuda:0")
flush = torch.empty(1 << 30, dtype=torch.uint8, device=dev)
ops = R.ops_per_point(0)
for lg in (8, 12, 16, 18, 20, 22, 24, 26):
    N = 1 << lg
    x = W.cfg1_x(N, device=dev)
    out = torch.empty((1, N), dtype=torch.float64, device=dev)
    for _ in range(3):
        boys(0, x, out=out, check=False)
    ts = []
    for _ in range(20):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); boys(0, x, out=out, check=False); b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    ms = sorted(ts)[len(ts) // 2]
    print(f"N=2^{lg}: {ms * 1e3:9.2f} us   {N / ms / 1e6:8.2f} Gpts/s   "
          f"{N * ops / (ms * 1e-3) / 1e12:6.2f} T algorithmic DP ops/s", flush=True)
