"""SoA write-stride experiment: kernel time vs N (power-of-two row stride or not)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
from paper_2504_07637_b200 import boys, workloads as W

dev = torch.device("cuda:0")
for N in (1 << 24, (1 << 24) + 512, (1 << 24) + 4096, (1 << 24) - 12288, 3 * (1 << 22)):
    x = W.cfg2_x(N, device=dev)
    out = torch.empty((9, N), dtype=torch.float64, device=dev)
    for _ in range(5):
        boys(8, x, out=out, check=False)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(50):
        boys(8, x, out=out, check=False)
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / 50
    gbs = N * 80 / (ms * 1e-3) / 1e9
    print(f"N={N} ({N / (1 << 24):.4f} x 2^24): {ms:.4f} ms  {gbs:.0f} GB/s  {gbs / 6542.1:.3f}", flush=True)
