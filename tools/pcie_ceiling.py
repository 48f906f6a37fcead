"""Host link ceilings: pinned cudaMemcpyAsync D2H / H2D (the e2e path's bound)."""
import torch

dev = torch.device("cuda:0")
n = 2 << 30
d = torch.empty(n, dtype=torch.uint8, device=dev)
h = torch.empty(n, dtype=torch.uint8, pin_memory=True)
for name, fn in (("D2H", lambda: h.copy_(d, non_blocking=True)),
                 ("H2D", lambda: d.copy_(h, non_blocking=True))):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(5):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); fn(); b.record(); torch.cuda.synchronize()
        best = min(best, a.elapsed_time(b))
    print(f"{name} pinned 2 GiB: {n / best / 1e6:.1f} GB/s", flush=True)
