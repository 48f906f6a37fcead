"""HBM ceilings on this box: copy (read+write, the MEASURED_PEAKS method) and
write-only (memset) over the cfg3 output size."""
import torch

dev = torch.device("cuda:0")
nbytes = 9_663_676_416           # cfg3 bytes per launch (0.54 GB in + 9.13 GB out)
buf = torch.empty(nbytes, dtype=torch.uint8, device=dev)
src = torch.empty(1 << 30, dtype=torch.bfloat16, device=dev)
dst = torch.empty_like(src)


def timeit(fn, reps=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); fn(); b.record(); torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return min(ts), sorted(ts)[len(ts) // 2]


mn, md = timeit(lambda: buf.fill_(1))
print(f"write-only memset {nbytes/1e9:.2f} GB: best {nbytes/mn/1e6:.0f} GB/s, median {nbytes/md/1e6:.0f} GB/s")
mn, md = timeit(lambda: dst.copy_(src))
cb = 2 * src.numel() * 2
print(f"copy 1Gi bf16 (read+write {cb/1e9:.2f} GB): best {cb/mn/1e6:.0f} GB/s, median {cb/md/1e6:.0f} GB/s")
