"""Launch each config's kernel a few times (for ncu capture / launch lists)."""
import argparse
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2504_07637_b200 import boys, boys_ragged, eval_with_split, ragged_offsets  # noqa: E402
from paper_2504_07637_b200 import workloads as W  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--configs", default="cfg3,cfg1,cfg2,cfg4,cfg4f32")
ap.add_argument("--launches", type=int, default=3)
a = ap.parse_args()
dev = torch.device("cuda:0")
for name in a.configs.split(","):
    if name == "hermite":                    # fused consumer, 4096^2 quartets at L = 4
        from paper_2504_07637_b200 import hermite_coulomb
        b, k = W.shell_pairs(4096, seed=21, device=dev), W.shell_pairs(4096, seed=22, device=dev)
        for _ in range(a.launches):
            hermite_coulomb(4, b, k, check=False)
        torch.cuda.synchronize()
        print(name, "ok", flush=True)
        continue
    if name == "split":                      # eval_with_split(16, 8) on the cfg3 inputs, AoS
        x = W.config_x("cfg3", device=dev)
        out = torch.empty((x.numel(), 17), dtype=torch.float64, device=dev)
        for _ in range(a.launches):
            eval_with_split(16, 8, x, layout="aos", check=False, out=out)
        torch.cuda.synchronize()
        print(name, "ok", flush=True)
        continue
    c = W.CONFIGS[name]
    if c.layout == "ragged":
        x, nm = (W.cfg4f32_batch if c.dtype == torch.float32 else W.cfg4_batch)(c.N, device=dev)
        off = ragged_offsets(nm)
        out = torch.empty(int(off[-1]), dtype=c.dtype, device=dev)
        for _ in range(a.launches):
            boys_ragged(x, nm, off, out=out, check=False)
    else:
        x = W.config_x(name, n=min(c.N, W.CHUNK), device=dev)
        for _ in range(a.launches):
            boys(c.n_max, x, layout=c.layout, check=False)
    torch.cuda.synchronize()
    print(name, "ok", flush=True)
